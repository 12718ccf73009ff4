"""Summarise an ncu launch-list CSV (gpu__time_duration / dram bytes per launch)
into per-kernel totals: share of device time, mean duration, mean DRAM bytes.

    python scripts/summarize_launches.py launches.csv [--only REGEX]
"""
import collections
import csv
import json
import re
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    idx = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                     "Metric Value")}
    launches = collections.OrderedDict()
    for r in rows[1:]:
        lid = r[idx["ID"]]
        d = launches.setdefault(lid, {"name": r[idx["Kernel Name"]]})
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        scale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        d[r[idx["Metric Name"]]] = v * scale
    return list(launches.values())


def summarize(path, only=None):
    ls = load(path)
    agg = collections.OrderedDict()
    for d in ls:
        name = d["name"].split("(")[0].replace("void ", "")
        if only and not re.search(only, name):
            continue
        a = agg.setdefault(name, {"n": 0, "t": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["t"] += d.get("gpu__time_duration.sum", 0.0)
        a["rd"] += d.get("dram__bytes_read.sum", 0.0)
        a["wr"] += d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["t"] for a in agg.values()) or 1.0
    out = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        out.append({"kernel": k, "launches": a["n"], "share": round(a["t"] / tot, 4),
                    "mean_us": round(a["t"] / a["n"] * 1e6, 2),
                    "mean_dram_bytes": int((a["rd"] + a["wr"]) / a["n"])})
    return out


if __name__ == "__main__":
    only = None
    if "--only" in sys.argv:
        only = sys.argv[sys.argv.index("--only") + 1]
    for row in summarize(sys.argv[1], only):
        print(json.dumps(row))
