"""Aggregate ncu per-line instruction counts into line ranges:
python scripts/ncu_phases.py src.csv file.cu name:lo-hi ... --px N"""
import collections
import csv
import sys

src, fname = sys.argv[1], sys.argv[2]
rngs = []
px = 1.0
args = sys.argv[3:]
i = 0
while i < len(args):
    if args[i] == "--px":
        px = float(args[i + 1])
        i += 2
        continue
    n, lh = args[i].split(":")
    lo, hi = map(int, lh.split("-"))
    rngs.append((n, lo, hi))
    i += 1
rows = list(csv.reader(open(src)))
cur = None
hdr = None
agg = collections.Counter()
tot = 0
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 3 or r[2] != "-":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    ie = int(r[hdr.index("Instructions Executed")] or 0)
    tot += ie
    key = "other:" + cur
    if cur == fname:
        for n, lo, hi in rngs:
            if lo <= ln <= hi:
                key = n
                break
        else:
            key = "rest"
    agg[key] += ie
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:24s} {v / tot * 100:5.1f}%  thread-inst/unit {v * 32 / px:7.1f}")
