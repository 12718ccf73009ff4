"""Rewrite profiles/traffic.json (the `roofline.traffic` of bench.py) from the
ncu launch lists of one profiles/<round> directory: per config, the mean
DRAM bytes per launch of the kernel with the largest time share."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01i"
out = {"_note": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of "
                "each config's dominant kernel, from the ncu launch lists in "
                f"{d}/ncu_launches_<cfg>.csv (written by scripts/update_traffic.py)."}
for cfg, name in (("cfg1", "default"), ("cfg0", "cfg0"), ("cfg2", "cfg2"), ("cfg3", "cfg3"),
                  ("cfg4a", "cfg4a"), ("cfg4b", "cfg4b")):
    csv = os.path.join(ROOT, d, f"ncu_launches_{name}.csv")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "summarize_launches.py"),
                          csv], capture_output=True, text=True, check=True)
    top = json.loads(res.stdout.splitlines()[0])
    out[cfg] = int(round(top["mean_dram_bytes"]))
    out[cfg + "_kernel"] = top["kernel"]
with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
