"""Per-source-line instruction / stall-sample shares from an ncu source CSV
(ncu -i X.ncu-rep --page source --csv --print-source cuda,sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
cur = None
out = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if r[2] != "-":
        continue
    ie = int(r[hdr.index("Instructions Executed")] or 0)
    samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    if ie or samp:
        out.append((cur, ln, ie, samp, r[1][:90]))
tot = sum(o[2] for o in out)
ts = sum(o[3] for o in out)
print("instructions", tot, "samples", ts)
for o in sorted(out, key=lambda o: -o[2])[:top]:
    print(f"{o[0][:14]:14s} {o[1]:4d} {o[2] / tot * 100:5.1f}% {o[3] / ts * 100:5.1f}%  {o[4]}")
