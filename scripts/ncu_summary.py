"""Headline metrics + stall breakdown of every kernel in an ncu report."""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
want = ["Kernel Name", "Block Size", "Grid Size", "gpu__time_duration.sum", "inst_executed",
        "sm__inst_executed.avg.per_cycle_active", "sass__inst_executed_shared_loads",
        "sass__inst_executed_shared_stores", "sass__inst_executed_global_loads",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sass__inst_executed_register_spilling"]
for r in rows[2:]:
    for k in want:
        if k in h:
            print(f"{k:55s} {r[h.index(k)]}")
    st = {}
    for k, v in zip(h, r):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
            except ValueError:
                pass
    t = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k} {100 * v / t:.1f}" for k, v in
                                sorted(st.items(), key=lambda x: -x[1])[:9]))
