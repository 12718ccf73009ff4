#!/bin/bash
# quick A/B for the joint kernels: bench cfg4b + cfg3 lines and the cfg4b launch list (GPU box)
cd "$(dirname "$0")/.."
for c in cfg4b cfg3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_$c.json 2>&1; done
python bench.py --config cfg4b --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"^k_" -c 200 --csv --log-file gpurun_out/ncu_launches_cfg4b.csv \
    python bench.py --config cfg4b --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
