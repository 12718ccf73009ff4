#!/bin/bash
# Round-end measurement set (GPU box): bench suite + ncu launch list of the
# default bench + one full ncu capture of the default bench's top kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/bench_suite.sh
python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/ncu_launches_default.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/ncu_launch.log 2>&1
bash scripts/prof_hr.sh prof_hr_final
echo measure done
