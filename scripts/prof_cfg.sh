#!/bin/bash
# ncu --set full of one launch of a kernel in a bench config (run on the GPU box)
# usage: prof_cfg.sh <config> <kernel-regex> <out-name> [launch-skip]
set -e
cfg=$1; kre=$2; out=$3; skip=${4:-0}
python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e > gpurun_out/${out}_plain.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:$kre -s $skip -c 1 \
    -o gpurun_out/$out python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e \
    > gpurun_out/${out}_ncu.log 2>&1
tail -1 gpurun_out/${out}_plain.json | cut -c1-200
