#!/bin/bash
# ncu --set full of one full-res launch of the default bench (run on the GPU box)
set -e
out=${1:-prof_hr}
python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/${out}_plain.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_highres_fused -c 1 \
    -o gpurun_out/$out python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/${out}_ncu.log 2>&1
tail -1 gpurun_out/${out}_plain.json | cut -c1-250
