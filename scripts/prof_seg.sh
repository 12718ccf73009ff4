#!/bin/bash
# ncu --set full of one segment-kernel launch at config-1 shape (GPU box)
out=${1:-prof_seg}
r=${2:-8}
python scripts/time_highres_variants.py $r > gpurun_out/${out}_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_highres_seg -c 1 \
    -o gpurun_out/$out python scripts/time_highres_variants.py $r > gpurun_out/${out}_ncu.log 2>&1
cat gpurun_out/${out}_plain.log
