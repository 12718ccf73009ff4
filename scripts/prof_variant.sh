#!/bin/bash
# ncu --set full of one full-res forward launch of a kernel family at config-1 shape (GPU box)
# usage: prof_variant.sh OUT KERNEL_REGEX [r]
out=${1:-prof_v}
k=${2:-k_highres}
r=${3:-8}
python scripts/time_highres_variants.py $r > gpurun_out/${out}_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/$out python scripts/time_highres_variants.py $r > gpurun_out/${out}_ncu.log 2>&1
cat gpurun_out/${out}_plain.log
