#!/bin/bash
# Round-end measurement set (GPU box): bench suite, ncu launch lists of the
# default bench and every config, one full ncu capture of the default bench's
# kernel (k_highres_seg at config 1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/bench_suite.sh
bash scripts/launch_lists.sh
bash scripts/prof_seg.sh prof_seg_final 8
echo measure done
