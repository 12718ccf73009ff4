#!/bin/bash
# ncu launch lists (duration + DRAM bytes per launch) of our kernels for the
# default bench (config 4a) and every config (GPU box); after plain runs exit 0.
cd "$(dirname "$0")/.."
D=gpurun_out/${SUITE_DIR:-suite}
mkdir -p $D
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() {  # name, bench args
  local n=$1; shift
  python bench.py "$@" --steps 2 --warmup 3 --no-e2e --no-cpu > $D/ll_plain_$n.json 2>&1 || return
  ncu --metrics $M --clock-control none -k regex:'^k_' -c 200 --csv \
      --log-file $D/ncu_launches_$n.csv python bench.py "$@" --steps 2 --warmup 3 \
      --no-e2e --no-cpu > $D/ll_ncu_$n.log 2>&1
}
run cfg4a
for c in cfg0 cfg1 cfg2 cfg3 cfg4b; do run $c --config $c; done
echo lists done
