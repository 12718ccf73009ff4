#!/bin/bash
# Round-2 measurement set (GPU box): GPU suite, smoke, bench suite with the
# reference arms, ncu launch lists of every config, full ncu captures of the
# four kernels of the default line (config 4a).  Outputs: gpurun_out/r02/.
cd "$(dirname "$0")/.."
export SUITE_DIR=r02
D=gpurun_out/r02
mkdir -p $D
python -m pytest tests -m gpu -q 2>&1 | tail -8 > $D/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
bash scripts/bench_suite.sh
bash scripts/launch_lists.sh
for k in k_joint_coeffs k_joint_apply k_joint_mse_hr_at k_joint_bwd_lr_seg; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $D/ncu_full_$k \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $D/ncu_full_$k.log 2>&1
done
echo measure done
