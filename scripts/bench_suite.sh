#!/bin/bash
# Run every BASELINE config through bench.py on one GPU; JSON lines -> gpurun_out/suite_<cfg>.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in cfg1 cfg0 cfg3 cfg4a cfg4b cfg2; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 > gpurun_out/suite_$cfg.json 2> gpurun_out/suite_$cfg.err
  echo "$cfg rc=$?"
done
for r in 1 2 4 8; do
  timeout 600 python bench.py --config cfg3 --radius $r --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/suite_cfg3_r$r.json 2> gpurun_out/suite_cfg3_r$r.err
done
for hr in 1024 2048 3072; do
  timeout 600 python bench.py --config cfg3 --hr $hr --batch 1 --no-cpu --no-e2e --steps 20 --warmup 3 > gpurun_out/suite_cfg3_b1_h$hr.json 2> gpurun_out/suite_cfg3_b1_h$hr.err
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/suite_reference_cfg1.json 2> gpurun_out/suite_reference_cfg1.err
echo suite done
