#!/bin/bash
# Every BASELINE config through bench.py on one GPU; JSON lines -> gpurun_out/<dir>/suite_<cfg>.json
cd "$(dirname "$0")/.."
D=gpurun_out/${SUITE_DIR:-suite}
mkdir -p $D
timeout 900 python bench.py > $D/suite_default_cfg4a.json 2> $D/suite_default_cfg4a.err
echo "default rc=$?"
for cfg in cfg4b cfg1 cfg0 cfg3 cfg2; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 > $D/suite_$cfg.json 2> $D/suite_$cfg.err
  echo "$cfg rc=$?"
done
for r in 1 2 4 8; do
  timeout 600 python bench.py --config cfg3 --radius $r --no-cpu --no-e2e --steps 10 --warmup 3 > $D/suite_cfg3_r$r.json 2> $D/suite_cfg3_r$r.err
done
for hr in 1024 2048 3072; do
  timeout 600 python bench.py --config cfg3 --hr $hr --batch 1 --no-cpu --no-e2e --steps 20 --warmup 3 > $D/suite_cfg3_b1_h$hr.json 2> $D/suite_cfg3_b1_h$hr.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $D/suite_reference_cfg4a.json 2> $D/suite_reference_cfg4a.err
timeout 900 python bench.py --impl reference --config cfg1 --steps 5 --warmup 3 > $D/suite_reference_cfg1.json 2> $D/suite_reference_cfg1.err
echo suite done
