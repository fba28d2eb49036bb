#!/bin/bash
# onesweep keys per thread A/B on the cfg2 / cfg4 steps (graph-timed).  Under gpurun.
mkdir -p gpurun_out
for v in "" "-DDGSM_OS_ITEMS=4" "-DDGSM_OS_ITEMS=2"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; tail -3 gpurun_out/ab_build.log; continue; }
  for c in 2 4; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abo.json 2>/dev/null || { echo "[$v $c] failed"; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abo.json'))
print('[$v] cfg$c step', round(d['ms_per_step'],4), 'non-acc', round(d['ms_per_step']-d['accumulate_ms'],4))"
  done
done
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
