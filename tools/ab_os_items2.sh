#!/bin/bash
# onesweep partition size (keys per thread) x CTAs/SM bound, on whole steps (graph-timed).  Under gpurun.
mkdir -p gpurun_out
V=("" "-DDGSM_OS_ITEMS=12" "-DDGSM_OS_ITEMS=12 -DDGSM_OS_MINB=3" "-DDGSM_OS_ITEMS=16 -DDGSM_OS_MINB=2" "")
for v in "${V[@]}"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; tail -3 gpurun_out/ab_build.log; continue; }
  for c in ${AB_CFGS:-2 4 5}; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abo.json 2>/dev/null || { echo "[$v $c] failed"; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abo.json'))
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('[$v] cfg$c step', round(d['ms_per_step'],4), 'non-acc', round(d['ms_per_step']-acc,4))"
  done
done
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
