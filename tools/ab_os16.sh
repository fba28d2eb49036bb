#!/bin/bash
# 16 keys/thread at 2 CTAs/SM (the default) vs 8 at 4 on whole steps, then the gpu suite.  Under gpurun.
mkdir -p gpurun_out
for r in 1 2; do for v in "-DDGSM_OS_ITEMS=8 -DDGSM_OS_MINB=4" ""; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  for c in 2 3 5; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abo.json 2>/dev/null || { echo "[$v $c] failed"; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abo.json'))
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('[$v] cfg$c step', round(d['ms_per_step'],4), 'non-acc', round(d['ms_per_step']-acc,4))"
  done
done; done
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -2
