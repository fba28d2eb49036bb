#!/bin/bash
# A/B of accumulate build variants: bash tools/ab_acc.sh "<nvcc extra A>" "<nvcc extra B>" ...  (under gpurun)
mkdir -p gpurun_out
for v in "$@"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer > gpurun_out/ab.log 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.log')); print('[$v]', 'acc_ms', round(d['accumulate_ms'],4), 'step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
  done
done
