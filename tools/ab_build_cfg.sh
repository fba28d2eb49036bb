#!/bin/bash
# A/B of compile-time variants on a config's step: bash tools/ab_build_cfg.sh <cfg> "<nvcc extra A>" ... (under gpurun)
mkdir -p gpurun_out
c=$1; shift
for v in "$@"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; tail -5 gpurun_out/ab_build.log; continue; }
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/ab.log 2> gpurun_out/ab.err || { echo "[$v] bench failed"; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.log'))
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('cfg$c [$v]', 'step', round(d['ms_per_step'],4), 'acc', round(acc,4), 'rest', round(d['ms_per_step']-acc,4))"
done
