#!/bin/bash
# onesweep keys-per-thread A/B on cfg5 and cfg2 steps.  Under gpurun.
mkdir -p gpurun_out
for v in "" "-DDGSM_OS_ITEMS=12" "-DDGSM_OS_ITEMS=16"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; tail -3 gpurun_out/ab_build.log; continue; }
  for c in 5 2; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abs.log 2> gpurun_out/abs.err || { echo "[$v $c] failed"; tail -3 gpurun_out/abs.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abs.log'))
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('[$v] cfg$c step', round(d['ms_per_step'],4), 'acc', round(acc,4), 'non-acc', round(d['ms_per_step']-acc,4))"
  done
done
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
