#!/bin/bash
# k_query_chunks launch-bound A/B on the cfg5 strong step (query_ms).  Under gpurun.
mkdir -p gpurun_out
for v in "-DDGSM_QMINB=1" "-DDGSM_QMINB=6" "-DDGSM_QMINB=8"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  for c in 5 3; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abq.log 2> gpurun_out/abq.err || { echo "[$v $c] failed"; tail -3 gpurun_out/abq.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abq.log'))
print('[$v] cfg$c query_ms', round(d['query_ms'],4), 'qfrac', round(d['query_roofline']['frac'],4))"
  done
done
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
