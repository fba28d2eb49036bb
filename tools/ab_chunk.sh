#!/bin/bash
# adaptive chunk (kMinChunk / kMinUnits) A/B on the cfg4 step and sequence.  Under gpurun.
mkdir -p gpurun_out
for v in ${AB_VARIANTS:-"" "-DDGSM_MIN_UNITS=4096 -DDGSM_MIN_CHUNK=64" "-DDGSM_MIN_UNITS=8192 -DDGSM_MIN_CHUNK=32"}; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong > gpurun_out/abc.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abc.json')); c=d['cfg4_sequence']
print('[$v] step', round(d['ms_per_step'],4), 'acc', round(d['accumulate_ms'],4), 'seq full', round(c['full']['stream']['ms_per_frame'],4), 'slab', round(c['roi_slab']['stream']['ms_per_frame'],4))"
done
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
