#!/bin/bash
# programmatic dependent launch A/B (DGSM_PDL) + the whole -m gpu suite with PDL.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
for v in "-DDGSM_PDL=0" "" "-DDGSM_PDL=0" ""; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  for c in 2 4 3; do
    timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-transfer --no-strong --no-sequence > gpurun_out/abp.json 2>/dev/null || { echo "[$v $c] failed"; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abp.json')); acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
e=d.get('e2e') or {}
print('[$v] cfg$c step', round(d['ms_per_step'],4), 'stream', round(d.get('ms_per_step_stream_launches', 0),4), 'e2e', round(e.get('ms_per_step', 0),4))"
  done
done
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
