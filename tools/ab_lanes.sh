#!/bin/bash
# per-light lanes (concurrent depth-sort chains): tests + cfg3/cfg5/cfg2 steps against the previous commit.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
for c in 3 5 2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abl.json 2>/dev/null || { echo "[$c] failed"; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/abl.json')); acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('cfg$c step', round(d['ms_per_step'],4), 'non-acc', round(d['ms_per_step']-acc,4))"
done
