#!/bin/bash
# band kernel (K > 64) verification: whole -m gpu suite at the default band rows, cfg2 + cfg5 bench lines.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=10 > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -14 gpurun_out/gpu_tests.log
for c in 2 5 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/b$c.json 2> gpurun_out/b$c.err || { echo "bench $c failed"; tail -3 gpurun_out/b$c.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/b$c.json')); r=d['roofline']
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('cfg$c acc_ms', round(acc,4), 'step', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), 'work', round(r['work_frac'],4), 'clk', d['clocks']['sm_mhz'])"
done
