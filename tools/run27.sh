#!/bin/bash
# per-light tile sort: binning parity + cfg5/cfg3 steps + launch list.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/gpu_tests.log
for c in 5 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/b27.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b27.json')); acc=d.get('accumulate_ms_rank0')
print('cfg$c step', round(d['ms_per_step'],4), 'acc', round(acc,4), 'non-acc', round(d['ms_per_step']-acc,4), 'launches', d['gpu_launches'])"
done
SMALL="bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg5_pl.csv python $SMALL > /dev/null 2>&1
echo "ncu exit $?"
