#!/bin/bash
# accumulation parity after the 24-record stage.  Under gpurun.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/b25.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b25.json')); print('cfg2 step', round(d['ms_per_step'],4), 'acc', round(d['accumulate_ms'],4), 'frac', round(d['roofline']['frac'],4))"
