#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_bench_contract.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for a in "" "--no-graph"; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-transfer --no-strong --no-sequence $a > gpurun_out/b29.json 2> gpurun_out/b29.err || tail -5 gpurun_out/b29.err
python -c "
import json; d=json.load(open('gpurun_out/b29.json'))
print('[$a]', d['launch_mode'], 'step', round(d['ms_per_step'],4), 'stream', round(d['ms_per_step_stream_launches'],4), 'acc', round(d['accumulate_ms'],4), 'frac', round(d['roofline']['frac'],4), 'value %.4g' % d['value'], 'launches', d['gpu_launches'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
