#!/bin/bash
# FrameStream test + the bench's e2e record (cfg2).  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_framestream.py tests/test_gpu_async.py tests/test_bench_contract.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-transfer --no-strong --no-sequence > gpurun_out/be2e.json 2> gpurun_out/be2e.err || tail -5 gpurun_out/be2e.err
python -c "
import json; d=json.load(open('gpurun_out/be2e.json')); e=d['e2e']
print('step', round(d['ms_per_step'],4), 'e2e', round(e['ms_per_step'],4), 'value %.4g' % e['value'], 'frame_host', round(e['frame_host_ms_per_step'],4), 'iso', round(e['isolated_ms_per_frame'],4))"
