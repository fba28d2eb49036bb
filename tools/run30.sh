#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong > gpurun_out/b30.json 2> gpurun_out/b30.err || tail -5 gpurun_out/b30.err
python -c "
import json; d=json.load(open('gpurun_out/b30.json')); c=d['cfg4_sequence']
for m in ('full','roi_slab'):
    r=c[m]; print(m, 'per-frame mean', round(r['ms_per_frame_mean'],4), 'p50', round(r['ms_per_frame_p50'],4), 'stream', round(r['stream']['ms_per_frame'],4), 'overflow', r['overflow_frames'], r['stream']['overflow_frames'], 'vs paper', r['stream']['vs_paper_s_per_frame'])
print('step', d['ms_per_step'], d['launch_mode'])"
