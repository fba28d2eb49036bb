#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for v in "" "DGSM_FRAME_EV_SORT=1" "" "DGSM_FRAME_EV_SORT=1"; do
env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-transfer --no-strong --no-sequence > gpurun_out/b22.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b22.json')); e=d['e2e']
print('[$v] step', round(d['ms_per_step'],4), 'e2e', round(e['ms_per_step'],4), 'iso', round(e['isolated_ms_per_frame'],4))"
done
