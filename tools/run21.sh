#!/bin/bash
# frame_host upload ordering: tests + e2e.  Under gpurun.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -k "frame or e2e or bench or host" -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/e2e_probe2.py 2>&1 | head -4
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-transfer --no-strong --no-sequence > gpurun_out/b21.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b21.json')); e=d['e2e']
print('step', round(d['ms_per_step'],4), 'e2e', round(e['ms_per_step'],4), 'iso', round(e['isolated_ms_per_frame'],4))"
done
