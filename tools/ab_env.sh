#!/bin/bash
# A/B of runtime switches on one config: bash tools/ab_env.sh <config> "<ENV=V ...>" ...   (under gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
c=$1; shift
for v in "$@"; do
  for rep in 1 2; do
    env $v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/ab_env.log 2> gpurun_out/ab_env.err || { echo "[$v] failed"; tail -3 gpurun_out/ab_env.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/ab_env.log')); r=d['roofline']
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
w=d.get('accumulate_work', d.get('accumulate_work_rank0', {}))
br=w.get('band_records', 0) / max(1, w.get('warp_records', 2) // 2)
print('cfg$c [$v]', 'acc_ms', round(acc,4), 'step', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), 'work', round(r['work_frac'],4), 'band_rec/P', round(br, 4))"
  done
done
