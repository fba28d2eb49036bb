#!/bin/bash
# A/B of accumulate.cu variants (files under variants/<name>/accumulate.cu) on configs with
# env settings: bash tools/ab_variants.sh "<cfg list>" "<env list>" name1 name2 ...  (under gpurun)
mkdir -p gpurun_out
cfgs=$1; envs=$2; shift 2
cp paper_2601_01660_b200/csrc/accumulate.cu /tmp/accumulate.cu.keep
for name in "$@"; do
  cp variants/$name/accumulate.cu paper_2601_01660_b200/csrc/accumulate.cu
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$name.log 2>&1 || { echo "build $name failed"; tail -5 gpurun_out/build_$name.log; continue; }
  for c in $cfgs; do
    for v in $envs; do
      env $v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abv.log 2> gpurun_out/abv.err || { echo "[$name $c $v] failed"; tail -3 gpurun_out/abv.err; continue; }
      python -c "
import json; d=json.load(open('gpurun_out/abv.log')); r=d['roofline']
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
w=d.get('accumulate_work', d.get('accumulate_work_rank0', {}))
br=w.get('band_records', 0) / max(1, w.get('warp_records', 2) // 2)
print('$name cfg$c [$v]', 'acc_ms', round(acc,4), 'step', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), 'work', round(r['work_frac'],4), 'band_rec/P', round(br, 4))"
    done
  done
done
cp /tmp/accumulate.cu.keep paper_2601_01660_b200/csrc/accumulate.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
