#!/bin/bash
# A/B of the working csrc against alternate copies of some of its files (variants/<name>/csrc/*),
# interleaved: bash tools/ab_tree.sh "<cfg list>" <reps> name ...  (under gpurun)
mkdir -p gpurun_out /tmp/ab_tree_keep
cfgs=$1; reps=$2; shift 2
C=paper_2601_01660_b200/csrc
cp -p $C/* /tmp/ab_tree_keep/ 2>/dev/null
build() { python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed"; tail -5 gpurun_out/ab_build.log; return 1; }
          mkdir -p /tmp/ab_so/$1; cp paper_2601_01660_b200/*.so /tmp/ab_so/$1/; }
build cur
for name in "$@"; do cp variants/$name/csrc/* $C/; build $name; cp -p /tmp/ab_tree_keep/* $C/; done
for r in $(seq $reps); do
  for name in cur "$@"; do
    cp /tmp/ab_so/$name/*.so paper_2601_01660_b200/
    for c in $cfgs; do
      timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/ab.log 2> gpurun_out/ab.err || { echo "[$name cfg$c] failed"; tail -3 gpurun_out/ab.err; continue; }
      python -c "
import json; d=json.load(open('gpurun_out/ab.log'))
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('$name cfg$c', 'step', round(d['ms_per_step'],4), 'acc', round(acc,4), 'rest', round(d['ms_per_step']-acc,4))"
    done
  done
done
cp /tmp/ab_so/cur/*.so paper_2601_01660_b200/
