#!/bin/bash
# ncu --set full capture of one k_accumulate launch per config (one ncu run each), 1 GPU.
# usage: bash tools/gpu_prof_acc.sh [configs...]   (default: 2)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in ${@:-2}; do
  SMALL="bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong"
  timeout 600 python $SMALL > gpurun_out/b_small_$c.log 2>&1 || { echo "bench cfg$c failed"; tail -3 gpurun_out/b_small_$c.log; continue; }
  ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -o gpurun_out/prof_acc_cfg$c \
      python $SMALL > gpurun_out/ncu_acc_$c.log 2>&1
  echo "ncu cfg$c exit $?"
done
