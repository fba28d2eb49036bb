#!/bin/bash
# ncu --set full of k_accumulate for accumulate.cu variants:  bash tools/prof_variants.sh "<name:cfg:ENV=V> ..."  (under gpurun)
mkdir -p gpurun_out
cp paper_2601_01660_b200/csrc/accumulate.cu /tmp/accumulate.cu.keep
for spec in $1; do
  IFS=: read name c envv <<< "$spec"
  cp variants/$name/accumulate.cu paper_2601_01660_b200/csrc/accumulate.cu
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  SMALL="bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
  env $envv timeout 600 python $SMALL > gpurun_out/b_small.log 2>&1 || { echo "bench $spec failed"; tail -3 gpurun_out/b_small.log; continue; }
  env $envv ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -o gpurun_out/prof_${name}_cfg$c \
      python $SMALL > gpurun_out/ncu_${name}_$c.log 2>&1
  echo "ncu $spec exit $?"
done
cp /tmp/accumulate.cu.keep paper_2601_01660_b200/csrc/accumulate.cu
