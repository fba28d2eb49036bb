#!/bin/bash
# ncu --set full of selected kernels of one bench step: bash tools/gpu_prof_kernels.sh <cfg> <regex> <count>  (1 GPU)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
c=${1:-2}; rx=${2:-k_project}; n=${3:-1}
SMALL="bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
timeout 600 python $SMALL > gpurun_out/b_small.log 2>&1 || { echo bench failed; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$rx" -c $n -o gpurun_out/prof_k_cfg$c python $SMALL > gpurun_out/ncu_k.log 2>&1
echo "ncu exit $?"
