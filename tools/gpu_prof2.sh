#!/bin/bash
# Profile the non-accumulate kernels of one bench step (ncu --set full), 1 GPU.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
SMALL="bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 python $SMALL > gpurun_out/b_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_duplicate_ranked" -s 1 -c 1 -o gpurun_out/prof2 \
    python $SMALL > gpurun_out/ncu3.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu3.log
