#!/bin/bash
# ncu --set full capture of one k_accumulate launch of a bench step (one ncu run), 1 GPU.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
SMALL="bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer"
timeout 300 python $SMALL > gpurun_out/b_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -o gpurun_out/prof \
    python $SMALL > gpurun_out/ncu2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu2.log
