#!/bin/bash
# ncu --set full of the small binning kernels of one bench step (one ncu run), 1 GPU.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
SMALL="bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer"
timeout 300 python $SMALL > gpurun_out/b_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k "regex:k_duplicate_ranked|k_ranges|k_gather_counts|k_depth_keys|k_hist|k_units_lpt|k_query" -c 8 -o gpurun_out/prof3 \
    python $SMALL > gpurun_out/ncu4.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu4.log
