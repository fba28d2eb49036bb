#!/bin/bash
# ncu --set full of the non-accumulation kernels of a cfg2 step (k_project, k_pass, k_duplicate_ranked).  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
SMALL="bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
timeout 300 python $SMALL > gpurun_out/b_small.log 2>&1 || { echo bench failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_project|k_pass|k_duplicate_ranked|k_depth_keys|k_units_fused" -s 21 -c 12 -o gpurun_out/prof_other_cfg2 python $SMALL > gpurun_out/ncu_other.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_other.log
