#!/bin/bash
# ncu launch list (gpu__time_duration per kernel) of one bench step of a config.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
c=${1:-2}
SMALL="bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
timeout 600 python $SMALL > gpurun_out/b_small_$c.log 2>&1 || { echo "bench failed"; tail -3 gpurun_out/b_small_$c.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg$c.csv python $SMALL > gpurun_out/ncu_l_$c.log 2>&1
echo "ncu exit $?"
