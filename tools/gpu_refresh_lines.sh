#!/bin/bash
# The bench lines and launch lists of profiles/ only (no ncu --set full).  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?"
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-strong --no-sequence > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "bench cfg$c exit $?"
done
for c in 2 5; do
  SMALL="bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
  timeout 600 python $SMALL > gpurun_out/b_small_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg$c.csv python $SMALL > gpurun_out/ncu_l_$c.log 2>&1
  echo "ncu launches cfg$c exit $?"
done
