#!/bin/bash
# Round-end refresh of every measurement under profiles/ (1 GPU, under gpurun):
# gpu tests, smoke, the default bench (cfg2 + strong_cfg5 + cfg4_sequence + transfer),
# cfg3/cfg4/cfg5 lines, reference arm, launch lists (cfg2, cfg5), ncu --set full of
# k_accumulate (cfg2, cfg5) and of the query (cfg2, cfg5).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?"
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-strong --no-sequence > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "bench cfg$c exit $?"
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
nproc > gpurun_out/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/nproc.txt
for c in 2 5; do
  SMALL="bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
  timeout 600 python $SMALL > gpurun_out/b_small_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg$c.csv python $SMALL > gpurun_out/ncu_l_$c.log 2>&1
  echo "ncu launches cfg$c exit $?"
  SMALL="bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -o gpurun_out/prof_acc_cfg$c \
      python $SMALL > gpurun_out/ncu_acc_$c.log 2>&1
  echo "ncu acc cfg$c exit $?"
done
timeout 300 python tools/query_prof.py > gpurun_out/qp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_query -c 2 -o gpurun_out/prof_q python tools/query_prof.py > gpurun_out/ncu_q.log 2>&1
echo "ncu query exit $?"
