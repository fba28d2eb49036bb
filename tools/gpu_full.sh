#!/bin/bash
# Round-end style measurement: build, gpu tests, smoke, full bench (cfg2 line with cpu_baseline,
# strong_cfg5, cfg4_sequence), cfg3/cfg4/cfg5 lines, reference arm, ncu launch list of a cfg2 step.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?"
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-strong --no-sequence > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "bench cfg$c exit $?"
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
nproc > gpurun_out/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/nproc.txt
SMALL="bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
timeout 300 python $SMALL > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python $SMALL > gpurun_out/ncu1.log 2>&1
echo "ncu exit $?"
