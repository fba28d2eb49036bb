#!/bin/bash
# One GPU iteration (run under gpurun from the repo root):
#   build -> gpu tests -> bench (no cpu baseline) -> ncu launch list -> ncu full capture of a kernel.
# Usage: tools/gpu_iter.sh [kernel-regex] [extra bench args...]
KREGEX=${1:-k_accumulate}
shift || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
SMALL="bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e $*"
timeout 300 python $SMALL > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python $SMALL > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 2 -c 1 -o gpurun_out/prof \
    python $SMALL > gpurun_out/ncu2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu2.log
