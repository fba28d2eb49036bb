#!/bin/bash
# build, query/chunk tests, default bench (cfg2 + strong_cfg5), cfg3 and cfg5 lines.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k "query or bench" -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/q_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench cfg2 exit $?"; tail -3 gpurun_out/bench_cfg2.err
for c in 3 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "bench cfg$c exit $?"; tail -3 gpurun_out/bench_cfg$c.err
done
