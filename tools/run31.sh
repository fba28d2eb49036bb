#!/bin/bash
# gpu tests + the default bench line + cfg4 line.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
# (tests ran in the previous call)


t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $? wall $(( $(date +%s) - t0 )) s"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-strong --no-sequence > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 exit $?"
