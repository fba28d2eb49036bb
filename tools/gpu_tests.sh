#!/bin/bash
# build + the whole -m gpu suite (durations) + a short cfg2 bench.  Run under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=15 "$@" > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -25 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench exit $?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.log"))
print("step_ms", round(d["ms_per_step"], 4), "acc_ms", round(d["accumulate_ms"], 4), "query_ms", round(d["query_ms"], 4),
      "frac", round(d["roofline"]["frac"], 4), "value", "%.4g" % d["value"], "clocks", d["clocks"]["sm_mhz"])
PY
