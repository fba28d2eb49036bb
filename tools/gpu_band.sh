#!/bin/bash
# Shell-band A/B (DGSM_BAND_ROWS) + the accumulation parity tests.  Run under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/gpu_tests.log
bash tools/ab_env.sh 2 "DGSM_BAND_ROWS=64" "DGSM_BAND_ROWS=32"
bash tools/ab_env.sh 5 "DGSM_BAND_ROWS=128" "DGSM_BAND_ROWS=64" "DGSM_BAND_ROWS=32"
