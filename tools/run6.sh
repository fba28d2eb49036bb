#!/bin/bash
# band-kernel parity tests.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bands.py -m gpu -q --timeout 600 -p no:cacheprovider --durations=5 > gpurun_out/gpu_bands.log 2>&1
echo "pytest exit $?"; tail -30 gpurun_out/gpu_bands.log
