#!/bin/bash
# epilogue (ex2-based T, select-free band epilogue) A/B + accumulation parity.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bands.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_largeshapes.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/gpu_tests.log
bash tools/ab_variants.sh "2 5" "X=1" base v10
