#!/bin/bash
# A/B of query build variants: bash tools/gpu_query_ab.sh "<nvcc extra A>" ...  (under gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -k "query" -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "query tests exit $?"; tail -3 gpurun_out/q_tests.log
for v in "$@"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  echo "== [$v]"; timeout 300 python tools/query_bench2.py 2 5
done
