#!/bin/bash
# A/B of build variants on the binning time: bash tools/ab_sort.sh "<nvcc extra A>" ...  (under gpurun)
mkdir -p gpurun_out
for v in "$@"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  echo "[$v] $(python tools/bins_bench.py 40)"
done
