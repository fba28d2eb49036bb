#!/bin/bash
# 64-record stages in the band kernel against the 48-row bands.  Under gpurun.
mkdir -p gpurun_out
bash tools/ab_variants.sh "5" "X=1" base s64
cp paper_2601_01660_b200/csrc/accumulate.cu /tmp/acc.keep
cp variants/s64/accumulate.cu paper_2601_01660_b200/csrc/accumulate.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_bands.py tests/test_gpu_largeshapes.py tests/test_gpu_sweep.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
cp /tmp/acc.keep paper_2601_01660_b200/csrc/accumulate.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
