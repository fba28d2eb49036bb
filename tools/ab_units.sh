#!/bin/bash
# work-unit builder path A/B (single CTA up to DGSM_FUSED_TILES, else the multi-kernel path).  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_largeshapes.py -m gpu -q -x -k "unit or cfg5 or cfg3" -p no:cacheprovider 2>&1 | tail -1
for v in "" "-DDGSM_FUSED_TILES=16384" "-DDGSM_FUSED_TILES=4096"; do
  DGSM_NVCC_EXTRA="$v" python paper_2601_01660_b200/build_ext.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; continue; }
  for c in 2 3 5; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/abu.json 2>/dev/null || { echo "[$v $c] failed"; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abu.json')); acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('[$v] cfg$c step', round(d['ms_per_step'],4), 'non-acc', round(d['ms_per_step']-acc,4))"
  done
done
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
