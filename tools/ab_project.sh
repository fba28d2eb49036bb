#!/bin/bash
# A/B of project.cu variants (variants/<name>/project.cu): steps and the k_project launch time.  Under gpurun.
mkdir -p gpurun_out
cp paper_2601_01660_b200/csrc/project.cu /tmp/project.cu.keep
for name in "$@"; do
  cp variants/$name/project.cu paper_2601_01660_b200/csrc/project.cu
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "binning" -p no:cacheprovider > gpurun_out/pt_$name.log 2>&1; echo "[$name] binning tests exit $?"
  for c in 2 3 5; do
    SMALL="bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
    timeout 600 python $SMALL > gpurun_out/abp.json 2>/dev/null || { echo "[$name $c] failed"; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/abp.json'))
acc=d.get('accumulate_ms', d.get('accumulate_ms_rank0'))
print('[$name] cfg$c step', round(d['ms_per_step'],4), 'non-acc', round(d['ms_per_step']-acc,4))"
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_project -c 3 --csv python ${SMALL/--steps 5/--steps 1} 2>/dev/null | grep k_project | tail -1 | awk -F'","' '{print "  k_project us", $NF}'
  done
done
cp /tmp/project.cu.keep paper_2601_01660_b200/csrc/project.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
