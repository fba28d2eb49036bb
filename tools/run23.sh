#!/bin/bash
# ncu --set full of k_accumulate at cfg2 with TMA staging forced (the staging A/B evidence).  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
SMALL="bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
for st in tma reg; do
  DGSM_ACC_STAGING=$st timeout 300 python $SMALL > gpurun_out/b_$st.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_$st.json')); print('$st acc_ms', round(d['accumulate_ms'],4), 'step', round(d['ms_per_step'],4))"
done
DGSM_ACC_STAGING=tma timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -o gpurun_out/prof_acc_cfg2_tma python $SMALL > gpurun_out/ncu_tma.log 2>&1
echo "ncu exit $?"
