#!/bin/bash
# cfg2 record staging A/B at the current kernel (register vs TMA bulk copies), ncu of the TMA
# launch, and the cfg1 bench line.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for r in 1 2; do for v in reg tma; do
  DGSM_ACC_STAGING=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence > gpurun_out/st_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/st_$v.json')); print('$v', 'step', round(d['ms_per_step'],4), 'acc', round(d['accumulate_ms'],4))"
done; done
SMALL="bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence"
DGSM_ACC_STAGING=tma timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -o gpurun_out/prof_acc_cfg2_tma python $SMALL > gpurun_out/ncu_tma.log 2>&1
echo "ncu tma exit $?"
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "cfg1 exit $?"
