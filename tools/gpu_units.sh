#!/bin/bash
# work-unit builder: parity tests + k_units_fused times at cfg2 and cfg4.  Under gpurun.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
for c in 2 4; do
  SMALL="bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-transfer --no-strong --no-sequence --no-graph"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_units|k_accumulate|k_combine" -c 6 --csv python $SMALL 2>/dev/null | grep -E "k_units|k_accumulate|k_combine" | awk -F'","' '{print "cfg'$c'", substr($5,1,40), $NF}'
done
