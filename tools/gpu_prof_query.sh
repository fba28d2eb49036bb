#!/bin/bash
# ncu --set full of the query kernel on Morton-ordered receivers (cfg2, cfg5), 1 GPU.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/query_prof.py "$@" > gpurun_out/qp.log 2>&1 || { echo qp failed; tail gpurun_out/qp.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_query -c 2 -o gpurun_out/prof_q \
    python tools/query_prof.py "$@" > gpurun_out/ncu_q.log 2>&1
echo "ncu exit $?"
