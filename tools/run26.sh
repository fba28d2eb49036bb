#!/bin/bash
# persistent software-pipelined query A/B.  Under gpurun.
bash tools/gpu_query_ab.sh "" "-DDGSM_QPERSIST=1" "-DDGSM_QPERSIST=1 -DDGSM_QMINB=6" "-DDGSM_QPERSIST=2"
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
