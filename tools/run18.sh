#!/bin/bash
# query: receivers per thread x CTAs/SM A/B.  Under gpurun.
bash tools/gpu_query_ab.sh "-DDGSM_QMINB=8" "-DDGSM_QPT=2 -DDGSM_QMINB=6" "-DDGSM_QPT=2 -DDGSM_QMINB=5" "-DDGSM_QPT=2 -DDGSM_QMINB=4"
python paper_2601_01660_b200/build_ext.py --force > /dev/null 2>&1
