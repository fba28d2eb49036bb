#!/bin/bash
# query occupancy A/B (launch-bounds min blocks).  Under gpurun.
bash tools/gpu_query_ab.sh "" "-DDGSM_QMINB=5" "-DDGSM_QMINB=6" "-DDGSM_QMINB=8"
