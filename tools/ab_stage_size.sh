#!/bin/bash
# stage size 24 / 16 (12 CTAs/SM register staging; 11 CTAs/SM TMA staging) at K = 64.  Under gpurun.
bash tools/ab_variants.sh "2 3" "DGSM_ACC_STAGING=reg DGSM_ACC_STAGING=tma" base v9 v13
