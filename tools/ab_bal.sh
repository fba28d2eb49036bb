#!/bin/bash
# balanced record transform (half a stage per warp) vs base, cfg2 + cfg3.  Under gpurun.
bash tools/ab_variants.sh "2 3" "DGSM_ACC_STAGING=reg" base bal bal12 base bal12
