#!/bin/bash
# band live-path constants from shared memory A/B.  Under gpurun.
bash tools/ab_variants.sh "5" "X=1" base v12
