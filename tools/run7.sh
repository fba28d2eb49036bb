#!/bin/bash
# half-tile cull A/B.  Under gpurun.
bash tools/ab_variants.sh "2 5" "X=1" base v7 v7b
