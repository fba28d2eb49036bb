#!/bin/bash
# stage size A/B (non-band kernel).  Under gpurun.
bash tools/ab_variants.sh "2 3" "X=1" base v8
