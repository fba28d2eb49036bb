#!/bin/bash
# band pre-pass guard A/B + ncu of the band kernel.  Under gpurun.
bash tools/ab_variants.sh "5" "X=1" base v11
bash tools/prof_variants.sh "base:5:X=1"
