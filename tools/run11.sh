#!/bin/bash
# band height A/B at K = 128 (cfg5).  Under gpurun.
bash tools/ab_variants.sh "5" "DGSM_BAND_ROWS=43 DGSM_BAND_ROWS=48 DGSM_BAND_ROWS=56 DGSM_BAND_ROWS=40" base
