#!/bin/bash
# band height A/B at K = 64 (cfg2) and K = 128 (cfg5).  Under gpurun.
bash tools/ab_variants.sh "2" "DGSM_BAND_ROWS=32 DGSM_BAND_ROWS=48" base
bash tools/ab_variants.sh "5" "DGSM_BAND_ROWS=32 DGSM_BAND_ROWS=48 DGSM_BAND_ROWS=64" base
