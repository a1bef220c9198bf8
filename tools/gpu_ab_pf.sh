#!/bin/bash
# EXPERIMENT RECORD: the MSK_PF prefetch code was removed after the measurement (profiles/r02_kcg_ab.txt)
# A/B: L2 prefetch of the next CSR pieces in k_cg (MSK_PF = 0 / 1 / 2 pieces ahead of the ring)
bash tools/ab_variants.sh base pf1 pf2
LEVEL=4 bash tools/ab_variants.sh base pf1 pf2
CFG=C2 bash tools/ab_variants.sh base pf1 pf2
