#!/bin/bash
# A/B: L2 prefetch of the next CSR pieces in k_cg (MSK_PF = 0 / 1 / 2 pieces ahead of the ring)
bash tools/ab_variants.sh base pf1 pf2
LEVEL=4 bash tools/ab_variants.sh base pf1 pf2
CFG=C2 bash tools/ab_variants.sh base pf1 pf2
