#!/bin/bash
# A/B of the fused BN-statistics policy (experiments build): graph step times
export PBD_LIB_VARIANT=exp
for cfg in "PBD_FUSE_MIN_K=576" "PBD_FUSE_MIN_K=0" "PBDK_NO_FUSED_STATS=1" "PBD_FUSE_MIN_K=1152"; do
  echo "== $cfg"; env $cfg python scripts/quick_step.py 2>&1 | grep -E 'graph step|block'
done
