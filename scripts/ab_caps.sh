#!/bin/bash
# A/B of the student-conv SM cap and the BN-pass grids with the round-2 kernels (experiments build)
export PBD_LIB_VARIANT=exp
for cfg in "PBDK_SCONV_CTAS=64" "PBDK_SCONV_CTAS=48" "PBDK_SCONV_CTAS=80" "PBDK_SCONV_CTAS=96" "PBDK_SCONV_CTAS=148" "PBDK_RED_TARGET=296" "PBDK_APPLY_PIPE_DIV=1"; do
  echo "== $cfg"; for i in 1 2; do env $cfg python scripts/quick_step.py 2>&1 | grep -E 'graph step'; done
done
