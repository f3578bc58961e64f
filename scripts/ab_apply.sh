#!/bin/bash
# A/B of the staged apply passes (experiments build): graph step times, 3 runs each
export PBD_LIB_VARIANT=exp
for cfg in "PBDK_APPLY_PIPE=0" "PBDK_APPLY_PIPE_DIV=1" "PBDK_APPLY_PIPE_DIV=2" "PBDK_APPLY_PIPE_DIV=4"; do
  echo "== $cfg"; for i in 1 2 3; do env $cfg python scripts/quick_step.py 2>&1 | grep -E 'graph step'; done
done
