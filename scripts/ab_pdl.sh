#!/bin/bash
# programmatic dependent launch A/B (experiments build): graph step + phases at b=256
export PBD_LIB_VARIANT=exp
for cfg in "PBD_PDL=0" "PBD_PDL=1"; do
  echo "== $cfg"; for i in 1 2; do env $cfg python scripts/quick_step.py 2>&1 | grep -E 'graph step'; done
  env $cfg python scripts/phase_graphs.py 2>&1
done
