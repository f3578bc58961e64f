#!/bin/bash
# programmatic dependent launch A/B on the MBConv workloads (experiments build)
export PBD_LIB_VARIANT=exp
for cfg in "PBD_PDL=0" "PBD_PDL=1" "PBD_PDL=0" "PBD_PDL=1"; do
  for m in mbv2 effb0; do
    echo "== $cfg $m $(env $cfg MODEL=$m STEPS=20 python scripts/mb_step.py 256 224 0 2>&1 | grep -E '^step' | head -1)"
  done
done
