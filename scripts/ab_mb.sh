#!/bin/bash
# MBConv A/B (experiments build): graph step ms of mbv2 / effb0 at b=256, 224^2
export PBD_LIB_VARIANT=exp
for cfg in "PBDK_PW_BN_CAP=0" "PBDK_PW_BN_CAP=1" "PBD_MB_EPW=2"; do
  for m in mbv2 effb0; do
    echo "== $cfg $m $(env $cfg MODEL=$m STEPS=20 python scripts/mb_step.py 256 224 0 2>&1 | grep -E '^step' | head -1)"
  done
done
