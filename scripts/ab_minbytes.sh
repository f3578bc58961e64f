#!/bin/bash
# minimum input bytes per CTA of the staged BN / loss passes (experiments build): CIFAR graph step
export PBD_LIB_VARIANT=exp
for f in 0 131072 262144 524288 1048576; do
  for a in 0 262144; do
    r=$(PBDK_FIX_MIN_BYTES=$f PBDK_APPLY_MIN_BYTES=$a python scripts/quick_step.py 2>&1 | grep 'graph step')
    r2=$(PBDK_FIX_MIN_BYTES=$f PBDK_APPLY_MIN_BYTES=$a python scripts/quick_step.py 2>&1 | grep 'graph step')
    echo "fix $f apply $a : $r | $r2"
  done
done
