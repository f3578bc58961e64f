#!/bin/bash
# cluster-multicast conv A/B (experiments build): per-shape times for each cluster shape, then kernel tests
export PBD_LIB_VARIANT=exp
shapes=("256 16 128 128 3 1" "256 8 256 256 3 1" "256 4 512 512 3 1" "256 32 64 128 3 2" "256 16 128 256 3 2" "256 8 256 512 3 2")
for sh in "${shapes[@]}"; do
  line="$sh:"
  for mc in "" "2x1" "4x1" "2x2" "1x2" "1x4"; do
    t=$(PBDK_M2=0 PBDK_MC=$mc timeout 60 python scripts/time_conv.py $sh 2>&1 | tail -1 | awk '{print $1}')
    line="$line  [$mc]$t"
  done
  t=$(timeout 60 python scripts/time_conv.py $sh 2>&1 | tail -1 | awk '{print $1}')
  echo "$line  [default]$t"
done
for mc in 2x1 4x1 2x2 1x2; do
  echo "== tests PBDK_MC=$mc"; PBDK_M2=0 PBDK_MC=$mc timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
done
