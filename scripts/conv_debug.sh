#!/bin/bash
# timing breakdown of the fprop kernel variants: normal / no epilogue stores / no MMAs
for shape in "256 32 64 64 3 1" "256 8 256 256 3 1"; do
  for halo in 0 1; do
    for dbg in 0 1 2 3; do
      r=$(PBDK_NO_HALO=$((1-halo)) PBDK_CONV_DEBUG=$dbg python scripts/time_conv.py $shape)
      echo "shape=[$shape] halo=$halo debug=$dbg $r"
    done
  done
done
