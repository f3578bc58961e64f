#!/bin/bash
# A/B of an env toggle ($1=VAR) over the step's conv shapes (n h c k r stride epi)
VAR=${1:-PBDK_CHIP_MODEL}
for shape in "256 32 16 64 3 1 2" "256 32 64 64 3 1 2" "256 32 64 64 3 1 3" "256 32 64 128 3 2 2" "256 32 64 128 1 2 1" "256 16 128 128 3 1 2" "256 16 128 128 3 1 3" \
             "256 16 128 256 3 2 2" "256 16 128 256 1 2 1" "256 8 256 256 3 1 2" "256 8 256 256 3 1 3" "256 8 256 512 3 2 2" "256 8 256 512 1 2 1" \
             "256 4 512 512 3 1 2" "256 4 512 512 3 1 3" "256 32 32 64 3 1 0" "256 16 64 128 3 1 0" "256 8 128 256 3 1 0" "256 4 256 512 3 1 0" \
             "256 32 64 32 3 1 4" "256 16 128 64 3 1 4" "256 8 256 128 3 1 4" "256 4 512 256 3 1 4"; do
  echo "[$shape] off $(env $VAR=0 python scripts/time_conv.py $shape) | on $(env $VAR=1 python scripts/time_conv.py $shape)"
done
