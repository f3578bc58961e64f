#!/bin/bash
# full ncu captures of representative teacher convs: 128->128 3x3 @16x16 and 256->256 @8x8 (b=256)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:conv_fprop -c 1 -s 3 \
    -o gpurun_out/conv128 -f python scripts/time_conv.py 256 16 128 128 3 1 > gpurun_out/ncu_conv128.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:conv_fprop -c 1 -s 3 \
    -o gpurun_out/conv256 -f python scripts/time_conv.py 256 8 256 256 3 1 > gpurun_out/ncu_conv256.log 2>&1
for s in "256 32 64 64 3 1" "256 16 128 128 3 1" "256 8 256 256 3 1" "256 4 512 512 3 1" "256 16 64 128 3 2"; do
  echo "[$s] $(python scripts/time_conv.py $s)"
done
