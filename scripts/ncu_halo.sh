#!/bin/bash
# one full ncu capture (with source counters) of the 64->64 halo conv
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:conv_fprop_halo -c 1 -s 3 \
    -o gpurun_out/halo64 -f python scripts/time_conv.py 256 32 64 64 3 1 > gpurun_out/ncu_halo.log 2>&1
tail -3 gpurun_out/ncu_halo.log
