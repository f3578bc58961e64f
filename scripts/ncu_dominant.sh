#!/bin/bash
# full ncu capture of the bench's dominant kernel exactly as bench.py launches it
# (64->64 3x3 @32x32, b=256, bias+ReLU epilogue = PBDK_EPI_BIAS_RELU, the step's plan settings)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:conv_fprop -c 1 -s 3 \
    -o gpurun_out/dominant -f env STEP_SCOPE=1 python scripts/time_conv.py 256 32 64 64 3 1 2 > gpurun_out/ncu_dominant.log 2>&1
tail -2 gpurun_out/ncu_dominant.log
