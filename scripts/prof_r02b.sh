#!/bin/bash
# MBConv step launch list (eager, with DRAM bytes) + full ncu of the dominant CIFAR conv with the step's plan settings
mkdir -p gpurun_out
bash scripts/mb_profile.sh 256 224
python scripts/launch_summary.py gpurun_out/mb_launches.csv > gpurun_out/mb_launch_summary.txt 2>&1
bash scripts/ncu_dominant.sh
ncu -i gpurun_out/dominant.ncu-rep --page details --csv > gpurun_out/dominant_details.csv 2>&1
ncu -i gpurun_out/dominant.ncu-rep --page raw --csv > gpurun_out/dominant_raw.csv 2>&1
head -30 gpurun_out/mb_launch_summary.txt
