#!/bin/bash
# launch list (per-kernel durations) of one eager MBConv step at b=256, S=224
mkdir -p gpurun_out
PROFILE=1 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/mb_launches.csv python scripts/mb_step.py ${1:-256} ${2:-224} 0 > gpurun_out/mb_prof.log 2>&1
tail -2 gpurun_out/mb_prof.log
