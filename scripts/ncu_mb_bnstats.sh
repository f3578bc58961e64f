mkdir -p gpurun_out
PROFILE=1 timeout 600 ncu --nvtx --nvtx-include "step/" --set full --clock-control none -k regex:bn_stats_fix -s 10 -c 1 -o gpurun_out/bnstats -f python scripts/mb_step.py 256 224 0 > gpurun_out/bnstats.log 2>&1
ncu -i gpurun_out/bnstats.ncu-rep --page details --csv > gpurun_out/bnstats_details.csv 2>&1
tail -3 gpurun_out/bnstats.log
