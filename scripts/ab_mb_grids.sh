#!/bin/bash
# MBConv step vs BN/loss pass grids (experiments build): PBDK_MB_RED (reduction CTAs), PBDK_MB_APPLY
# (apply CTAs), PBDK_FIX_MIN_BYTES; MobileNetV2 b=256 224^2 graph step
mkdir -p gpurun_out
export PBD_LIB_VARIANT=exp
run() {
  ms=$(env "$@" timeout 300 python bench.py --workload mbv2 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "$* : $ms" >> gpurun_out/ab_mb_grids.txt
}
run X=0
run PBDK_MB_RED=148
run PBDK_MB_RED=444
run PBDK_MB_RED=592
run PBDK_MB_APPLY=296
run PBDK_MB_APPLY=592
run PBDK_MB_APPLY=2368
run PBDK_FIX_MIN_BYTES=0
run PBDK_FIX_MIN_BYTES=1048576
run X=0
cat gpurun_out/ab_mb_grids.txt
