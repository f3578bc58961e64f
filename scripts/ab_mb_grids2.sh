#!/bin/bash
# MBConv step: combinations of the pass-grid knobs (experiments build), MobileNetV2 + EfficientNet-B0
mkdir -p gpurun_out
export PBD_LIB_VARIANT=exp
run() {
  for w in mbv2 effb0; do
    ms=$(env "$@" timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "$w $* : $ms" >> gpurun_out/ab_mb_grids2.txt
  done
}
run X=0
run PBDK_MB_RED=148
run PBDK_MB_RED=96
run PBDK_MB_RED=148 PBDK_MB_APPLY=296
run PBDK_MB_RED=148 PBDK_MB_APPLY=296 PBDK_FIX_MIN_BYTES=1048576
run PBDK_MB_RED=148 PBDK_FIX_MIN_BYTES=1048576
run PBDK_MB_APPLY=148
run X=0
cat gpurun_out/ab_mb_grids2.txt
