#!/bin/bash
# MBConv step: student conv SM cap (PBDK_MB_SCONV), elementwise MB kernel grid cap (PBDK_MB_CTAS), pass grids
mkdir -p gpurun_out
export PBD_LIB_VARIANT=exp
run() {
  for w in mbv2 effb0; do
    ms=$(env "$@" timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "$w $* : $ms" >> gpurun_out/ab_mb_grids3.txt
  done
}
run X=0
run PBDK_MB_SCONV=64
run PBDK_MB_SCONV=96
run PBDK_MB_SCONV=120
run PBDK_MB_CTAS=592
run PBDK_MB_CTAS=1184
run PBDK_MB_RED=96 PBDK_MB_APPLY=148
run X=0
cat gpurun_out/ab_mb_grids3.txt
