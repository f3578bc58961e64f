#!/bin/bash
# CIFAR step vs student conv SM cap / reduction grid after the rotating-accumulator changes (experiments build = HEAD)
mkdir -p gpurun_out
export PBD_LIB_VARIANT=exp
run() {
  ms=$(env "$@" timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "$* : $ms" >> gpurun_out/ab_caps_r2.txt
}
for rep in 1 2; do
  run X=0
  run PBDK_SCONV_CTAS=48
  run PBDK_SCONV_CTAS=80
  run PBDK_SCONV_CTAS=96
  run PBDK_RED_TARGET=296
done
cat gpurun_out/ab_caps_r2.txt
