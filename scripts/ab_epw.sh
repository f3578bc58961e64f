#!/bin/bash
# A/B (experiments build = HEAD): epilogue warps per TMEM lane quarter with the rotating accumulators
mkdir -p gpurun_out
export PBD_LIB_VARIANT=exp
for v in 0 1 0 1; do
  ms=$(PBDK_EPW=$v timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "cifar PBDK_EPW=$v (0 = plan default: 2 on every ResNet conv) : $ms" >> gpurun_out/ab_epw.txt
done
cat gpurun_out/ab_epw.txt
