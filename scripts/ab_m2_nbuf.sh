#!/bin/bash
# A/B: m2 conv (two M tiles per filter load) with four rotating accumulator pairs for BN = 64 (product)
# vs two (experiments build = previous HEAD)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
for v in exp prod exp prod; do
  if [ $v = exp ]; then export PBD_LIB_VARIANT=exp; else unset PBD_LIB_VARIANT; fi
  echo "$v [256 16 128 64 3 1 2] $(STEP_SCOPE=1 timeout 120 python scripts/time_conv.py 256 16 128 64 3 1 2)" >> gpurun_out/ab_m2_nbuf.txt
  ms=$(timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "$v cifar step : $ms" >> gpurun_out/ab_m2_nbuf.txt
done
tail -3 gpurun_out/pytest_sel.log; cat gpurun_out/ab_m2_nbuf.txt
