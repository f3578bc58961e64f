#!/bin/bash
# A/B: PDL for the split-K wgrad reduction (product)
# vs plain launch (experiments build = previous HEAD)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
for v in exp prod exp prod; do
  if [ $v = exp ]; then export PBD_LIB_VARIANT=exp; else unset PBD_LIB_VARIANT; fi
  
  ms=$(timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "$v cifar step : $ms" >> gpurun_out/ab_splitred_pdl.txt
done
tail -3 gpurun_out/pytest_sel.log; cat gpurun_out/ab_splitred_pdl.txt
