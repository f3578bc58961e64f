#!/bin/bash
# A/B: PDL for the fp32 workload's tcgen05 convs (product) vs plain launches (experiments build = previous HEAD)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_tf32.py -x -q > gpurun_out/pytest_f3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f3.log
for v in exp prod exp prod; do
  if [ $v = exp ]; then export PBD_LIB_VARIANT=exp; else unset PBD_LIB_VARIANT; fi
  ms=$(timeout 300 python bench.py --workload cifar_fp32 --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "$v cifar_fp32 step : $ms" >> gpurun_out/ab_f3_pdl.txt
done
tail -2 gpurun_out/pytest_f3.log; cat gpurun_out/ab_f3_pdl.txt
