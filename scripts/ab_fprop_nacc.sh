#!/bin/bash
# A/B: 4 rotating TMEM accumulators for N <= 64 tiles in the halo and generic fprop kernels (product) vs 2
# (experiments build = the commit before both)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_parity_full.py tests/test_gpu_mb.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
for v in exp prod exp prod; do
  if [ $v = exp ]; then export PBD_LIB_VARIANT=exp; else unset PBD_LIB_VARIANT; fi
  for shape in "256 16 128 128 3 1 2" "256 8 256 128 3 1 2" "256 4 512 512 3 1 2" "256 16 64 128 3 1 2" "256 32 64 128 1 2 2"; do
    echo "$v [$shape] $(STEP_SCOPE=1 timeout 120 python scripts/time_conv.py $shape)" >> gpurun_out/ab_fprop_nacc128.txt
  done
  ms=$(timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "$v cifar step : $ms" >> gpurun_out/ab_fprop_nacc128.txt
  ms=$(timeout 300 python bench.py --workload mbv2 --steps 100 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "$v mbv2 step : $ms" >> gpurun_out/ab_fprop_nacc128.txt
done
tail -3 gpurun_out/pytest_sel.log; cat gpurun_out/ab_fprop_nacc128.txt
