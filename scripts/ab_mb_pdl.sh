#!/bin/bash
# A/B: programmatic dependent launch for the MBConv kernels (product) vs plain (experiments build = previous
# HEAD); bitwise comparison of two steps, MB GPU tests, step times
mkdir -p gpurun_out
PBD_LIB_VARIANT=exp timeout 300 python scripts/ab_bitwise_mb.py a > gpurun_out/abmb.log 2>&1
timeout 300 python scripts/ab_bitwise_mb.py b >> gpurun_out/abmb.log 2>&1
python scripts/ab_bitwise_mb.py cmp >> gpurun_out/abmb.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mb.py tests/test_gpu_dw.py tests/test_gpu_nas.py tests/test_gpu_parity_full.py -x -q > gpurun_out/pytest_mb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mb.log
for v in exp prod exp prod; do
  if [ $v = exp ]; then export PBD_LIB_VARIANT=exp; else unset PBD_LIB_VARIANT; fi
  for w in mbv2 effb0; do
    ms=$(timeout 300 python bench.py --workload $w --steps 100 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "$v $w step : $ms" >> gpurun_out/ab_mb_pdl.txt
  done
done
tail -1 gpurun_out/abmb.log; tail -2 gpurun_out/pytest_mb.log; cat gpurun_out/ab_mb_pdl.txt
