#!/bin/bash
# A/B: fused update with tiled flip transposes (product build) vs the scattering version (experiments build)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_parity_full.py tests/test_gpu_driver.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
for v in exp prod exp prod; do
  if [ $v = exp ]; then export PBD_LIB_VARIANT=exp; else unset PBD_LIB_VARIANT; fi
  ms=$(timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "cifar $v : $ms" >> gpurun_out/ab_sgd_tiles.txt
done
unset PBD_LIB_VARIANT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sgd -c 20 --csv --log-file gpurun_out/sgd_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/pytest_sel.log; cat gpurun_out/ab_sgd_tiles.txt; grep -o '"[a-z_]*sgd[a-z_]*kernel[^"]*","[^"]*","[0-9.,]*"' gpurun_out/sgd_launches.csv | tail -5; tail -5 gpurun_out/sgd_launches.csv | cut -c1-300
