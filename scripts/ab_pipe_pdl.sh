#!/bin/bash
# A/B: programmatic dependent launch of the staged HBM passes (experiments build, PBDK_PIPE_PDL), then the
# GPU suite on the product build
mkdir -p gpurun_out
export PBD_LIB_VARIANT=exp
for v in 1 0 1 0; do
  for w in cifar mbv2; do
    ms=$(PBDK_PIPE_PDL=$v timeout 300 python bench.py --workload $w --steps $([ $w = cifar ] && echo 1000 || echo 100) --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "$w PBDK_PIPE_PDL=$v : $ms" >> gpurun_out/ab_pipe_pdl.txt
  done
done
unset PBD_LIB_VARIANT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/ab_pipe_pdl.txt; tail -3 gpurun_out/pytest_gpu.log
