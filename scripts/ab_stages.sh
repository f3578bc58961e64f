#!/bin/bash
# A/B: fprop stage-ring depth for 16/32-channel inputs (A = lib-exp built before the change, B = lib)
mkdir -p gpurun_out
for v in exp prod exp prod; do
  if [ $v = exp ]; then export PBD_LIB_VARIANT=exp; else unset PBD_LIB_VARIANT; fi
  echo "== $v" >> gpurun_out/ab_stages.txt
  timeout 300 python scripts/conv_shape_shares.py 2>&1 | grep -E " (16|32)->" >> gpurun_out/ab_stages.txt
  timeout 300 python bench.py --steps 500 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step ms', d['ms_per_step'])" >> gpurun_out/ab_stages.txt
done
cat gpurun_out/ab_stages.txt
