#!/bin/bash
# MB kernel changes: bitwise A/B vs the pre-change build (lib-exp), GPU MB tests, MB benches, MB launch list
mkdir -p gpurun_out
env PBD_LIB_VARIANT=exp $AB_ENV timeout 300 python scripts/ab_bitwise_mb.py a > gpurun_out/abmb.log 2>&1
timeout 300 python scripts/ab_bitwise_mb.py b >> gpurun_out/abmb.log 2>&1
python scripts/ab_bitwise_mb.py cmp >> gpurun_out/abmb.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mb.py tests/test_gpu_dw.py tests/test_gpu_nas.py tests/test_gpu_parity_full.py -x -q > gpurun_out/pytest_mb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mb.log
for w in mbv2 effb0; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
bash scripts/mb_profile.sh 256 224
python scripts/launch_summary.py gpurun_out/mb_launches.csv > gpurun_out/mb_launch_summary.txt 2>&1
tail -5 gpurun_out/abmb.log; tail -3 gpurun_out/pytest_mb.log
for w in mbv2 effb0; do python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['ms_per_step'],d['value'],d['gpu_launches'])"; done
head -25 gpurun_out/mb_launch_summary.txt
