#!/bin/bash
# Round-end style verification of HEAD on one B200: gpu tests, smoke, all bench workloads, the
# reference arm, and the warm launch list of the default bench command.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for w in cifar_fp32 mbv2 effb0; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
cat gpurun_out/bench*.json
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1
bash scripts/ncu_dominant.sh
ncu -i gpurun_out/dominant.ncu-rep --page raw --csv > gpurun_out/dominant_raw.csv 2>&1
timeout 300 python scripts/conv_shape_shares.py > gpurun_out/conv_shapes.txt 2>&1
head -12 gpurun_out/launch_summary.txt
