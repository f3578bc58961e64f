mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_mb.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
timeout 300 python bench.py --workload mbv2 --no-cpu-baseline > gpurun_out/bench_mbv2.json 2> gpurun_out/bench_mbv2.err
timeout 300 python scripts/conv_shape_shares.py > gpurun_out/conv_shapes.txt 2>&1
tail -3 gpurun_out/pytest_sel.log; cat gpurun_out/conv_shapes.txt; python -c "import json;d=json.load(open('gpurun_out/bench_mbv2.json'));print(d['ms_per_step'],d['value'],d['gpu_launches'])"
