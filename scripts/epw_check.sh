timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k fprop 2>&1 | tail -1
for e in 1 2; do echo "PBDK_EPW=$e"; for s in "256 32 16 64 3 1 2" "256 32 16 32 3 1 0" "256 32 32 64 3 1 0" "256 32 16 64 1 1 0" "256 16 64 128 1 2 0" "256 32 64 64 3 1 2"; do PBDK_EPW=$e python scripts/time_conv.py $s; done; done
for e in 1 0 1 0; do PBDK_EPW=$e python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('epw', $e, d['ms_per_step'])"; done
