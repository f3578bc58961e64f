python -m pytest tests/test_gpu_kernels.py -q -x -k wgrad 2>&1 | tail -3
for mt in 1 0; do echo "PBDK_WGRAD_MT=$mt"; for s in "256 32 16 32 3 1" "256 32 32 64 3 1" "256 32 16 64 3 1" "256 16 32 64 3 2"; do PBDK_WGRAD_MT=$mt python scripts/time_wgrad.py $s; done; done
