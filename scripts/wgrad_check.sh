python -m pytest tests/test_gpu_kernels.py -q -x -k wgrad 2>&1 | tail -2
for mt in 2 1; do echo "PBDK_WGRAD_MT=$mt"; for s in "256 32 64 64 3 2" "256 16 64 128 3 1" "256 16 128 128 3 2" "256 8 128 256 3 1" "256 8 256 256 3 2" "256 4 256 512 3 1"; do PBDK_WGRAD_MT=$mt python scripts/time_wgrad.py $s; done; done
