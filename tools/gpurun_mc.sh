timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm" 2>&1 | tail -1
