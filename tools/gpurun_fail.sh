timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lanes.py -q -x -p no:cacheprovider 2>&1 | grep -E "Error|assert|FAILED|^E " | head -20
