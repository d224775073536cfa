timeout 900 python -m pytest tests/test_gpu_rank.py tests/test_gpu_lanes.py -q -x -p no:cacheprovider 2>&1 | tail -2
PF_LANES=1 timeout 900 python -m pytest tests/test_gpu_rank.py -q -x -p no:cacheprovider 2>&1 | tail -1
