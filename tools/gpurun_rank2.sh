timeout 900 python -m pytest tests/test_gpu_rank.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -3
PF_RANK_COPY=1 timeout 900 python -m pytest tests/test_gpu_rank.py -q -x -p no:cacheprovider 2>&1 | tail -2
