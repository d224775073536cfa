set -x
timeout 600 python -m pytest tests/test_gpu_rank.py -q -x -p no:cacheprovider 2>&1 | tail -25
