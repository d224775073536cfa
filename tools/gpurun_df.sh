timeout 900 python -m pytest tests/test_gpu_distrifusion.py -q -x -p no:cacheprovider 2>&1 | tail -15
