timeout 600 python -m pytest tests/test_gpu_launch_count.py -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
