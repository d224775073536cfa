timeout 900 python -m pytest tests/test_gpu_timeline.py -q -x -p no:cacheprovider -k "4-4" 2>&1 | grep -E "assert|Error" | head -10
