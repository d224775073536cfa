timeout 900 python -m pytest tests/test_gpu_lanes.py tests/test_gpu_distrifusion.py -q -x -p no:cacheprovider -o faulthandler_timeout=300 2>&1 | tail -1
for L in 1 4; do PF_LANES=$L timeout 600 python tools/distrifusion_time.py 4 2>&1 | tail -1; done
