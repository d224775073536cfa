timeout 900 python -m pytest tests/test_gpu_lanes.py tests/test_gpu_rank.py tests/test_gpu_joint.py -q -x -p no:cacheprovider -o faulthandler_timeout=300 2>&1 | tail -2
for v in 1 4; do
PF_LANES=$v timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --config c4 --patches 8 > gpurun_out/b_c4l$v.json 2> gpurun_out/b_c4l$v.err
python tools/summarize_bench.py gpurun_out/b_c4l$v.json 2>/dev/null | head -1
done
