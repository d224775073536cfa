timeout 500 python -m pytest tests/test_gpu_joint.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err
python tools/summarize_bench.py gpurun_out/bench_c4.json
