timeout 500 python -m pytest tests/test_gpu_joint.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err
python tools/summarize_bench.py gpurun_out/bench_c5.json
