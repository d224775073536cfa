timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_gpu_distrifusion.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_e2e.json 2> gpurun_out/b_e2e.err
python tools/summarize_bench.py gpurun_out/b_e2e.json | head -1
