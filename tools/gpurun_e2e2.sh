timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b_e2e2.json 2> gpurun_out/b_e2e2.err
python tools/summarize_bench.py gpurun_out/b_e2e2.json | head -1
