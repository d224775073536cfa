timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -3
for M in 1 8; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_m$M.json 2> gpurun_out/b_m$M.err
python tools/summarize_bench.py gpurun_out/b_m$M.json | grep -E "value|attention"
done
