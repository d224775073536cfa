timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -2
for shp in "512 3456 1152" "128 128 64"; do
timeout 120 python tools/gemm_trace.py $shp 2>&1 | grep rows
done
for M in 8 1; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_m$M.json 2> gpurun_out/b_m$M.err
python tools/summarize_bench.py gpurun_out/b_m$M.json | grep -vE "sampler"
done
