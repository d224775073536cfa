timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lanes.py -q -x -p no:cacheprovider -o faulthandler_timeout=300 2>&1 | tail -1
for v in 0 1; do
for M in 4 8; do
PF_ATTN_HALVES=$v timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_h$v$M.json 2> gpurun_out/b_h$v$M.err
echo "halves=$v $(python tools/summarize_bench.py gpurun_out/b_h$v$M.json 2>/dev/null | head -1)"
done; done
PF_LANES=1 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches 8 > gpurun_out/b_h1l.json 2> gpurun_out/b_h1l.err
echo "halves=1 lanes=1 $(python tools/summarize_bench.py gpurun_out/b_h1l.json 2>/dev/null | grep -E 'value|attention')"
