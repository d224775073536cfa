timeout 900 python -m pytest tests/test_gpu_lanes.py -q -x -p no:cacheprovider 2>&1 | tail -2
for NL in 2 3 4; do
for M in 4 8; do
PF_LANES=$NL timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_l$M.json 2> gpurun_out/b_l$M.err
echo "lanes $NL: $(python tools/summarize_bench.py gpurun_out/b_l$M.json 2>/dev/null | head -1)"
done; done
