timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider -o faulthandler_timeout=300 2>&1 | tail -1
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
for M in 1 8; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/b_fin$M.json 2> gpurun_out/b_fin$M.err
python tools/summarize_bench.py gpurun_out/b_fin$M.json 2>/dev/null | head -1 | cut -c1-90
done
