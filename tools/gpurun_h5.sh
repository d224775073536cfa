timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider -o faulthandler_timeout=300 2>&1 | tail -1
for M in 2 4 8; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/final_c2_m$M.json 2> gpurun_out/final_c2_m$M.err
python tools/summarize_bench.py gpurun_out/final_c2_m$M.json 2>/dev/null | head -1
done
for C in c2px c4; do
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --config $C --patches 8 > gpurun_out/final_${C}_m8.json 2> gpurun_out/final_${C}_m8.err
python tools/summarize_bench.py gpurun_out/final_${C}_m8.json 2>/dev/null | head -1
done
