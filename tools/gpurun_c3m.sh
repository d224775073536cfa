for M in 4 8; do
timeout 1200 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --config c3 --patches $M > gpurun_out/final_c3_m$M.json 2> gpurun_out/final_c3_m$M.err
python tools/summarize_bench.py gpurun_out/final_c3_m$M.json 2>/dev/null | head -1 | cut -c1-90
done
