for M in 2 4 8; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/final_c2_m$M.json 2> gpurun_out/final_c2_m$M.err
python tools/summarize_bench.py gpurun_out/final_c2_m$M.json 2>/dev/null | head -1
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config c3 --patches 4 > gpurun_out/final_c3_m4.json 2> gpurun_out/final_c3_m4.err
python tools/summarize_bench.py gpurun_out/final_c3_m4.json 2>/dev/null | head -1
