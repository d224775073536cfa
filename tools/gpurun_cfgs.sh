for C in c2px c3 c4 c5; do
timeout 1200 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --config $C > gpurun_out/final_$C.json 2> gpurun_out/final_$C.err
python tools/summarize_bench.py gpurun_out/final_$C.json 2>/dev/null | head -3
done
