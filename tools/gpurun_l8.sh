for L in 4 6 8; do
PF_LANES=$L timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches 8 > gpurun_out/b_l.json 2> gpurun_out/b_l.err
echo "lanes=$L $(python tools/summarize_bench.py gpurun_out/b_l.json 2>/dev/null | head -1 | cut -c1-80)"
done
