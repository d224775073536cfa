for M in 8; do
PF_ATTN_ONE_ITEM_PER_CTA=1 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_pi$M.json 2> gpurun_out/b_pi$M.err
echo "per-item $(python tools/summarize_bench.py gpurun_out/b_pi$M.json 2>/dev/null | head -1)"
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_d$M.json 2> gpurun_out/b_d$M.err
echo "default $(python tools/summarize_bench.py gpurun_out/b_d$M.json 2>/dev/null | head -1)"
done
