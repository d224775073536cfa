for rep in 1 2; do
for v in 1 0; do
for M in 4 8; do
PF_ATTN_HALVES=$v timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_p.json 2> gpurun_out/b_p.err
echo "halves=$v $(python tools/summarize_bench.py gpurun_out/b_p.json 2>/dev/null | head -1 | cut -c1-60)"
done; done; done
