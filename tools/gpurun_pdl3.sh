for rep in 1 2; do
for v in 0 1; do
for M in 2 4 8; do
PF_LANES_PDL=$v timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_p.json 2> gpurun_out/b_p.err
echo "lanes_pdl=$v $(python tools/summarize_bench.py gpurun_out/b_p.json 2>/dev/null | head -1 | cut -c1-60)"
done; done; done
