for rep in 1 2; do
for v in 0 1; do
for M in 4 8; do
PF_NO_PDL=$v timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_pdl.json 2> gpurun_out/b_pdl.err
echo "nopdl=$v $(python tools/summarize_bench.py gpurun_out/b_pdl.json 2>/dev/null | head -1 | cut -c1-80)"
done; done; done
