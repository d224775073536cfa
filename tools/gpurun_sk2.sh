for v in 0 1; do
for M in 4 8; do
PF_NO_RESID_SPLITK=$v timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_sk$v$M.json 2> gpurun_out/b_sk$v$M.err
echo "nosplitk=$v $(python tools/summarize_bench.py gpurun_out/b_sk$v$M.json 2>/dev/null | head -1)"
done; done
