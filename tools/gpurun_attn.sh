timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
for M in 1 8; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_m$M.json 2> gpurun_out/b_m$M.err
python tools/summarize_bench.py gpurun_out/b_m$M.json | grep -E "value|attention"
PF_ATTN_ONE_ITEM_PER_CTA=1 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_m${M}_old.json 2> gpurun_out/b_m${M}_old.err
python tools/summarize_bench.py gpurun_out/b_m${M}_old.json | grep -E "value|attention"
done
