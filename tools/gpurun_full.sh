timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
for C in c4 c2px; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --config $C > gpurun_out/b_$C.json 2> gpurun_out/b_$C.err
python tools/summarize_bench.py gpurun_out/b_$C.json | grep -E "value|attention"
done
