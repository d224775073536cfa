timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pixart.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in c2 c4; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
echo "== $c"; python tools/summarize_bench.py gpurun_out/b_$c.json | grep -E "value|out_proj|mlp_out"
done
