set -x
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -4
for M in 1 8; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/bench_sk_m$M.json 2> gpurun_out/bench_sk_m$M.err
  python tools/summarize_bench.py gpurun_out/bench_sk_m$M.json
done
timeout 600 python bench.py --config c2px --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sk_px.json 2> gpurun_out/bench_sk_px.err
python tools/summarize_bench.py gpurun_out/bench_sk_px.json
