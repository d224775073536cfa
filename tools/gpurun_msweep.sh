set -x
for M in 1 2 4 8; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/bench_m$M.json 2> gpurun_out/bench_m$M.err
  python tools/summarize_bench.py gpurun_out/bench_m$M.json
done
