for M in 1 2 4; do
  timeout 900 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --patches $M > gpurun_out/bench_c3_m$M.json 2> gpurun_out/bench_c3_m$M.err
  python tools/summarize_bench.py gpurun_out/bench_c3_m$M.json
done
