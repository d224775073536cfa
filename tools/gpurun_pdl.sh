set -x
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
for M in 1 8; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/bench_pdl_m$M.json 2> gpurun_out/bench_pdl_m$M.err
  PF_NO_PDL=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/bench_nopdl_m$M.json 2> gpurun_out/bench_nopdl_m$M.err
done
python tools/summarize_bench.py gpurun_out/bench_pdl_m1.json gpurun_out/bench_nopdl_m1.json gpurun_out/bench_pdl_m8.json gpurun_out/bench_nopdl_m8.json | grep value
