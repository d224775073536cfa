for M in 1 8; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_m$M.json 2> gpurun_out/b_m$M.err
python tools/summarize_bench.py gpurun_out/b_m$M.json | grep -E "value|attention|gemm_qkv|out_proj"
done
