for M in 8 1; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/b_m$M.json 2> gpurun_out/b_m$M.err
python tools/summarize_bench.py gpurun_out/b_m$M.json | grep -vE "sampler"
done
PF_NO_WEIGHT_PREFETCH=1 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches 8 > gpurun_out/b_m8n.json 2> gpurun_out/b_m8n.err
python tools/summarize_bench.py gpurun_out/b_m8n.json | grep -vE "sampler"
