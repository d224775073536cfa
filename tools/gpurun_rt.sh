for v in 0 1; do
PF_NO_RESID_TMA=$v timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b_rt$v.json 2> gpurun_out/b_rt$v.err
python tools/summarize_bench.py gpurun_out/b_rt$v.json | grep -E "value|out_proj"
done
