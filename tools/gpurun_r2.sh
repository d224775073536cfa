for v in 0 1; do
PF_RESID_2SM=$v timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches 1 > gpurun_out/b_r$v.json 2> gpurun_out/b_r$v.err
python tools/summarize_bench.py gpurun_out/b_r$v.json | grep -E "value|out_proj|mlp_out"
done
