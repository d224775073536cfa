# A/B of GEMM dispatch switches at M=1 and M=8
for M in 1 8; do
for cfg in "base" "PF_RESID_2SM=1" "PF_GEMM_2SM_192=1" "PF_RESID_2SM=1 PF_GEMM_2SM_192=1"; do
  if [ "$cfg" = base ]; then envs=""; else envs="$cfg"; fi
  env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "== M=$M $cfg"; python tools/summarize_bench.py gpurun_out/ab.json | grep -E "value|qkv|out_proj|mlp"
done; done
