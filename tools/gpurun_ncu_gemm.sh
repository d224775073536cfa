set -x
# kernel order per layer: qkv(EpiQKV), attn, out-proj(EpiResidual), mlp-in(EpiTanh), mlp-out(EpiResidual)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 10 -c 4 -o gpurun_out/prof_gemm_v2 -f python tools/one_image.py --steps 2 > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
