# ncu captures of the top kernels (one GPU, one image with 2 diffusion steps)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_attn_v3 -f python tools/one_image.py --steps 2 > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:EpiResidual -s 4 -c 2 -o gpurun_out/prof_resid -f python tools/one_image.py --steps 2 > gpurun_out/ncu_resid.log 2>&1; tail -2 gpurun_out/ncu_resid.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:EpiTanh -s 2 -c 1 -o gpurun_out/prof_tanh -f python tools/one_image.py --steps 2 > gpurun_out/ncu_tanh.log 2>&1; tail -2 gpurun_out/ncu_tanh.log
