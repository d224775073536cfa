set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_attn_v4 -f python tools/one_image.py --steps 2 > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
