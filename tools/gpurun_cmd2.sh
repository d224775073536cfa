set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
nproc; lscpu | grep "Model name"
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -25
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -5 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/one_image.py --steps 2 > gpurun_out/ncu_list.log 2>&1; tail -3 gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 4 -c 4 -o gpurun_out/prof_gemm python tools/one_image.py --steps 2 > gpurun_out/ncu_gemm.log 2>&1; tail -3 gpurun_out/ncu_gemm.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_attn python tools/one_image.py --steps 2 > gpurun_out/ncu_attn.log 2>&1; tail -3 gpurun_out/ncu_attn.log
