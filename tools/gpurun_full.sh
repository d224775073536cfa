# full round check: GPU tests, smoke, bench (with CPU baseline), reference arm, launch list, ncu captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
nproc; lscpu | grep "Model name"
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1; tail -3 gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_attn -f python tools/one_image.py --steps 2 > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 10 -c 8 -o gpurun_out/prof_gemm -f python tools/one_image.py --steps 2 > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"patch_prepare|latent_update" -s 2 -c 2 -o gpurun_out/prof_sampler -f python tools/one_image.py --steps 2 > gpurun_out/ncu_sampler.log 2>&1; tail -2 gpurun_out/ncu_sampler.log
