# end-of-round measurement: tests, smoke, bench (+CPU baseline), reference arm, ncu
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
nproc; lscpu | grep "Model name"
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -6
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; tail -2 gpurun_out/final_c2.err
python tools/summarize_bench.py gpurun_out/final_c2.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2>&1; tail -c 400 gpurun_out/final_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3500 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final_ncu_list.log 2>&1; tail -2 gpurun_out/final_ncu_list.log
python tools/launch_summary.py gpurun_out/final_launches.csv | head -12
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"attn_fwd|gemm" -s 12 -c 6 -o gpurun_out/final_prof -f python tools/one_image.py --steps 2 > gpurun_out/final_ncu_full.log 2>&1; tail -2 gpurun_out/final_ncu_full.log
python tools/ncu_summary.py gpurun_out/final_prof.ncu-rep > gpurun_out/final_ncu_full_summary.txt 2>&1; head -60 gpurun_out/final_ncu_full_summary.txt
for M in 2 4 8; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --patches $M > gpurun_out/final_c2_m$M.json 2> gpurun_out/final_c2_m$M.err
python tools/summarize_bench.py gpurun_out/final_c2_m$M.json | head -1
done
