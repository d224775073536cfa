timeout 600 ncu --set full --clock-control none --import-source on -k gemm_bf16_tn_kernel -s 30 -c 3 -o gpurun_out/m8_gemms -f python tools/one_image.py --steps 2 --warmup 1 --patches 8 > gpurun_out/ncu_qkv.log 2>&1
tail -2 gpurun_out/ncu_qkv.log
python tools/ncu_summary.py gpurun_out/m8_gemms.ncu-rep
ncu -i gpurun_out/m8_gemms.ncu-rep --page details --csv 2>/dev/null | grep -iE "Warp Cycles Per Issued|L2 Hit Rate|Duration|Elapsed Cycles|SM Frequency|Memory Throughput" | head -30
