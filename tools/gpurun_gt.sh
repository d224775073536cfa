for shp in "512 3456 1152" "128 128 64"; do
timeout 120 python tools/gemm_trace.py $shp 2>&1 | tail -11
done
