set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"EpiGeluAffine" -s 1 -c 1 -o gpurun_out/prof_px_gelu -f python tools/one_image.py --config c2px --steps 2 > gpurun_out/ncu_px.log 2>&1; tail -2 gpurun_out/ncu_px.log
