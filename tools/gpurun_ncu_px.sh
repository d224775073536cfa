set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_px.csv python tools/one_image.py --config c2px --steps 2 > gpurun_out/ncu_list_px.log 2>&1; tail -2 gpurun_out/ncu_list_px.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"EpiGeluAffine|EpiQKVAffine|px_fold|px_gemv" -s 0 -c 6 -o gpurun_out/prof_px -f python tools/one_image.py --config c2px --steps 2 > gpurun_out/ncu_px.log 2>&1; tail -2 gpurun_out/ncu_px.log
