set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_m8.csv python tools/one_image.py --config c2 --steps 3 --patches 8 > gpurun_out/ncu_m8.log 2>&1; tail -2 gpurun_out/ncu_m8.log
python tools/launch_summary.py gpurun_out/launches_m8.csv
