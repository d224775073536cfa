timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_m8.csv python tools/one_image.py --steps 2 --warmup 1 --patches 8 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_m8.csv | head -20
