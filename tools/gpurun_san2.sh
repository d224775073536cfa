export PYTHONWARNINGS=ignore
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python tools/san_streamk.py > gpurun_out/san_sk.log 2>&1; echo "streamk memcheck rc=$?"; tail -4 gpurun_out/san_sk.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python tools/san_streamk.py > gpurun_out/san_sk_race.log 2>&1; echo "streamk racecheck rc=$?"; tail -4 gpurun_out/san_sk_race.log
