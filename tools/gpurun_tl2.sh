rm -rf gpurun_out/timeline
PF_TIMELINE_OUT=gpurun_out/timeline timeout 900 python -m pytest tests/test_gpu_timeline.py -q -p no:cacheprovider 2>&1 | tail -1
cat gpurun_out/timeline/timeline_vs_simulator.jsonl
