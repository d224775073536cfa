set -x
rm -rf gpurun_out/timeline; mkdir -p gpurun_out/timeline
PF_TIMELINE_OUT=gpurun_out/timeline timeout 900 python -m pytest tests/test_gpu_timeline.py -q -x -p no:cacheprovider 2>&1 | tail -15
cat gpurun_out/timeline/timeline_vs_simulator.jsonl
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
