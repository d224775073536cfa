timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export PF_ATTN_SINGLE=1; fi
  timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "== single=$v"; python tools/summarize_bench.py gpurun_out/ab.json | grep -E "value|attention"
done
unset PF_ATTN_SINGLE
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
