for v in 0 1 2 3 4 5; do
  PF_ATTN_VARIANT=$v timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "== variant $v"; python tools/summarize_bench.py gpurun_out/ab.json | grep -E "value|attention"
done
