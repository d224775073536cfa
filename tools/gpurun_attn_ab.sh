for v in 0 1 2 3 0; do
  PF_ATTN_POLY=$v timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "== poly variant $v"; python tools/summarize_bench.py gpurun_out/ab.json | grep -E "attention"
done
PF_ATTN_SINGLE=1 timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
echo "== single"; python tools/summarize_bench.py gpurun_out/ab.json | grep -E "attention"
