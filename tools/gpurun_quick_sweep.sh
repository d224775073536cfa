set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for M in 1 2 4 8; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --patches $M > gpurun_out/bench_m$M.json 2> gpurun_out/bench_m$M.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_m$M.json'))
ks={k: (round(v['ms_per_image'],1), v['launches']) for k,v in d['kernels'].items()}
print('M=$M', 'value', round(d['value'],4), 'e2e', round(d['e2e']['value'],4), 'tc', round(d['tc_frac_image'],3), ks)
"
done
