# quick loop: GPU tests + bench (no CPU baseline)
set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -3 gpurun_out/bench_quick.err
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'tc_frac', d['tc_frac_image'], 'clocks', d['clocks'])
for k,v in d['kernels'].items(): print(k, {a: round(b,3) for a,b in v.items()})
"
