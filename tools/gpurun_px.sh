# PixArt block: GPU parity tests, then toy + pixart bench (no CPU baseline)
set -x
timeout 900 python -m pytest tests/test_gpu_pixart.py -q -x 2>&1 | tail -25
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -3 gpurun_out/bench_quick.err
timeout 600 python bench.py --config c2px --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_px.json 2> gpurun_out/bench_px.err; tail -3 gpurun_out/bench_px.err
python - <<'PY'
import json
for f in ["gpurun_out/bench_quick.json", "gpurun_out/bench_px.json"]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, 'value', d['value'], 'e2e', d['e2e']['value'], 'tc', d['tc_frac_image'], 'clocks', d['clocks'])
    for k, v in d['kernels'].items(): print('  ', k, {a: round(b, 3) for a, b in v.items()})
PY
