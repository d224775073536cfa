timeout 900 python bench.py > gpurun_out/final2_c2.json 2> gpurun_out/final2_c2.err; tail -2 gpurun_out/final2_c2.err
python tools/summarize_bench.py gpurun_out/final2_c2.json
python -c "
import json; d=json.loads(open('gpurun_out/final2_c2.json').read().strip().splitlines()[-1]); print(sorted(d.keys())); print(d['roofline']); print(d['cpu_baseline']); print(d['e2e']); print(d['gpu_launches'], d['clocks'])"
