set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_rank2.json 2> gpurun_out/bench_rank2.err; tail -5 gpurun_out/bench_rank2.err
python -c "
import json; d=json.load(open('gpurun_out/bench_rank2.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'proc', d['processes'], 'finite', d['finite'], 'launches', d['gpu_launches'])
"
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_single2.json 2> gpurun_out/bench_single2.err; tail -3 gpurun_out/bench_single2.err
python -c "
import json; d=json.load(open('gpurun_out/bench_single2.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'proc', d['processes'])
"
