for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_rank$N.json 2> gpurun_out/bench_rank$N.err; tail -2 gpurun_out/bench_rank$N.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_rank$N.json').read().strip().splitlines()[-1])
print('N=$N value', d['value'], 'e2e', d['e2e']['value'], 'proc', d['processes'], 'finite', d['finite'], 'launches', d['gpu_launches'])
"
PF_LANES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_rank${N}_1l.json 2> gpurun_out/bench_rank${N}_1l.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_rank${N}_1l.json').read().strip().splitlines()[-1])
print('N=$N one lane value', d['value'], 'e2e', d['e2e']['value'])
"
done
