import torch
x = torch.zeros(1024, device="cuda")
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for _ in range(20):
            x.add_(1)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print("torch add_ in graph: %.2f us per kernel" % (e0.elapsed_time(e1) * 1e3 / 20))
