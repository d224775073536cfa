"""Rank-mode liveness probe on one GPU: N same-process ranks (device 0) run
the toy PipeFusion plan with graphs on/off; prints OK/mismatch per run.
Run each configuration in its own process under `timeout`.

    python tools/rank_debug.py N M S W graphs(0|1) runs
"""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_14430_b200 as pf  # noqa: E402

N, M, S, W, graphs, runs = (int(a) for a in sys.argv[1:7])
warm = len(sys.argv) > 7 and sys.argv[7] == "warm"  # one graph-less run first
L, hs, heads, p = 4, 128, 4, 256
x0 = pf.make_initial_latent(0, p, hs)
with pf.ToyDiTCuda(0, L, hs, heads, 4.0, p, N) as m:
    ref = m.run_pipefusion(x0, S, M, W, 0.1).final_x
ranks = [pf.ToyDiTCuda.rank_stage(0, L, hs, heads, 4.0, p, r, N, 0) for r in range(N)]
pf.connect_ranks(ranks)
for m in ranks:
    m.set_graphs(bool(graphs) and not warm)
streams = [torch.cuda.Stream() for _ in ranks]
x = torch.from_numpy(x0.astype(np.float32)).cuda()
for it in range(runs):
    x.copy_(torch.from_numpy(x0.astype(np.float32)))
    torch.cuda.synchronize()
    t0 = time.time()
    for r, m in enumerate(ranks):
        m.run_pipefusion_device(x.data_ptr() if r == 0 else 0, S, M, W, 0.1,
                                streams[r].cuda_stream)
        print(f"run {it}: rank {r} enqueued ({time.time() - t0:.2f}s)", flush=True)
    for r, m in enumerate(ranks):
        m.synchronize(streams[r].cuda_stream)
        print(f"run {it}: rank {r} done ({time.time() - t0:.2f}s)", flush=True)
    got = x.double().cpu().numpy()
    print(f"run {it}: {'OK' if np.array_equal(got, ref) else 'MISMATCH'}", flush=True)
    if warm:
        for m in ranks:
            m.set_graphs(bool(graphs))
