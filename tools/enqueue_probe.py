"""Host enqueue time of one image (graphs off, as in rank mode) vs its device
time, C2 shape at a given M: probe, not a bench."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2405_14430_b200 as pf  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p, hs = 4096, 1152
with pf.ToyDiTCuda(0, 28, hs, 16, 4.0, p, 1) as m:
    m.set_graphs(False)
    x = torch.from_numpy(pf.make_initial_latent(0, p, hs).astype(np.float32)).cuda()
    st = torch.cuda.Stream()
    for _ in range(2):
        m.run_pipefusion_device(x.data_ptr(), 20, M, 1, 0.1, st.cuda_stream)
        m.synchronize(st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record()
    t0 = time.perf_counter()
    m.run_pipefusion_device(x.data_ptr(), 20, M, 1, 0.1, st.cuda_stream)
    t1 = time.perf_counter()
    with torch.cuda.stream(st):
        e1.record()
    m.synchronize(st.cuda_stream)
    t2 = time.perf_counter()
    print(f"M={M}: host enqueue {1e3 * (t1 - t0):.1f} ms, device {e0.elapsed_time(e1):.1f} ms, "
          f"wall {1e3 * (t2 - t0):.1f} ms, launches {m.last_launch_count()}")
