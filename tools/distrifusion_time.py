"""DistriFusion on one B200 (all workers' shards on the stage's patch lanes),
C2 shape: device seconds per image through run_distrifusion_device. Probe
for profiles/, not the bench."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2405_14430_b200 as pf  # noqa: E402

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p, hs = 4096, 1152
with pf.ToyDiTCuda(0, 28, hs, 16, 4.0, p, 1) as m:
    x = torch.from_numpy(pf.make_initial_latent(0, p, hs).astype(np.float32)).cuda()
    st = torch.cuda.Stream()
    x0 = pf.make_initial_latent(0, p, hs)
    for _ in range(2):
        m.run_distrifusion(x0, 20, workers, 1, 0.1)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record()
        m.run_distrifusion_device(x.data_ptr(), 20, workers, 1, 0.1, st.cuda_stream)
        with torch.cuda.stream(st):
            e1.record()
        m.synchronize(st.cuda_stream)
        ts.append(e0.elapsed_time(e1) / 1e3)
    print(json.dumps({"executor": "distrifusion", "workers": workers, "steps": 20, "warmup": 1,
                      "sec_per_image": min(ts), "all": ts}))
