"""Run one PipeFusion image (for ncu launch lists / captures; not a bench).

    python tools/one_image.py [--config c2] [--steps S] [--patches M] [--stages N]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14430_b200 as pf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--patches", type=int, default=1)
ap.add_argument("--stages", type=int, default=1)
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
c = bench.CONFIGS[a.config]
if c.get("block") == "pixart":
    m = pf.PixArtCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], c["T"], a.stages,
                      [0] * a.stages)
elif c.get("block") == "mmdit":
    m = pf.MMDiTCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], c["T"], a.stages,
                     [0] * a.stages, double_layers=c["D"], rope=c["rope"])
elif c.get("block") == "joint":
    m = pf.JointDiTCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], c["T"], a.stages,
                        [0] * a.stages, double_layers=c.get("D"))
else:
    m = pf.ToyDiTCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], a.stages, [0] * a.stages)
x0 = torch.from_numpy(pf.make_initial_latent(0, c["p"], c["hs"]).astype(np.float32)).cuda()
s = torch.cuda.Stream()
for _ in range(a.repeat):
    x = x0.clone()
    m.run_pipefusion_device(x.data_ptr(), a.steps, a.patches, a.warmup, 0.1, s.cuda_stream)
    m.synchronize(s.cuda_stream)
print("launches", m.last_launch_count(), "finite", bool(torch.isfinite(x).all()))
