"""compute-sanitizer workload for the stream-K attention schedules (fused
in-kernel merge, halves, one CTA per item, separate merge kernel) of both
attention kernels (triple-buffered attn3 with the row-sum column, and the
single-buffered one), patch lanes, the MMDiT blocks (QK-norm, RoPE, clipped
text-row residual tiles), the opt-in residual split-K and the stream-K
residual GEMM. Sanitizer input,
not a test."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_14430_b200 as pf  # noqa: E402

lib = pf.load_library()
s = torch.cuda.current_stream().cuda_stream
for P, heads, hs, rows, row0 in [(4096, 16, 1152, 4096, 0), (4096, 16, 1152, 512, 1024),
                                 (4096, 16, 1152, 2048, 0), (3000, 12, 768, 3000, 0)]:
    q, k, v = [(torch.rand(P, hs, device="cuda") - 0.5).to(torch.bfloat16) for _ in range(3)]
    out = torch.zeros(P, hs, dtype=torch.bfloat16, device="cuda")
    for sumcol in (0, 1):
        assert lib.pf_debug_attention_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                         out.data_ptr(), P, rows, row0, heads, hs, s,
                                         sumcol) == 0
    torch.cuda.synchronize()
with pf.MMDiTCuda(1, 2, 128, 4, 4.0, 256, 20, 1, double_layers=1, rope=True) as mm:
    c = mm.run_pipefusion(pf.make_initial_latent(0, 256, 128), 3, 2, 1, 0.1)
assert np.isfinite(c.final_x).all()
x0 = pf.make_initial_latent(0, 512, 128)
with pf.ToyDiTCuda(0, 2, 128, 4, 4.0, 512, 1) as m:
    a = m.run_pipefusion(x0, 3, 4, 1, 0.1)
os.environ["PF_RESID_SPLITK"] = "1"
os.environ["PF_LANES"] = "1"
with pf.ToyDiTCuda(0, 1, 1152, 16, 4.0, 1024, 1) as m:
    b = m.run_pipefusion(pf.make_initial_latent(0, 1024, 1152), 2, 8, 1, 0.1)
# stream-K residual GEMM (MLP-out of a 4096-row patch: 96 pair tiles of
# 256 x 192 on 74 pairs, cut tiles' partials through the split-K workspace)
rng = np.random.default_rng(3)
h, kk, vv = [rng.uniform(-1, 1, (4096, 1152)) for _ in range(3)]
with pf.ToyDiTCuda(0, 1, 1152, 16, 4.0, 4096, 1) as m:
    g = m.layer_forward(0, h, kk, vv, 0)[0]
print("ok", np.isfinite(a.final_x).all(), np.isfinite(b.final_x).all(), np.isfinite(g).all())
