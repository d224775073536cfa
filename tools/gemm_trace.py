"""Per-CTA timeline of one 1-SM GEMM launch (pf_debug_gemm, fp32 store
epilogue) at a given shape: debug instrumentation, not a bench.

    python tools/gemm_trace.py rows N K
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2405_14430_b200 as pf  # noqa: E402

rows, N, K = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (512, 3456, 1152)
lib = pf.load_library()
a = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.empty(rows, N, device="cuda")
s = torch.cuda.current_stream().cuda_stream
run = lambda: lib.pf_debug_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), rows, 0, rows, N, K, s)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
# 20 launches replayed from a CUDA graph (no host work between them), warm L2
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    s = st.cuda_stream
    with torch.cuda.graph(g, stream=st):
        for _ in range(20):
            run()
g.replay()
torch.cuda.synchronize()
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 20
print(f"rows {rows} N {N} K {K}: {us:.1f} us per launch (graph, warm L2), "
      f"{2 * rows * N * K / us / 1e6:.0f} TF/s")
s = torch.cuda.current_stream().cuda_stream
buf = (ctypes.c_ulonglong * 2048)()
lib.pf_debug_gemm_trace(1, None)
flush.zero_()
run()
torch.cuda.synchronize()
lib.pf_debug_gemm_trace(1, buf)
lib.pf_debug_gemm_trace(0, None)
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(128, 16)
t = t[t[:, 0] > 0]
if not len(t):
    sys.exit(0)
# clock64 per CTA (SM clock cycles) relative to kernel entry (slot 7)
rel = t[:, [7, 9, 10, 0, 1, 8, 2, 3, 4, 5]] - t[:, [7]]
names = ["entry", "pre_alloc", "post_alloc(w2)", "after_sync", "after_pdl", "A_issued", "first_full",
         "mma_issued", "acc_ready", "exit"]
for i, nme in enumerate(names):
    col = rel[:, i]
    print(f"  {nme:17s} min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d} clk")
