"""Time the attention kernel alone at a given shape and dump the clock64
timeline of CTA (0,0,0) (debug instrumentation; not a bench)."""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2405_14430_b200 as pf  # noqa: E402

P, heads, hs, rows, row0 = [int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (4096, 16, 1152, 4096, 0))]
lib = pf.load_library()
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: ((torch.rand(P, hs, device="cuda", generator=g) * 2 - 1) * 2).to(torch.bfloat16)
q, k, v = mk(), mk(), mk()
out = torch.zeros(P, hs, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.current_stream().cuda_stream
sumcol = int(__import__("os").environ.get("PF_DEBUG_SUMCOL", "1"))  # production V layout
run = lambda: lib.pf_debug_attention_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                        out.data_ptr(), P, rows, row0, heads, hs, s, sumcol)
for _ in range(3):
    run()
torch.cuda.synchronize()
# pf_debug_attention includes repacking kernels; time the whole call and note it
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
print("debug_attention call (incl. repack) us:", e0.elapsed_time(e1) / 10 * 1e3)
buf = (ctypes.c_ulonglong * (8192 + 4096 + 1024))()
lib.pf_debug_attention_trace(1, None)
run()
torch.cuda.synchronize()
lib.pf_debug_attention_trace(1, buf)
lib.pf_debug_attention_trace(0, None)
allb = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
a = allb[:8192]
cta = allb[8192:12288].reshape(1024, 4)
cta = cta[cta[:, 0] > 0]
if len(cta):
    t0 = cta[:, 0].min()
    ent, go, end = (cta[:, 0] - t0) / 1e3, (cta[:, 1] - t0) / 1e3, (cta[:, 2] - t0) / 1e3
    dur = end - go
    print(f"CTAs {len(cta)}: entry max {ent.max():.1f} us, after-wait max {go.max():.1f}, "
          f"end min/median/max {end.min():.1f}/{np.median(end):.1f}/{end.max():.1f} us; "
          f"duration min/median/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f}")
    order = np.argsort(dur)
    print("slowest CTAs (idx, sm, dur us):", [(int(i), int(cta[i, 3]), round(float(dur[i]), 1)) for i in order[-8:]])
    print("fastest CTAs:", [(int(i), int(cta[i, 3]), round(float(dur[i]), 1)) for i in order[:8]])
base = a[a > 0].min()
t = np.where(a > 0, a - base, -1)
nblk = int(((t[0:2048].reshape(256, 8)[:, 1]) >= 0).sum())  # blocks CTA 0 processed
res = {"softmax0": t[0:8 * nblk].reshape(nblk, 8).tolist(),
       "softmax1": t[2048:2048 + 8 * nblk].reshape(nblk, 8).tolist(),
       "mma": t[4096:4096 + 8 * nblk].reshape(nblk, 8).tolist(),
       "tma": t[6144:6144 + 8 * nblk].reshape(nblk, 8)[:, :4].tolist()}
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/attn_trace.json").write_text(json.dumps(res))
s1 = [r[1] for r in res["softmax0"]]
print("CTA 0 blocks:", nblk, "s_full-ready deltas (clk):", np.diff(s1).tolist())
print("first/last", res["softmax0"][0], res["softmax0"][-1])

for i in range(nblk):
    if res["softmax0"][i][6] >= 0 or res["mma"][i][6] >= 0 or res["tma"][i][3] >= 0:
        print("boundary/seg-start", i, "sm0", res["softmax0"][i], "sm1", res["softmax1"][i][6:],
              "mma", res["mma"][i], "tma", res["tma"][i])

ep = allb[12288:12288 + 128]
epr = np.where(ep > 0, ep - base, -1).reshape(2, 8, 8)
print("epilogue probes wg0:", epr[0][:3].tolist(), "wg1:", epr[1][:3].tolist())

# per-phase means over CTA 0's steady blocks (clk): S wait, load+max, exp+P store, row sum
for name in ("softmax0", "softmax1"):
    arr = np.array(res[name][2:nblk - 1], dtype=np.int64)
    if len(arr) == 0:
        continue
    ok = (arr[:, :6] >= 0).all(axis=1)
    arr = arr[ok]
    d = lambda a, b: float(np.mean(arr[:, b] - arr[:, a]))
    per = float(np.mean(np.diff(arr[:, 1])))
    print(f"{name}: period {per:.0f} clk | wait S {d(0, 1):.0f} | load+max {d(1, 2):.0f} | "
          f"pp {d(2, 3):.0f} | exp+store {d(3, 4):.0f} | sum {d(4, 5):.0f}")
mm = np.array(res["mma"][2:nblk - 1], dtype=np.int64)
if len(mm):
    print("mma: wait V", float(np.mean(mm[:, 1] - mm[:, 0])), "wait P0",
          float(np.mean(mm[:, 2] - mm[:, 1])), "issue0->P1", float(np.mean(mm[:, 4] - mm[:, 3])))
