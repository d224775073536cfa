"""Kernel-level parity of the sm_100a kernels against plain fp32 torch.

GEMM  <- ditsim::matmul_rows   (toy_model.cpp:93-102)
Attn  <- ditsim::attention_rows (toy_model.cpp:104-143)
Inputs are bf16 (the kernels' operand type); the reference computation is
fp32 on the same bf16 values, so the only differences are accumulation order
(GEMM) and bf16 rounding of P plus exp2 approximation (attention).
"""
import ctypes

import pytest

torch = pytest.importorskip("torch")

from paper_2405_14430_b200 import load_library  # noqa: E402

pytestmark = pytest.mark.gpu


def _gemm(A, B, rows, row0):
    lib = load_library()
    N, K = B.shape
    C = torch.empty(rows, N, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    err = lib.pf_debug_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), rows, row0,
                            A.shape[0], N, K, s)
    torch.cuda.synchronize()
    assert err == 0, f"cuda error {err}"
    return C


@pytest.mark.parametrize("total,rows,row0,N,K", [
    (128, 128, 0, 128, 64),
    (256, 256, 0, 128, 128),
    (64, 64, 0, 32, 32),        # reference config hs=32
    (64, 16, 48, 96, 32),       # patch block, fused QKV width
    (32, 32, 0, 16, 16),        # hs=16 (K < BK, N < BN)
    (300, 170, 100, 200, 72),   # ragged everything
    (4096, 512, 1536, 3456, 1152),  # PixArt patch QKV
    (4096, 4096, 0, 1152, 4608),    # PixArt MLP-out full sequence (2-SM, BN 128)
    (4096, 4096, 0, 4608, 1152),    # PixArt MLP-in (2-SM, BN 256)
    (4096, 4096, 0, 3456, 1152),    # PixArt QKV (2-SM, BN 192)
    (1024, 1000, 24, 4608, 1152),   # 2-SM with a ragged last row tile
    (512, 300, 100, 96, 64),        # 2-SM with N < BN (B half partly out of range)
    (2048, 256, 1792, 3456, 1152),  # one 2-SM row tile, BN 192 (split-K 2 on 1-SM tiles)
    (4096, 512, 512, 1152, 1152),   # out-proj of a 512-row patch: split-K
    (4096, 512, 3584, 1152, 4608),  # MLP-out of a 512-row patch: split-K 4
    (1024, 100, 7, 1152, 1152),     # ragged rows, split-K
])
def test_gemm_matches_fp32(total, rows, row0, N, K):
    g = torch.Generator(device="cuda").manual_seed(total + N + K)
    A = (torch.rand(total, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    C = _gemm(A, B, rows, row0)
    assert torch.equal(C, _gemm(A, B, rows, row0))  # deterministic (split-K order fixed)
    ref = A[row0:row0 + rows].float() @ B.float().T
    err = (C - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-4 * max(1.0, scale) + 1e-3, (err, scale)


@pytest.mark.parametrize("total,rows,row0,N,K", [
    (4096, 4096, 0, 4608, 1152),
    (4096, 4096, 0, 3456, 1152),
    (4096, 3000, 96, 4608, 1152),   # ragged last row tile
])
def test_gemm_a_multicast_matches_fp32(monkeypatch, total, rows, row0, N, K):
    # opt-in 4-CTA clusters (two CTA pairs multicasting the A tile)
    monkeypatch.setenv("PF_A_MULTICAST", "1")
    test_gemm_matches_fp32(total, rows, row0, N, K)


def _attn(q, k, v, heads, rows, row0, sumcol=False):
    lib = load_library()
    P, hs = q.shape
    out = torch.zeros(P, hs, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    err = lib.pf_debug_attention_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                    P, rows, row0, heads, hs, s, int(sumcol))
    torch.cuda.synchronize()
    assert err == 0, f"cuda error {err}"
    return out


def _attn_ref(q, k, v, heads, rows, row0):
    P, hs = q.shape
    dh = hs // heads
    qf = q[row0:row0 + rows].float().view(rows, heads, dh).transpose(0, 1)
    kf = k.float().view(P, heads, dh).transpose(0, 1)
    vf = v.float().view(P, heads, dh).transpose(0, 1)
    s = qf @ kf.transpose(1, 2) / dh ** 0.5
    p = torch.softmax(s, dim=-1)
    return (p @ vf).transpose(0, 1).reshape(rows, hs)


@pytest.mark.parametrize("P,heads,hs,rows,row0,scale", [
    (64, 4, 32, 64, 0, 1.0),        # reference config, dh = 8
    (64, 4, 32, 16, 32, 1.0),       # one patch of four
    (32, 4, 16, 32, 0, 1.0),        # dh = 4
    (256, 4, 128, 64, 128, 3.0),    # tiny config patch, dh = 32
    (256, 4, 128, 256, 0, 3.0),
    (1024, 8, 512, 1024, 0, 4.0),   # dh = 64, two CTAs per item (halves, in-kernel merge)
    (4096, 16, 1152, 512, 1024, 3.0),  # PixArt patch, dh = 72, one CTA per item
    (4096, 16, 1152, 4096, 0, 3.0),    # PixArt full sequence
    (520, 2, 256, 136, 384, 2.0),   # ragged P / rows, dh = 128
    (6144, 24, 1536, 6144, 0, 2.0),  # stream-K, in-kernel merge, dh = 64
    (5000, 16, 1152, 4600, 200, 2.0),  # stream-K in-kernel merge, ragged P and rows
    (3000, 12, 768, 3000, 0, 2.0),  # stream-K, separate merge kernel
])
@pytest.mark.parametrize("sumcol", [False, True])
def test_attention_matches_fp32(P, heads, hs, rows, row0, scale, sumcol):
    # sumcol: the production V layout for padded head dims (row sum from the
    # PV MMA through V's padding column dh; no-op when dh is a multiple of 16)
    g = torch.Generator(device="cuda").manual_seed(P + hs + rows)
    mk = lambda: ((torch.rand(P, hs, device="cuda", generator=g) * 2 - 1) * scale).to(torch.bfloat16)
    q, k, v = mk(), mk(), mk()
    out = _attn(q, k, v, heads, rows, row0, sumcol)[row0:row0 + rows].float()
    ref = _attn_ref(q, k, v, heads, rows, row0)
    err = (out - ref).abs().max().item()
    # outputs reach |x| ~ scale: the bf16 output ulp there is scale * 2^-7
    # (0.031 at scale 4); P is rounded to bf16 before PV as well
    assert err < max(2e-2, 0.75 * scale * 2 ** -7), err
    rel = ((out - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel


def test_stream_k_attention_reruns_bitwise():
    # the in-kernel merge flags must be left zero after every launch: reruns
    # of a full-size (fused-merge) configuration are bitwise identical
    import numpy as np
    import paper_2405_14430_b200 as pf
    x0 = pf.make_initial_latent(0, 4096, 1152)
    with pf.ToyDiTCuda(0, 2, 1152, 16, 4.0, 4096, 1) as m:
        m.set_graphs(False)
        outs = [m.run_pipefusion(x0, 3, 1, 1, 0.1).final_x for _ in range(3)]
        m.set_graphs(True)
        outs += [m.run_pipefusion(x0, 3, 1, 1, 0.1).final_x for _ in range(2)]
    assert all(np.array_equal(o, outs[0]) for o in outs)


def test_residual_split_k_opt_in(monkeypatch):
    # opt-in split-K of skinny long-K residual GEMMs (workspace partials +
    # resid_reduce_kernel), one lane: same result as the unsplit GEMMs up to
    # fp32 summation order, and deterministic
    import numpy as np
    import paper_2405_14430_b200 as pf
    monkeypatch.setenv("PF_LANES", "1")
    x0 = pf.make_initial_latent(0, 4096, 1152)

    def run(split):
        if split:
            monkeypatch.setenv("PF_RESID_SPLITK", "1")
        else:
            monkeypatch.delenv("PF_RESID_SPLITK", raising=False)
        with pf.ToyDiTCuda(0, 2, 1152, 16, 4.0, 4096, 1) as m:
            return [m.run_pipefusion(x0, 3, 8, 1, 0.1).final_x for _ in range(2)]

    a, b = run(False), run(True)
    assert np.array_equal(b[0], b[1])
    rel = float(np.linalg.norm(a[0] - b[0]) / np.linalg.norm(a[0]))
    assert rel <= 1e-3, rel


@pytest.mark.parametrize("P,heads,hs,rows,row0", [
    (4096, 16, 1152, 4096, 0),   # C2 full sequence (stream-K, in-kernel merge)
    (4096, 16, 1152, 512, 2048),  # M = 8 patch
    (2048, 16, 1024, 2048, 0),   # dh 64
])
@pytest.mark.parametrize("sumcol", [False, True])
def test_attention_peaked_rows_rescale(P, heads, hs, rows, row0, sumcol):
    """Each query row's largest score sits at its own KV row (q = k), so the
    running max jumps mid-sequence and the lazy O rescale runs at a later
    block (random data rarely reaches it)."""
    g = torch.Generator(device="cuda").manual_seed(P + hs)
    x = (torch.rand(P, hs, device="cuda", generator=g) * 2 - 1) * 3.0
    ramp = torch.linspace(0.2, 1.6, P, device="cuda")[:, None]  # growing row norms
    q = (x * ramp).to(torch.bfloat16)
    k = q.clone()
    v = ((torch.rand(P, hs, device="cuda", generator=g) * 2 - 1)).to(torch.bfloat16)
    out = _attn(q, k, v, heads, rows, row0, sumcol)[row0:row0 + rows].float()
    ref = _attn_ref(q, k, v, heads, rows, row0)
    assert torch.isfinite(out).all()
    rel = ((out - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel


@pytest.mark.parametrize("P,heads,hs,rows,row0", [
    (520, 2, 256, 136, 384),      # dh 128 (64-row blocks), ragged
    (2048, 16, 2048, 2048, 0),    # dh 128, stream-K in-kernel merge
    (1000, 8, 768, 1000, 0),      # dh 96 (96-row blocks)
])
def test_attention_triple_buffered_wide_heads(monkeypatch, P, heads, hs, rows, row0):
    """The triple-buffered kernel at head dims above 80 (opt-in PF_ATTN3=2:
    measured slower than the single-buffered kernel at dh 128)."""
    monkeypatch.setenv("PF_ATTN3", "2")
    import subprocess
    import sys
    code = f"""
import torch, sys
sys.path.insert(0, {str(__import__('pathlib').Path(__file__).resolve().parents[1])!r})
sys.path.insert(0, {str(__import__('pathlib').Path(__file__).resolve().parent)!r})
from test_gpu_kernels import _attn, _attn_ref
g = torch.Generator(device="cuda").manual_seed(7)
mk = lambda: ((torch.rand({P}, {hs}, device="cuda", generator=g) * 2 - 1) * 2).to(torch.bfloat16)
q, k, v = mk(), mk(), mk()
out = _attn(q, k, v, {heads}, {rows}, {row0})[{row0}:{row0} + {rows}].float()
ref = _attn_ref(q, k, v, {heads}, {rows}, {row0})
rel = ((out - ref).norm() / ref.norm()).item()
assert rel < 1e-2, rel
print("ok", rel)
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr



@pytest.mark.parametrize("P,heads,hs", [(16896, 24, 3072), (16384, 24, 1536)])
def test_attention_strided_schedule_large_kv(P, heads, hs):
    """K/V of all heads beyond the L2 (Flux 2048 px: 24 heads x 16896 rows x
    dh 128): whole items dealt round-robin over the CTAs (AttnSchedule.strided).
    Checked on a sample of query rows of every head."""
    import numpy as np
    lib = load_library()
    g = torch.Generator(device="cuda").manual_seed(P + heads)
    mk = lambda: ((torch.rand(P, hs, device="cuda", generator=g) * 2 - 1) * 2).to(torch.bfloat16)
    q, k, v = mk(), mk(), mk()
    out = _attn(q, k, v, heads, P, 0).float()
    dh = hs // heads
    rows = torch.cat([torch.arange(0, 200), torch.arange(P // 2, P // 2 + 100),
                      torch.arange(P - 200, P)]).cuda()
    errs = []
    for h in range(heads):
        c = slice(h * dh, (h + 1) * dh)
        s = q[rows, c].float() @ k[:, c].float().T / dh ** 0.5
        ref = torch.softmax(s, dim=-1) @ v[:, c].float()
        got = out[rows, c]
        errs.append(((got - ref).norm() / ref.norm()).item())
    assert max(errs) < 1e-2, errs
