"""fp64 numpy spec of the MMDiT block variants (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
anything under oracle/. This module is the checker of the GPU `block=mmdit`
path (pf_create_mmdit, include/pipefusion_b200.h): the SD3-medium and Flux.1
configurations BASELINE.json names (configs 4 and 5). The reference
(/root/reference/proj) has no such blocks -- its only block is the toy block
of toy_model.cpp:145-177 -- so, like oracle/px_oracle.c for PixArt, this is
the builder's own restatement of the public block definitions, run under
the reference's PipeFusion loop (run_pipefusion_inline, execute.cpp:167-223:
warmup, patch order, in-place K/V row writes, sampler x -= eta eps,
h = x_j + condition_bias) with the joint-row convention of the `joint`
block: T text rows precede the P image rows in every activation and K/V
buffer, and the text rows re-enter (from the text tokens y) with patch 0 of
every step.

Double-stream block (SD3 MM-DiT block / Flux double block), per stream
(image rows: stream 0, text rows: stream 1), at timestep index t of S:

    shift1, scale1, gate1, shift2, scale2, gate2 = mod[l, stream](t)   (adaLN-Zero)
    a = LN(h) (1 + scale1) + shift1               LN without affine, eps 1e-6
    q, k, v = a Wqkv + bqkv
    q, k <- RMSNorm per head (eps 1e-6) * g_q / g_k     (QK-norm)
    q, k <- RoPE (Flux only)                      k, v rows written in place
    h += gate1 (attention(q, K_joint, V_joint) Wo + bo)
    h += gate2 (gelu_tanh((LN(h) (1 + scale2) + shift2) W1 + b1) W2 + b2)

Single-stream block (Flux single block; one weight set for all joint rows,
attention and MLP read the same modulated input):

    shift, scale, gate = mod[l](t)
    a = LN(h) (1 + scale) + shift
    q, k, v = a Wqkv + bqkv;  z = gelu_tanh(a W1 + b1)
    q, k <- RMSNorm * g, RoPE;  k, v rows written in place
    h += gate (attention(q, K, V) Wo + z W2 + b2)

Conditioning: tau = 1000 t / S; sinusoid(tau) [256] = [cos(tau f_i), sin(tau f_i)],
f_i = exp(-ln(10000) i / 128); c = silu(sinusoid Wt1 + bt1) Wt2 + bt2 + y_pooled;
mod[l, stream](t) = silu(c) Wmod + bmod ([6 hs] double, [3 hs] single).

RoPE (Flux, theta 10000, axes (dh/8, 7 dh/16, 7 dh/16)): position ids
(0, 0, 0) for text rows, (0, i // W, i % W) for image row i, W = isqrt(P);
in axis a's segment [o_a, o_a + d_a) of each head, pair (o_a + 2j, o_a + 2j + 1)
is rotated by pos_a theta^(-2j / d_a).

Parameters: element i of tensor `tid` is U[-1,1) = (splitmix64(key ^ (i *
0xD1B54A32D192ED03)) >> 11) 2^-52 * 2 - 1 with key = splitmix64(seed + tid *
0x9E3779B97F4A7C15), times the tensor's scale (1/sqrt(fan_in) for matrices,
0.1 for biases, 1 + 0.1 u for RMS gains). A counter-based stream lets the GPU
generate a 12B-parameter Flux model in parallel on the device
(csrc/mmdit.cu) with the same values. Matrices are x.W oriented [in x out].
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLD = 0x9E3779B97F4A7C15
MIXI = 0xD1B54A32D192ED03

# tensor ids: layer l, stream s (0 image, 1 text), param k -> l * 64 + s * 32 + k
P_WQKV, P_BQKV, P_WO, P_BO, P_W1, P_B1, P_W2, P_B2, P_WMOD, P_BMOD, P_GQ, P_GK = range(12)
G_WT1, G_BT1, G_WT2, G_BT2, G_YP, G_CB, G_Y = range(7)
GLOBAL_TID = 1 << 20
FREQ = 256


def _splitmix(x):
    x = (x + np.uint64(GOLD)) if isinstance(x, np.ndarray) else np.uint64((int(x) + GOLD) & M64)
    z = x
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform(seed: int, tid: int, n: int) -> np.ndarray:
    """n values U[-1,1) of tensor `tid` (see the module docstring)."""
    with np.errstate(over="ignore"):
        key = _splitmix(np.uint64((seed + tid * GOLD) & M64))
        i = np.arange(n, dtype=np.uint64)
        z = _splitmix(key ^ (i * np.uint64(MIXI)))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def tid_of(layer, stream, k):
    return layer * 64 + stream * 32 + k


class MMDiT:
    """Parameters of pf_create_mmdit(seed, desc, text_tokens, double_layers, rope)."""

    def __init__(self, seed, layers, hs, heads, mlp, T, P, double_layers, rope=False):
        self.seed, self.L, self.hs, self.heads, self.mlp = seed, layers, hs, heads, mlp
        self.T, self.P, self.D, self.rope = T, P, double_layers, rope
        self.dh = hs // heads
        h, m, dh = hs, mlp, self.dh
        self.layers = []
        for l in range(layers):
            double = l < double_layers
            streams = []
            for s in range(2 if double else 1):
                def t(k, shape, scale, gain=False):
                    u = uniform(seed, tid_of(l, s, k), int(np.prod(shape))).reshape(shape)
                    return 1.0 + 0.1 * u if gain else u * scale
                w6 = 6 * h if double else 3 * h
                streams.append(dict(
                    wqkv=t(P_WQKV, (h, 3 * h), 1 / math.sqrt(h)), bqkv=t(P_BQKV, (3 * h,), 0.1),
                    wo=t(P_WO, (h, h), 1 / math.sqrt(h)), bo=t(P_BO, (h,), 0.1),
                    w1=t(P_W1, (h, m), 1 / math.sqrt(h)), b1=t(P_B1, (m,), 0.1),
                    w2=t(P_W2, (m, h), 1 / math.sqrt(m)), b2=t(P_B2, (h,), 0.1),
                    wmod=t(P_WMOD, (h, w6), 1 / math.sqrt(h)), bmod=t(P_BMOD, (w6,), 0.1),
                    gq=t(P_GQ, (dh,), 0, True), gk=t(P_GK, (dh,), 0, True)))
            self.layers.append(streams)

        def g(k, shape, scale):
            return uniform(seed, GLOBAL_TID + k, int(np.prod(shape))).reshape(shape) * scale
        self.wt1 = g(G_WT1, (FREQ, h), 1 / math.sqrt(FREQ))
        self.bt1 = g(G_BT1, (h,), 0.1)
        self.wt2 = g(G_WT2, (h, h), 1 / math.sqrt(h))
        self.bt2 = g(G_BT2, (h,), 0.1)
        self.yp = g(G_YP, (h,), 1.0)
        self.cb = g(G_CB, (h,), 1.0)
        self.y = g(G_Y, (T, h), 1.0)
        side = math.isqrt(P)
        self.pos = np.zeros((T + P, 3))
        self.pos[T:, 1] = np.arange(P) // side
        self.pos[T:, 2] = np.arange(P) % side

    # ---------------------------------------------------------------- pieces
    def cond(self, t, steps):
        tau = 1000.0 * t / steps
        f = np.exp(-math.log(10000.0) * np.arange(FREQ // 2) / (FREQ // 2))
        sinus = np.concatenate([np.cos(tau * f), np.sin(tau * f)])
        e1 = silu(sinus @ self.wt1 + self.bt1)
        c = e1 @ self.wt2 + self.bt2 + self.yp
        return silu(c)

    def mod(self, l, stream, t, steps):
        st = self.layers[l][stream]
        return self.cond(t, steps) @ st["wmod"] + st["bmod"]

    def qk_post(self, x, g, rows_pos):
        """RMSNorm per head (* gain), then RoPE (Flux) for rows at `rows_pos`."""
        n, hs = x.shape
        xh = x.reshape(n, self.heads, self.dh)
        xh = xh / np.sqrt((xh * xh).mean(axis=2, keepdims=True) + 1e-6) * g
        if self.rope:
            xh = rope(xh, rows_pos, self.dh)
        return xh.reshape(n, hs)


def silu(x):
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def ln_mod(h, shift, scale):
    mu = h.mean(axis=1, keepdims=True)
    var = ((h - mu) ** 2).mean(axis=1, keepdims=True)
    return (h - mu) / np.sqrt(var + 1e-6) * (1.0 + scale) + shift


def rope_axes(dh):
    return (dh // 8, 7 * dh // 16, 7 * dh // 16)


def rope(xh, pos, dh, theta=10000.0):
    out = xh.copy()
    off = 0
    for a, d in enumerate(rope_axes(dh)):
        j = np.arange(d // 2)
        w = theta ** (-2.0 * j / d)
        ang = pos[:, a:a + 1] * w[None, :]            # [n, d/2]
        c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
        x0 = xh[:, :, off + 2 * j]
        x1 = xh[:, :, off + 2 * j + 1]
        out[:, :, off + 2 * j] = c * x0 - s * x1
        out[:, :, off + 2 * j + 1] = s * x0 + c * x1
        off += d
    return out


def attention_rows(q, k, v, heads):
    dh = k.shape[1] // heads
    out = np.empty_like(q)
    for h in range(heads):
        c = slice(h * dh, (h + 1) * dh)
        s = q[:, c] @ k[:, c].T / np.sqrt(dh)
        s = s - s.max(axis=1, keepdims=True)
        e = np.exp(s)
        out[:, c] = (e @ v[:, c]) / e.sum(axis=1, keepdims=True)
    return out


def layer_forward(m: MMDiT, l, t, steps, h, kb, vb, row0):
    """Block l over joint rows [row0, row0 + len(h)) (text rows first)."""
    T, hs = m.T, m.hs
    n = h.shape[0]
    rows = np.arange(row0, row0 + n)
    txt = rows < T
    pos = m.pos[rows]
    streams = m.layers[l]
    if len(streams) == 2:
        a = np.empty_like(h)
        q = np.empty_like(h)
        mods = [m.mod(l, s, t, steps) for s in (0, 1)]
        for s, sel in ((0, ~txt), (1, txt)):
            if not sel.any():
                continue
            st, md = streams[s], mods[s]
            a[sel] = ln_mod(h[sel], md[:hs], md[hs:2 * hs])
            qkv = a[sel] @ st["wqkv"] + st["bqkv"]
            q[sel] = m.qk_post(qkv[:, :hs], st["gq"], pos[sel])
            kb[rows[sel]] = m.qk_post(qkv[:, hs:2 * hs], st["gk"], pos[sel])
            vb[rows[sel]] = qkv[:, 2 * hs:]
        o = attention_rows(q, kb, vb, m.heads)
        h = h.copy()
        for s, sel in ((0, ~txt), (1, txt)):
            if not sel.any():
                continue
            st, md = streams[s], mods[s]
            h[sel] += md[2 * hs:3 * hs] * (o[sel] @ st["wo"] + st["bo"])
            a2 = ln_mod(h[sel], md[3 * hs:4 * hs], md[4 * hs:5 * hs])
            h[sel] += md[5 * hs:] * (gelu_tanh(a2 @ st["w1"] + st["b1"]) @ st["w2"] + st["b2"])
        return h
    st = streams[0]
    md = m.mod(l, 0, t, steps)
    a = ln_mod(h, md[:hs], md[hs:2 * hs])
    qkv = a @ st["wqkv"] + st["bqkv"]
    z = gelu_tanh(a @ st["w1"] + st["b1"])
    q = m.qk_post(qkv[:, :hs], st["gq"], pos)
    kb[rows] = m.qk_post(qkv[:, hs:2 * hs], st["gk"], pos)
    vb[rows] = qkv[:, 2 * hs:]
    o = attention_rows(q, kb, vb, m.heads)
    return h + md[2 * hs:] * (o @ st["wo"] + z @ st["w2"] + st["b2"])


def pipefusion(m: MMDiT, x_init, steps, patches, warmup, eta):
    """run_pipefusion_inline (execute.cpp:167-223) with the MMDiT blocks."""
    p, hs = x_init.shape
    T = m.T
    r = p // patches
    kv = [[np.zeros((T + p, hs)), np.zeros((T + p, hs))] for _ in range(m.L)]
    x = np.array(x_init, dtype=np.float64)
    for w in range(warmup):
        t = steps - 1 - w
        h = np.concatenate([m.y, x + m.cb])
        for l in range(m.L):
            h = layer_forward(m, l, t, steps, h, kv[l][0], kv[l][1], 0)
        x = x - eta * h[T:]
    steady = steps - warmup
    eps = np.zeros_like(x)
    pending = np.zeros_like(x)
    for q in range(steady):
        t = steps - warmup - 1 - q
        for j in range(patches):
            rows = slice(j * r, (j + 1) * r)
            if q > 0:
                x[rows] -= eta * pending[rows]
            hi = x[rows] + m.cb
            h, row0 = (np.concatenate([m.y, hi]), 0) if j == 0 else (hi, T + j * r)
            for l in range(m.L):
                h = layer_forward(m, l, t, steps, h, kv[l][0], kv[l][1], row0)
            eps[rows] = h[-r:]
        pending = eps.copy()
    if steady > 0:
        x = x - eta * pending
    return x


def serial(m: MMDiT, x_init, steps, eta):
    """serial_reference (toy_model.cpp:201-214) with the MMDiT blocks."""
    return pipefusion(m, x_init, steps, 1, steps, eta)
