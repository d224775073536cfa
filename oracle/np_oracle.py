"""numpy fp64 restatement of the toy DiT block (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
anything under oracle/. This module is the quick, vectorised checker used for
random weights that do not come from the reference's mt19937_64 stream; it is
NOT bit-exact with the reference (numpy's matmul sums in a different order).
The bit-exact restatement is oracle/pf_oracle.c.

Follows /root/reference/proj/src/toy_model.cpp:
  matmul_rows        :93-102    -> x @ w
  attention_rows     :104-143   -> per-head softmax(q k^T / sqrt(dh)) v
  toy_layer_forward  :169-177   -> K/V rows written in place before attending
and the inline PipeFusion interpreter of execute.cpp:167-223.
"""
from __future__ import annotations

import numpy as np


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


def layer_forward(w, heads, h, k_buf, v_buf, row0):
    wq, wk, wv, wo, win, wout = w
    r = h.shape[0]
    q = h @ wq
    k_buf[row0:row0 + r] = h @ wk
    v_buf[row0:row0 + r] = h @ wv
    h = h + attention_rows(q, k_buf, v_buf, heads) @ wo
    h = h + np.tanh(h @ win) @ wout
    return h


def run_pipefusion(layers, cb, heads, x_init, steps, workers, patches, warmup, eta):
    """Inline interpreter (execute.cpp:167-223), staleness stats included."""
    p, hs = x_init.shape
    L = len(layers)
    bounds = [(d * L // workers, (d + 1) * L // workers) for d in range(workers)]
    kv = [[np.zeros((p, hs)), np.zeros((p, hs))] for _ in range(L)]
    x = x_init.astype(np.float64).copy()
    r = p // patches
    for w in range(warmup):
        h = x + cb
        for l in range(L):
            h = layer_forward(layers[l], heads, h, kv[l][0], kv[l][1], 0)
        x = x - eta * h
    steady = steps - warmup
    eps = np.zeros((p, hs))
    pending = np.zeros((p, hs))
    for q in range(steady):
        for j in range(patches):
            rows = slice(j * r, (j + 1) * r)
            if q > 0:
                x[rows] -= eta * pending[rows]
            h = x[rows] + cb
            for l in range(L):
                h = layer_forward(layers[l], heads, h, kv[l][0], kv[l][1], j * r)
            eps[rows] = h
        pending = eps.copy()
    if steady > 0:
        x = x - eta * pending
    return x


def serial_reference(layers, cb, heads, x_init, steps, eta):
    x = x_init.astype(np.float64).copy()
    p, hs = x.shape
    for _ in range(steps):
        h = x + cb
        for l in range(len(layers)):
            k = np.zeros((p, hs)); v = np.zeros((p, hs))
            h = layer_forward(layers[l], heads, h, k, v, 0)
        x = x - eta * h
    return x


def random_model(rng, L, hs, mlp):
    s = 1.0 / np.sqrt(hs)
    u = lambda *sh: rng.uniform(-1.0, 1.0, size=sh)
    layers = [(u(hs, hs) * s, u(hs, hs) * s, u(hs, hs) * s, u(hs, hs) * s,
               u(hs, mlp) * s, u(mlp, hs) * s) for _ in range(L)]
    return layers, u(hs)


# ---------------------------------------------------------------- PixArt block
# Independent numpy restatement of oracle/px_oracle.c (same spec, vectorised),
# used to cross-check the C oracle before it is trusted as the GPU checker.
def px_tvec(g, t, steps, hs):
    tau = 1000.0 * t / steps
    f = np.exp(-np.log(10000.0) * np.arange(128) / 128.0)
    sin_ = np.concatenate([np.cos(tau * f), np.sin(tau * f)])
    silu = lambda a: a / (1.0 + np.exp(-a))  # noqa: E731
    e1 = silu(sin_ @ g["wt1"] + g["bt1"])
    temb = e1 @ g["wt2"] + g["bt2"]
    return silu(temb) @ g["wt0"] + g["bt0"]


def _ln_mod(h, shift, scale):
    mu = h.mean(axis=1, keepdims=True)
    var = ((h - mu) ** 2).mean(axis=1, keepdims=True)
    return (h - mu) / np.sqrt(var + 1e-6) * (1.0 + scale) + shift


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def px_layer_forward(p, heads, mod, h, k_buf, v_buf, row0, y):
    """p: dict of one layer's parameters; mod = sst + tv [6 hs]; y text tokens."""
    hs = h.shape[1]
    sh1, sc1, g1, sh2, sc2, g2 = (mod[i * hs:(i + 1) * hs] for i in range(6))
    r = h.shape[0]
    a = _ln_mod(h, sh1, sc1)
    qkv = a @ p["wqkv"] + p["bqkv"]
    k_buf[row0:row0 + r] = qkv[:, hs:2 * hs]
    v_buf[row0:row0 + r] = qkv[:, 2 * hs:]
    h = h + g1 * (attention_rows(qkv[:, :hs], k_buf, v_buf, heads) @ p["wo"] + p["bo"])
    kc = y @ p["wkc"] + p["bkc"]
    vc = y @ p["wvc"] + p["bvc"]
    qc = h @ p["wqc"] + p["bqc"]
    h = h + attention_rows(qc, kc, vc, heads) @ p["woc"] + p["boc"]
    z = _gelu_tanh(_ln_mod(h, sh2, sc2) @ p["w1"] + p["b1"])
    return h + g2 * (z @ p["w2"] + p["b2"])


def px_pipefusion(o, x, steps, patches, warmup, eta):
    """Vectorised mirror of px_oracle.c pxo_pipefusion for an oracle model `o`
    (loader.PixArtOracle): same loop, numpy matmuls (not bit-exact with C)."""
    L, hs, heads = o.layers, o.hs, o.heads
    g = {n: o.glob(n) for n in ("wt1", "bt1", "wt2", "bt2", "wt0", "bt0", "cb", "y")}
    prm = [{n: o.param(l, n) for n in ("wqkv", "bqkv", "wo", "bo", "wqc", "bqc", "wkc", "bkc",
                                       "wvc", "bvc", "woc", "boc", "w1", "b1", "w2", "b2",
                                       "sst")} for l in range(L)]
    p = x.shape[0]
    r = p // patches
    x = np.array(x, dtype=np.float64)
    kb = [np.zeros((p, hs)) for _ in range(L)]
    vb = [np.zeros((p, hs)) for _ in range(L)]
    for w in range(warmup):
        t = steps - 1 - w
        tv = px_tvec(g, t, steps, hs)
        h = x + g["cb"]
        for l in range(L):
            h = px_layer_forward(prm[l], heads, prm[l]["sst"].reshape(-1) + tv, h, kb[l], vb[l],
                                 0, g["y"])
        x = x - eta * h
    steady = steps - warmup
    pending = np.zeros_like(x)
    eps = np.zeros_like(x)
    for q in range(steady):
        t = steady - 1 - q
        tv = px_tvec(g, t, steps, hs)
        for j in range(patches):
            sl = slice(j * r, (j + 1) * r)
            if q > 0:
                x[sl] = x[sl] - eta * pending[sl]
            h = x[sl] + g["cb"]
            for l in range(L):
                h = px_layer_forward(prm[l], heads, prm[l]["sst"].reshape(-1) + tv, h, kb[l],
                                     vb[l], j * r, g["y"])
            eps[sl] = h
        pending = eps.copy()
    if steady > 0:
        x = x - eta * pending
    return x


# ---------------------------------------------------------------- joint block
# SD3-style joint-attention (MMDiT double-stream) block with the toy block's
# arithmetic per stream (csrc/runtime.cpp layer_forward_joint): text rows
# [0, J) use the text weights, image rows the image weights, every query row
# attends over all joint K/V rows.
def joint_layer_forward(w_img, w_txt, heads, h, k_buf, v_buf, row0, J):
    rows = h.shape[0]
    t_rows = max(0, min(row0 + rows, J) - row0)
    parts = [(w_txt, 0, t_rows)] if t_rows else []
    if rows > t_rows:
        parts.append((w_img, t_rows, rows))
    q = np.empty_like(h)
    for w, a, b in parts:
        q[a:b] = h[a:b] @ w[0]
        k_buf[row0 + a:row0 + b] = h[a:b] @ w[1]
        v_buf[row0 + a:row0 + b] = h[a:b] @ w[2]
    att = attention_rows(q, k_buf, v_buf, heads)
    out = h.copy()
    for w, a, b in parts:
        out[a:b] = out[a:b] + att[a:b] @ w[3]
        out[a:b] = out[a:b] + np.tanh(out[a:b] @ w[4]) @ w[5]
    return out


def single_layer_forward(w, heads, h, k_buf, v_buf, row0):
    """Flux-style single-stream block, toy arithmetic: attention and MLP both
    read the block input; one weight set for every joint row."""
    r = h.shape[0]
    q = h @ w[0]
    k_buf[row0:row0 + r] = h @ w[1]
    v_buf[row0:row0 + r] = h @ w[2]
    z = np.tanh(h @ w[4])
    return h + attention_rows(q, k_buf, v_buf, heads) @ w[3] + z @ w[5]


def _joint_or_single(layer, heads, h, kb, vb, row0, J):
    wi, wt = layer
    if wt is None:
        return single_layer_forward(wi, heads, h, kb, vb, row0)
    return joint_layer_forward(wi, wt, heads, h, kb, vb, row0, J)


def joint_pipefusion(layers, cb, y, heads, x_init, steps, patches, warmup, eta):
    """The reference's inline PipeFusion loop (execute.cpp:167-223) with the
    joint block; the text rows re-enter from y with patch 0 of every step."""
    p, hs = x_init.shape
    J = y.shape[0]
    r = p // patches
    kv = [[np.zeros((J + p, hs)), np.zeros((J + p, hs))] for _ in layers]
    x = np.array(x_init, dtype=np.float64)
    for _ in range(warmup):
        h = np.concatenate([y, x + cb])
        for lw, (kb, vb) in zip(layers, kv):
            h = _joint_or_single(lw, heads, h, kb, vb, 0, J)
        x = x - eta * h[J:]
    steady = steps - warmup
    eps = np.zeros_like(x)
    pending = np.zeros_like(x)
    for q in range(steady):
        for j in range(patches):
            rows = slice(j * r, (j + 1) * r)
            if q > 0:
                x[rows] -= eta * pending[rows]
            hi = x[rows] + cb
            h, row0 = (np.concatenate([y, hi]), 0) if j == 0 else (hi, J + j * r)
            for lw, (kb, vb) in zip(layers, kv):
                h = _joint_or_single(lw, heads, h, kb, vb, row0, J)
            eps[rows] = h[-r:]
        pending = eps.copy()
    if steady > 0:
        x = x - eta * pending
    return x
