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
