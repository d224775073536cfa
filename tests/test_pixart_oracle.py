"""The fp64 PixArt-alpha block oracle (oracle/px_oracle.c) before it is
trusted as the GPU checker (CPU only).

The reference has no PixArt block (its only block is toy_model.cpp:145-177),
so this oracle is "parity unpinned" against the reference itself; it is
pinned instead (i) against an independent numpy restatement of the same
spec (oracle/np_oracle.py px_*), (ii) on the reference's own loop semantics:
W = S reproduces serial_reference bit for bit (test_execute.cpp:99-113),
staleness counts equal the toy block's for the same (N, M, W, S), and
(iii) its tvec/LayerNorm pieces against closed forms.
"""
import numpy as np
import pytest

from oracle import loader
from oracle import np_oracle as npo


@pytest.fixture(scope="module")
def px():
    return loader.PixArtOracle(3, 2, 64, 4, 4.0, 8)


def test_tvec_matches_numpy_restatement(px):
    g = {n: px.glob(n) for n in loader.PXO_GLOBALS}
    for t, s in [(0, 1), (3, 5), (19, 20)]:
        assert np.allclose(px.tvec(t, s), npo.px_tvec(g, t, s, 64), rtol=0, atol=1e-13)


@pytest.mark.parametrize("layer,row0,rows", [(0, 0, 32), (1, 16, 16), (1, 8, 8)])
def test_layer_matches_numpy_restatement(px, layer, row0, rows):
    rng = np.random.default_rng(layer * 100 + row0)
    g = {n: px.glob(n) for n in loader.PXO_GLOBALS}
    p = {n: px.param(layer, n) for n in loader.PXO_PARAMS}
    h = rng.uniform(-1, 1, (rows, 64))
    k = rng.uniform(-1, 1, (32, 64))
    v = rng.uniform(-1, 1, (32, 64))
    h1, k1, v1 = px.layer_forward(layer, 2, 5, h, k, v, row0)
    mod = p["sst"].reshape(-1) + npo.px_tvec(g, 2, 5, 64)
    k2, v2 = k.copy(), v.copy()
    h2 = npo.px_layer_forward(p, 4, mod, h, k2, v2, row0, g["y"])
    assert np.allclose(h1, h2, rtol=0, atol=1e-12)
    assert np.array_equal(k1, k2) or np.allclose(k1, k2, rtol=0, atol=1e-13)
    assert np.allclose(v1, v2, rtol=0, atol=1e-13)
    # only the patch's own K/V rows change (toy_model.cpp:174-175 semantics)
    mask = np.ones(32, bool)
    mask[row0:row0 + rows] = False
    assert np.array_equal(k1[mask], k[mask]) and np.array_equal(v1[mask], v[mask])


def test_full_warmup_equals_serial_bitwise(px):
    x = np.random.default_rng(1).uniform(-1, 1, (32, 64))
    a, (fresh, stale) = px.run_pipefusion(x, 4, 2, 4, 4, 0.1)
    b = px.serial_reference(x, 4, 0.1)
    assert np.array_equal(a, b)
    assert stale == 0 and fresh == 4 * 2 * 4


def test_staleness_counts_equal_toy_block(px):
    # the block does not change the schedule: counts equal the toy executor's
    x = np.random.default_rng(2).uniform(-1, 1, (32, 64))
    toy = loader.Restatement().build_toy_model(3, 2, 64, 4)
    for (n, m, w) in [(2, 4, 1), (1, 2, 0), (2, 8, 2)]:
        _, st_px = px.run_pipefusion(x, 5, n, m, w, 0.1)
        _, (fr, sl, _) = toy.run_pipefusion(x, 5, n, m, w, 0.1)
        assert st_px == (fr, sl)


def test_text_tokens_enter_through_cross_attention(px):
    rng = np.random.default_rng(4)
    o = loader.PixArtOracle(3, 2, 64, 4, 4.0, 8)
    h = rng.uniform(-1, 1, (8, 64))
    k = rng.uniform(-1, 1, (32, 64))
    v = rng.uniform(-1, 1, (32, 64))
    a, _, _ = o.layer_forward(0, 1, 4, h, k, v, 0)
    o.set_text(rng.uniform(-1, 1, (8, 64)))
    b, _, _ = o.layer_forward(0, 1, 4, h, k, v, 0)
    assert not np.allclose(a, b)


def test_numpy_pipefusion_mirror_matches_c(px):
    x = np.random.default_rng(5).uniform(-1, 1, (32, 64))
    for (m, w) in [(4, 1), (2, 0)]:
        a, _ = px.run_pipefusion(x, 4, 2, m, w, 0.1)
        b = npo.px_pipefusion(px, x, 4, m, w, 0.1)
        assert np.allclose(a, b, rtol=0, atol=1e-11)
