"""SD3-style joint-attention block on the GPU.

No reference semantics exist for it (the reference's only block is the toy
block, toy_model.cpp:145-177); the checker is the numpy restatement
oracle/np_oracle.py joint_* of the same spec (toy arithmetic per stream, text
rows first in the joint K/V buffer, re-entering with patch 0 each step),
with parameters regenerated from the same mt19937_64 stream
(oracle/loader.py joint_model). Staleness accounting is the toy executor's.
"""
import numpy as np
import pytest

from oracle import loader
from oracle import np_oracle as npo
from paper_2405_14430_b200 import JointDiTCuda, make_initial_latent

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


@pytest.mark.parametrize("N,M,W,S", [(1, 1, 1, 3), (2, 2, 1, 4), (2, 4, 0, 3), (4, 2, 2, 4)])
def test_joint_pipefusion_matches_numpy(N, M, W, S):
    seed, L, hs, heads, p, T = 1, 4, 64, 4, 256, 40
    layers, cb, y = loader.joint_model(seed, L, hs, 4 * hs, T)
    x0 = make_initial_latent(2, p, hs)
    ref = npo.joint_pipefusion(layers, cb, y, heads, x0, S, M, W, 0.1)
    toy = loader.Restatement().build_toy_model(0, L, hs, heads)
    _, (fresh, stale, _) = toy.run_pipefusion(x0, S, N, M, W, 0.1)
    with JointDiTCuda(seed, L, hs, heads, 4.0, p, T, N) as m:
        res = m.run_pipefusion(x0, S, M, W, 0.1)
    assert (res.stats.fresh_patch_reads, res.stats.stale_patch_reads) == (fresh, stale)
    assert rel(res.final_x, ref) <= TOL, rel(res.final_x, ref)


def test_joint_stage_invariance_rerun_and_text():
    seed, L, hs, heads, p, T = 3, 4, 64, 4, 256, 24
    x0 = make_initial_latent(4, p, hs)
    outs = []
    for n in (1, 2, 4):
        with JointDiTCuda(seed, L, hs, heads, 4.0, p, T, n) as m:
            a = m.run_pipefusion(x0, 3, 2, 1, 0.1).final_x
            assert np.array_equal(a, m.run_pipefusion(x0, 3, 2, 1, 0.1).final_x)
            outs.append(a)
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    layers, cb, _ = loader.joint_model(seed, L, hs, 4 * hs, T)
    y2 = np.random.default_rng(0).uniform(-1, 1, (T, hs))
    ref = npo.joint_pipefusion(layers, cb, y2, heads, x0, 3, 2, 1, 0.1)
    with JointDiTCuda(seed, L, hs, heads, 4.0, p, T, 1) as m:
        m.set_text(y2)
        got = m.run_pipefusion(x0, 3, 2, 1, 0.1).final_x
    assert rel(got, ref) <= TOL
    assert rel(outs[0], ref) > 3 * rel(got, ref)  # the text reaches the image rows


@pytest.mark.parametrize("D,N,M,W", [(2, 1, 2, 1), (1, 2, 2, 1), (0, 2, 4, 0)])
def test_flux_style_single_stream_layers(D, N, M, W):
    # Flux.1 layout: D double-stream layers, then single-stream parallel blocks
    seed, L, hs, heads, p, T, S = 5, 4, 64, 4, 256, 16, 3
    layers, cb, y = loader.joint_model(seed, L, hs, 4 * hs, T, double_layers=D)
    x0 = make_initial_latent(6, p, hs)
    ref = npo.joint_pipefusion(layers, cb, y, heads, x0, S, M, W, 0.1)
    with JointDiTCuda(seed, L, hs, heads, 4.0, p, T, N, double_layers=D) as m:
        res = m.run_pipefusion(x0, S, M, W, 0.1)
    assert rel(res.final_x, ref) <= TOL, rel(res.final_x, ref)
