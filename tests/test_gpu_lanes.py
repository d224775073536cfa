"""Multi-lane patch schedule (one stage, M >= 2) on the GPU.

Patch j runs on lane j % lanes with QKV(j, l) ordered after ATTN(j-1, l) (the
K/V-buffer hazard); every other buffer a patch touches is its own rows or its
lane's scratch. The result must equal the one-lane schedule (PF_LANES=1)
bit for bit, with and without CUDA graphs, and reruns must be bitwise stable.
"""
import numpy as np
import pytest

import paper_2405_14430_b200 as pf

pytestmark = pytest.mark.gpu


def _run(monkeypatch, lanes, L, hs, heads, p, S, M, W, graphs, reps=1, text=0, joint=None):
    monkeypatch.delenv("PF_ONE_LANE", raising=False)
    monkeypatch.setenv("PF_LANES", str(lanes))
    x0 = pf.make_initial_latent(1, p, hs)
    if joint is not None:
        model = pf.JointDiTCuda(0, L, hs, heads, 4.0, p, text, 1, double_layers=joint)
    elif text:
        model = pf.PixArtCuda(0, L, hs, heads, 4.0, p, text, 1)
    else:
        model = pf.ToyDiTCuda(0, L, hs, heads, 4.0, p, 1)
    with model as m:
        m.set_graphs(graphs)
        outs = [m.run_pipefusion(x0, S, M, W, 0.1) for _ in range(reps)]
    return outs


@pytest.mark.parametrize("L,hs,heads,p,S,M,W", [
    (4, 128, 4, 512, 5, 4, 1),
    (3, 128, 4, 768, 4, 3, 1),      # odd M: patch M-1 and patch 0 share a lane
    (2, 64, 4, 256, 3, 2, 0),       # no warmup: lanes from the first step
    (2, 1152, 16, 4096, 3, 8, 1),   # C2 patch shape: split-K GEMMs + stream-K combine on both lanes
])
@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("lanes", [2, 3, 4])
def test_lanes_equal_one_lane(monkeypatch, L, hs, heads, p, S, M, W, graphs, lanes):
    one = _run(monkeypatch, 1, L, hs, heads, p, S, M, W, graphs)[0]
    two = _run(monkeypatch, lanes, L, hs, heads, p, S, M, W, graphs, reps=2)
    for r in two:
        assert np.array_equal(r.final_x, one.final_x)
        assert (r.stats.fresh_patch_reads, r.stats.stale_patch_reads) == \
            (one.stats.fresh_patch_reads, one.stats.stale_patch_reads)
        assert r.stats.per_worker_fresh_fraction == one.stats.per_worker_fresh_fraction


@pytest.mark.parametrize("L,hs,heads,p,T,S,M,W", [
    (3, 128, 4, 512, 8, 4, 4, 1),
    (2, 1152, 16, 4096, 120, 3, 8, 1),  # PixArt-alpha patch shape
])
def test_lanes_pixart_equal_one_lane(monkeypatch, L, hs, heads, p, T, S, M, W):
    one = _run(monkeypatch, 1, L, hs, heads, p, S, M, W, True, text=T)[0]
    four = _run(monkeypatch, 4, L, hs, heads, p, S, M, W, True, reps=2, text=T)
    for r in four:
        assert np.array_equal(r.final_x, one.final_x)


@pytest.mark.parametrize("L,D,hs,heads,p,T,S,M", [
    (4, 2, 128, 4, 512, 24, 4, 4),     # double + single stream layers, text rows with patch 0
    (3, 3, 1536, 24, 4096, 333, 3, 8),  # SD3-medium-shaped joint blocks
])
def test_lanes_joint_equal_one_lane(monkeypatch, L, D, hs, heads, p, T, S, M):
    one = _run(monkeypatch, 1, L, hs, heads, p, S, M, 1, True, text=T, joint=D)[0]
    four = _run(monkeypatch, 4, L, hs, heads, p, S, M, 1, True, reps=2, text=T, joint=D)
    for r in four:
        assert np.array_equal(r.final_x, one.final_x)


@pytest.mark.parametrize("workers,L,S,W", [(4, 2, 4, 1), (2, 3, 3, 0)])
def test_distrifusion_lanes_equal_one_lane(monkeypatch, workers, L, S, W):
    x0 = pf.make_initial_latent(2, 4096, 1152)
    res = []
    for lanes in (1, 4):
        monkeypatch.setenv("PF_LANES", str(lanes))
        with pf.ToyDiTCuda(0, L, 1152, 16, 4.0, 4096, 1) as m:
            res.append([m.run_distrifusion(x0, S, workers, W, 0.1) for _ in range(2)])
    for r in res[1]:
        assert np.array_equal(r.final_x, res[0][0].final_x)
        assert r.stats.per_worker_fresh_fraction == res[0][0].stats.per_worker_fresh_fraction
