"""MMDiT blocks (SD3-medium / Flux.1 configurations, BASELINE configs 4 and 5)
on the GPU PipeFusion executor.

No reference semantics exist for these blocks (the reference's only block is
the toy block, toy_model.cpp:145-177); the checker is the fp64 numpy spec
oracle/mmdit_oracle.py run under the reference's inline PipeFusion loop
(execute.cpp:167-223) with the joint-row convention (text rows first,
re-entering with patch 0 of every step). Parameters come from the same
counter-based stream on both sides. Staleness accounting is the toy
executor's (the schedule does not depend on the block).
"""
import numpy as np
import pytest

import paper_2405_14430_b200 as pf
from oracle import loader
from oracle import mmdit_oracle as mo

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def _oracle(seed, L, hs, heads, p, T, D, rope):
    return mo.MMDiT(seed, L, hs, heads, 4 * hs, T, p, D, rope=rope)


@pytest.mark.parametrize("D,rope,N,M,W,S", [
    (4, False, 1, 1, 1, 3),   # SD3-style: every block double-stream, no RoPE
    (4, False, 2, 4, 1, 4),
    (4, False, 2, 2, 0, 3),   # W = 0: the first steady step reads zero K/V rows
    (2, True, 1, 2, 1, 3),    # Flux-style: 2 double + 2 single blocks, RoPE
    (2, True, 4, 4, 1, 4),
    (0, True, 2, 2, 2, 4),    # single-stream blocks only
])
def test_mmdit_pipefusion_matches_spec(D, rope, N, M, W, S):
    seed, L, hs, heads, p, T = 7, 4, 128, 4, 256, 16
    x0 = pf.make_initial_latent(3, p, hs)
    ref = mo.pipefusion(_oracle(seed, L, hs, heads, p, T, D, rope), x0, S, M, W, 0.1)
    toy = loader.Restatement().build_toy_model(0, L, 8, 2)
    _, (fresh, stale, _) = toy.run_pipefusion(pf.make_initial_latent(3, p, 8), S, N, M, W, 0.1)
    with pf.MMDiTCuda(seed, L, hs, heads, 4.0, p, T, N, double_layers=D, rope=rope) as m:
        res = m.run_pipefusion(x0, S, M, W, 0.1)
    assert (res.stats.fresh_patch_reads, res.stats.stale_patch_reads) == (fresh, stale)
    e = rel(res.final_x, ref)
    assert e <= TOL, e


def test_mmdit_stage_invariance_rerun_and_serial():
    seed, L, hs, heads, p, T, D = 11, 4, 128, 4, 256, 24, 2
    x0 = pf.make_initial_latent(5, p, hs)
    outs = []
    for n in (1, 2, 4):
        with pf.MMDiTCuda(seed, L, hs, heads, 4.0, p, T, n, double_layers=D, rope=True) as m:
            a = m.run_pipefusion(x0, 3, 2, 1, 0.1).final_x
            assert np.array_equal(a, m.run_pipefusion(x0, 3, 2, 1, 0.1).final_x)
            outs.append(a)
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    # W = S is the serial reference (execute.cpp:167-223 with no steady step)
    om = _oracle(seed, L, hs, heads, p, T, D, True)
    with pf.MMDiTCuda(seed, L, hs, heads, 4.0, p, T, 1, double_layers=D, rope=True) as m:
        got = m.serial_reference(x0, 3, 0.1)
    assert rel(got, mo.serial(om, x0, 3, 0.1)) <= TOL


def test_mmdit_rope_and_text_reach_the_output():
    seed, L, hs, heads, p, T, D = 13, 2, 128, 4, 256, 16, 1
    x0 = pf.make_initial_latent(6, p, hs)
    with pf.MMDiTCuda(seed, L, hs, heads, 4.0, p, T, 1, double_layers=D, rope=True) as m:
        a = m.run_pipefusion(x0, 2, 2, 1, 0.1).final_x
    with pf.MMDiTCuda(seed, L, hs, heads, 4.0, p, T, 1, double_layers=D, rope=False) as m:
        b = m.run_pipefusion(x0, 2, 2, 1, 0.1).final_x
    ref_b = mo.pipefusion(_oracle(seed, L, hs, heads, p, T, D, False), x0, 2, 2, 1, 0.1)
    assert rel(b, ref_b) <= TOL
    assert rel(a, b) > 10 * rel(b, ref_b)  # the rotation is not a no-op
    with pf.MMDiTCuda(seed, L, hs, heads, 4.0, p, T, 1, double_layers=D, rope=False) as m:
        y2 = np.random.default_rng(0).uniform(-1, 1, (T, hs))
        m.set_text(y2)
        c = m.run_pipefusion(x0, 2, 2, 1, 0.1).final_x
    om = _oracle(seed, L, hs, heads, p, T, D, False)
    om.y = y2
    assert rel(c, mo.pipefusion(om, x0, 2, 2, 1, 0.1)) <= TOL
    assert rel(c, b) > 10 * rel(b, ref_b)


def test_mmdit_memory_is_sharded_across_stages():
    """Layer sharding: each of N rank-mode stages holds 1/N of
    the layers' parameters and K/V buffers (plus the next stage's first
    modulation matrix)."""
    L, hs, heads, p, T, D = 8, 128, 4, 256, 16, 8  # equal layers: equal shares
    with pf.MMDiTCuda(1, L, hs, heads, 4.0, p, T, 1, double_layers=D) as m:
        full_p, full_kv = m.param_bytes(), m.kv_bytes()
    ranks = [pf.MMDiTCuda.rank_stage(1, L, hs, heads, 4.0, p, T, r, 4, 0, double_layers=D)
             for r in range(4)]
    per = [(r.param_bytes(), r.kv_bytes()) for r in ranks]
    for r in ranks:
        r.close()
    assert sum(b for b, _ in per) == full_p
    assert sum(k for _, k in per) == full_kv
    assert all(k == full_kv // 4 for _, k in per)
    assert max(b for b, _ in per) <= 0.3 * full_p
