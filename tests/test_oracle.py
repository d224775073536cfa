"""The CPU oracle is pinned before it is trusted (CPU-only, no GPU).

1. The reference's own doctest suites pass against oracle/_ref (the reference
   sources compiled here with the Eigen/doctest shims) -- this pins the shim
   build to the reference's goldens (test_execute.cpp:166-174, 259-275).
2. The plain-C restatement (oracle/pf_oracle.c) is bitwise equal to the
   reference on weights, latents, serial and PipeFusion runs, staleness stats,
   the schedule grid and the freshness series.
3. Both reproduce the committed golden fixtures (tests/golden/, generated from
   the reference by tests/golden/make_golden.py) and the SURVEY's pinned values.
"""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import loader

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


@pytest.fixture(scope="module")
def rs():
    if not loader.RESTATEMENT_LIB.exists():
        loader.build(reference=False)
    return loader.Restatement()


@pytest.fixture(scope="module")
def ref():
    if not loader.REFERENCE_LIB.exists():
        if not loader.REFERENCE_SRC.exists():
            pytest.skip("reference sources and oracle/_ref both absent")
        loader.build(reference=True)
    return loader.Reference()


# ---------------------------------------------------------------- 1. reference suites
@pytest.mark.parametrize("suite", ["test_execute", "test_schedule", "test_freshness"])
def test_reference_own_suites_pass(suite, ref):
    exe = ROOT / "oracle" / "_ref" / suite
    if not exe.exists():
        pytest.skip(f"{exe} not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


# ---------------------------------------------------------------- 2. restatement == reference
def test_weights_and_latent_bitwise(rs, ref):
    for seed, L, hs, heads, ratio in [(0, 4, 32, 4, 4.0), (7, 2, 16, 2, 2.0), (1, 3, 24, 3, 2.5)]:
        a, ca = rs.build_toy_model(seed, L, hs, heads, ratio).weights()
        b, cb = ref.build_toy_model(seed, L, hs, heads, ratio).weights()
        for la, lb in zip(a, b):
            for wa, wb in zip(la, lb):
                assert np.array_equal(wa, wb)
        assert np.array_equal(ca, cb)
        assert np.array_equal(rs.make_initial_latent(seed, 40, hs),
                              ref.make_initial_latent(seed, 40, hs))


def test_weights_bounded_and_seeded(rs):
    # test_execute.cpp:45-62
    a, _ = rs.build_toy_model(0, 4, 32, 4).weights()
    b, _ = rs.build_toy_model(1, 4, 32, 4).weights()
    assert not np.array_equal(a[0][0], b[0][0])
    assert np.abs(a[0][0]).max() <= 1 / np.sqrt(32) + 1e-12
    with pytest.raises(loader.OracleError):
        rs.build_toy_model(0, 4, 30, 4)
    with pytest.raises(loader.OracleError):
        rs.build_toy_model(0, 0, 32, 4)


@pytest.mark.parametrize("L,hs,heads,p,S,N,M,W", [
    (4, 32, 4, 64, 20, 4, 4, 1),    # reference_execute.cfg
    (4, 16, 4, 32, 6, 4, 4, 0),
    (4, 16, 4, 32, 6, 2, 8, 3),
    (4, 16, 2, 32, 5, 1, 1, 0),
    (8, 16, 4, 32, 6, 8, 2, 1),     # M < N
    (4, 16, 4, 32, 6, 4, 4, 6),     # W = S
])
def test_pipefusion_bitwise_vs_reference(rs, ref, L, hs, heads, p, S, N, M, W):
    ma = rs.build_toy_model(3, L, hs, heads)
    mb = ref.build_toy_model(3, L, hs, heads)
    x0 = rs.make_initial_latent(3, p, hs)
    xa, sa = ma.run_pipefusion(x0, S, N, M, W, 0.1)
    for backend in ("threads", "inline"):
        xb, sb = mb.run_pipefusion(x0, S, N, M, W, 0.1, backend=backend)
        assert np.array_equal(xa, xb)
        assert sa[0] == sb[0] and sa[1] == sb[1]
        assert sa[2] == sb[2]
    assert np.array_equal(ma.serial_reference(x0, S, 0.1), mb.serial_reference(x0, S, 0.1))


def test_layer_forward_bitwise(rs, ref):
    ma = rs.build_toy_model(5, 2, 32, 4)
    mb = ref.build_toy_model(5, 2, 32, 4)
    rng = np.random.default_rng(0)
    h = rng.uniform(-1, 1, (16, 32))
    k = rng.uniform(-1, 1, (64, 32))
    v = rng.uniform(-1, 1, (64, 32))
    for a, b in zip(ma.layer_forward(1, h, k, v, 32), mb.layer_forward(1, h, k, v, 32)):
        assert np.array_equal(a, b)


def test_validation_messages(rs, ref):
    # test_execute.cpp:277-287
    for impl in (rs, ref):
        m = impl.build_toy_model(0, 4, 16, 4)
        x0 = impl.make_initial_latent(0, 32, 16)
        with pytest.raises(loader.OracleError, match="divisible") as e:
            m.run_pipefusion(x0, 4, 3, 4, 0, 0.1)
        assert e.value.code == 2
        with pytest.raises(loader.OracleError, match="divisible"):
            m.run_pipefusion(x0, 4, 4, 5, 0, 0.1)
        with pytest.raises(loader.OracleError):
            m.run_pipefusion(x0, 4, 4, 4, 5, 0.1)


def test_non_finite_is_numeric_error(rs, ref):
    # a huge step size drives the latent to inf (test_cli.cpp:176-187)
    for impl in (rs, ref):
        m = impl.build_toy_model(0, 2, 16, 4)
        x0 = impl.make_initial_latent(0, 32, 16) * 1e300
        with pytest.raises(loader.OracleError, match="non-finite activation") as e:
            m.run_pipefusion(x0, 3, 2, 2, 0, 1e300)
        assert e.value.code == 1


@pytest.mark.parametrize("n,m,S,W", [(2, 2, 1, 0), (4, 4, 2, 0), (4, 2, 5, 1), (3, 7, 4, 2),
                                     (8, 8, 20, 1), (1, 1, 1, 0), (8, 2, 3, 3)])
def test_schedule_and_freshness_bitwise(rs, ref, n, m, S, W):
    a = rs.schedule(n, m, S, W)
    b = ref.schedule(n, m, S, W)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    assert a[3:] == b[3:]
    assert np.array_equal(rs.fresh_series(n, m, S, W), ref.fresh_series(n, m, S, W))


def test_schedule_slot_five_pattern(rs):
    # test_schedule.cpp:70-80 (Fig. 5)
    pa, ts, kd, ws, ss = rs.schedule(4, 4, 2, 0)
    assert [pa[5, d] for d in range(4)] == [1, 0, 3, 2]
    assert [ts[5, d] for d in range(4)] == [0, 0, 1, 1]


def test_auto_warmup(rs, ref):
    # test_execute.cpp:259-275
    for impl in (rs, ref):
        m = impl.build_toy_model(0, 4, 32, 4)
        x0 = impl.make_initial_latent(0, 64, 32)
        assert m.auto_warmup(x0, 20, 0.1, float("inf")) == (1, True)
        assert m.auto_warmup(x0, 20, 0.1, 0.0) == (20, False)
        assert m.auto_warmup(x0, 20, 0.1, 0.05) == (16, True)


# ---------------------------------------------------------------- 3. goldens
def _golden(name):
    return np.load(GOLDEN / f"{name}.npz")


def test_pinned_reference_divergence(rs):
    # test_execute.cpp:166-174: 0.024653651895269472 within 1e-6 relative
    m = rs.build_toy_model(0, 4, 32, 4)
    x0 = rs.make_initial_latent(0, 64, 32)
    pf, (fresh, stale, _) = m.run_pipefusion(x0, 20, 4, 4, 1, 0.1)
    div = rs.divergence(pf, m.serial_reference(x0, 20, 0.1))
    assert abs(div - 0.024653651895269472) <= 1e-6 * 0.024653651895269472
    assert (fresh, stale) == (776, 456)
    assert np.allclose(pf[0, :4], [0.40742689823440731, 0.33996202226467537,
                                   -1.1638292549974716, 0.75575538809186815], rtol=0, atol=1e-15)


@pytest.mark.parametrize("name", ["cref", "c1_s4", "c1_s5"])
def test_restatement_reproduces_golden_fixtures(rs, name):
    g = _golden(name)
    c = eval(str(g["config"]))
    m = rs.build_toy_model(c["seed"], c["L"], c["hs"], c["heads"])
    x0 = rs.make_initial_latent(c["seed"], c["p"], c["hs"])
    pf, (fresh, stale, ff) = m.run_pipefusion(x0, c["S"], c["N"], c["M"], c["W"], c["eta"])
    assert np.array_equal(pf, g["x_pipefusion"])
    assert (fresh, stale) == (int(g["fresh"]), int(g["stale"]))
    assert np.array_equal(np.asarray(ff), g["fresh_fraction"])
    if name != "cref":  # the C1 serial run is the slow part; cref covers it above
        return


def test_c1_survey_values():
    # SURVEY Appendix A.4 (probe of the reference): div, stats, x[0, 0..2]
    s4, s5 = _golden("c1_s4"), _golden("c1_s5")
    assert float(s4["divergence"]) == pytest.approx(0.037251379083572053, rel=1e-12)
    assert float(s5["divergence"]) == pytest.approx(0.040509167401966403, rel=1e-12)
    assert (int(s4["fresh"]), int(s4["stale"])) == (136, 72)
    assert (int(s5["fresh"]), int(s5["stale"])) == (176, 96)
    assert np.allclose(s4["x_pipefusion"][0, :3],
                       [0.32449335502956572, 0.24827867908782209, -0.39906740005157071],
                       rtol=0, atol=1e-15)
    assert float(s4["x_pipefusion"].sum()) == pytest.approx(271.39910203039642, rel=1e-12)


# ------------------------------------------------------ 4. numpy restatement pinned
def test_np_oracle_layer_forward_matches_reference(ref):
    """oracle/np_oracle.layer_forward (the vectorised fp64 checker the C2 / C3
    layer-unit GPU tests use at widths where the scalar restatement is too
    slow) against the reference's own toy_layer_forward (oracle/_ref) at
    hs=128: equal up to summation order."""
    from oracle import np_oracle
    hs, heads, p, rows, row0 = 128, 4, 256, 64, 64
    m = ref.build_toy_model(3, 2, hs, heads, 4.0)
    weights, _ = m.weights()
    rng = np.random.default_rng(11)
    h = rng.uniform(-1, 1, (rows, hs))
    k = rng.uniform(-1, 1, (p, hs))
    v = rng.uniform(-1, 1, (p, hs))
    for layer in range(2):
        rh, rk, rv = m.layer_forward(layer, h, k, v, row0)
        nk, nv = k.copy(), v.copy()
        nh = np_oracle.layer_forward(weights[layer], heads, h.copy(), nk, nv, row0)
        assert np.abs(nh - rh).max() <= 1e-12 * np.abs(rh).max()
        assert np.abs(nk - rk).max() <= 1e-12 and np.abs(nv - rv).max() <= 1e-12


@pytest.mark.parametrize("name", ["c2s_s1_w0", "c2s_s2_w1", "c2s_s4_w1"])
def test_c2_short_horizon_fixture_stats(rs, name):
    """The C2-shape fixtures (tests/golden/make_golden_c2.py) carry the
    staleness stats of their (p, M, S, W): they do not depend on the model's
    width or depth per layer, so a small model of the same depth reproduces
    them exactly; the latent is finite and of the C2 shape."""
    g = np.load(GOLDEN / f"{name}.npz")
    c = eval(str(g["config"]))  # noqa: S307 - our own fixture
    assert g["x_pipefusion"].shape == (c["p"], c["hs"])
    assert np.isfinite(g["x_pipefusion"]).all()
    m = rs.build_toy_model(0, c["L"], 8, 2)
    x0 = rs.make_initial_latent(0, c["p"], 8)
    _, (fresh, stale, ff) = m.run_pipefusion(x0, c["S"], 1, c["M"], c["W"], c["eta"])
    assert (fresh, stale) == (int(g["fresh"]), int(g["stale"]))
    assert np.array_equal(np.asarray(ff), g["fresh_fraction"])
