"""The MMDiT spec oracle (oracle/mmdit_oracle.py) on CPU: its counter-based
parameter stream, QK-norm / RoPE invariants and the PipeFusion properties
the reference guarantees for every block (W = S is serial; M = 1 is
staleness-free; the text rows reach the image rows)."""
import math

import numpy as np

from oracle import mmdit_oracle as mo


def _splitmix_py(x):
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def test_uniform_stream_matches_scalar_definition():
    seed, tid = 12345, mo.tid_of(3, 1, mo.P_WMOD)
    u = mo.uniform(seed, tid, 7)
    key = _splitmix_py((seed + tid * 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
    for i in range(7):
        z = _splitmix_py(key ^ ((i * 0xD1B54A32D192ED03) & ((1 << 64) - 1)))
        assert u[i] == (z >> 11) * 2.0 ** -52 - 1.0
    big = mo.uniform(0, 1, 200000)
    assert big.min() >= -1.0 and big.max() < 1.0 and abs(big.mean()) < 0.01


def test_rope_is_a_rotation_and_identity_at_position_zero():
    dh, heads, n = 32, 3, 5
    x = np.random.default_rng(0).standard_normal((n, heads, dh))
    pos = np.zeros((n, 3))
    assert np.allclose(mo.rope(x, pos, dh), x)
    pos[:, 1] = np.arange(n)
    pos[:, 2] = 7
    y = mo.rope(x, pos, dh)
    assert np.allclose(np.linalg.norm(y, axis=2), np.linalg.norm(x, axis=2))
    assert not np.allclose(y, x)
    assert sum(mo.rope_axes(128)) == 128 and mo.rope_axes(128) == (16, 56, 56)


def test_qk_norm_unit_rms_times_gain():
    m = mo.MMDiT(1, 1, 64, 2, 256, 4, 16, 1)
    x = np.random.default_rng(1).standard_normal((6, 64)) * 3
    g = np.full(32, 2.0)
    y = m.qk_post(x, g, m.pos[:6]).reshape(6, 2, 32)
    rms = np.sqrt((y * y).mean(axis=2))
    assert np.allclose(rms, 2.0, rtol=1e-5)


def test_pipefusion_properties():
    m = mo.MMDiT(2, 3, 64, 2, 256, 8, 64, 2, rope=True)
    x0 = np.random.default_rng(2).uniform(-1, 1, (64, 64))
    serial = mo.serial(m, x0, 3, 0.1)
    assert np.array_equal(mo.pipefusion(m, x0, 3, 4, 3, 0.1), serial)   # W = S
    assert np.allclose(mo.pipefusion(m, x0, 3, 1, 1, 0.1), serial)      # M = 1
    pf4 = mo.pipefusion(m, x0, 3, 4, 1, 0.1)
    div = np.linalg.norm(pf4 - serial) / np.linalg.norm(serial)
    assert 0 < div < 0.1 and math.isfinite(div)
    m.y = m.y * 0.5
    assert not np.allclose(mo.pipefusion(m, x0, 3, 4, 1, 0.1), pf4)     # text reaches x
