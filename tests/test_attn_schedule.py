"""Stream-K attention schedule invariants, on the CPU (host code of the
library, no GPU): every (item, KV block) unit is owned by exactly one CTA;
in-kernel merging (fused) is chosen only when every cut item meets exactly two
CTAs as one head segment and one tail segment (what the kernel's flag protocol
handles); otherwise cut items meet at most kAttnMaxParts = 8 CTAs (the merge
kernel's bound) and CTAs hold at most kAttnMaxSegs = 64 segments; schedules of
C2 shapes are the documented ones (full sequence: stream-K over 148 SMs with
in-kernel merge; patches: one CTA per item; a small full sequence: two CTAs
per item).
"""
import ctypes

import pytest

import paper_2405_14430_b200 as pf


def schedule(P, rows, heads, dhp, sms=148, with_strided=False):
    out = (ctypes.c_longlong * 7)()
    assert pf.load_library().pf_debug_attn_schedule(P, rows, heads, dhp, sms, out) == 0
    nq, blocks, units, grid, cut, fused, strided = list(out)
    res = (nq, blocks, units, grid, bool(cut), bool(fused))
    return res + (bool(strided),) if with_strided else res


def segments(units, grid, B, strided=False):
    """Segments of each CTA in natural order: (item, b0, n)."""
    if strided:  # whole items c, c + grid, ... (the kernel's segment table)
        return [[(x, 0, B) for x in range(c, units // B, grid)] for c in range(grid)]
    out = []
    for c in range(grid):
        u, u1, segs = c * units // grid, (c + 1) * units // grid, []
        while u < u1:
            x, b0 = divmod(u, B)
            n = min(u1 - u, B - b0)
            segs.append((x, b0, n))
            u += n
        out.append(segs)
    return out


SHAPES = [(P, rows, heads, dhp, sms)
          for P, heads, dhp in [(4096, 16, 80), (16384, 16, 80), (4429, 24, 64), (520, 2, 128),
                                (120, 16, 80), (256, 4, 32), (16896, 24, 128)]
          for rows in sorted({P, P // 2, P // 4, P // 8, 512, 136, 128})
          if 0 < rows <= P
          for sms in (148, 132)]


@pytest.mark.parametrize("P,rows,heads,dhp,sms", SHAPES)
def test_schedule_invariants(P, rows, heads, dhp, sms):
    nq, B, units, grid, cut, fused, strided = schedule(P, rows, heads, dhp, sms, True)
    assert nq == (rows + 255) // 256 and B == (P + 127) // 128 and units == nq * heads * B
    assert 1 <= grid
    if strided:  # K/V beyond the L2: whole items, no cuts, at least four per CTA
        assert not cut and not fused and 4 * heads * P * dhp > 96e6
        assert nq * heads >= 4 * sms
    segs = segments(units, grid, B, strided)
    owned = {}
    for c, ss in enumerate(segs):
        assert len(ss) <= 64
        for x, b0, n in ss:
            for b in range(b0, b0 + n):
                assert (x, b) not in owned
                owned[(x, b)] = c
    assert len(owned) == units
    parts = {}
    for c, ss in enumerate(segs):
        for x, b0, n in ss:
            if n < B:
                parts.setdefault(x, []).append((c, b0, n))
    if not cut:  # "cut" may be conservative, never optimistic
        assert not parts
    if fused:
        for x, ps in parts.items():
            assert len(ps) == 2, (x, ps)
            (c0, h0, hn), (c1, t0, tn) = sorted(ps)
            assert c1 == c0 + 1 and h0 == 0 and t0 == hn and t0 + tn == B
            assert segs[c0][-1][0] == x and segs[c1][0][0] == x  # head last, tail first
    else:
        for ps in parts.values():
            assert len(ps) <= 8


def test_c2_schedules():
    assert schedule(4096, 4096, 16, 80)[3:] == (148, True, True)   # stream-K, merged in-kernel
    assert schedule(4096, 512, 16, 80)[3:] == (32, False, False)    # one CTA per item
    assert schedule(1024, 1024, 8, 64)[3:] == (64, True, True)     # full sequence, two CTAs per item
    assert schedule(4096, 2048, 16, 80)[3:] == (128, False, False)  # one CTA per item


def test_flux_full_sequence_is_strided():
    # Flux 2048 px, dh 128: 24 heads x 16896 KV rows exceed the L2
    assert schedule(16896, 16896, 24, 128, with_strided=True)[3:] == (148, False, False, True)
    # C3 (16 heads x 16384 x dh 80, 84 MB of K/V) keeps stream-K
    assert schedule(16384, 16384, 16, 80, with_strided=True)[6] is False

