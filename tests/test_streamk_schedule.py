"""Invariants of the stream-K walk of the CTA-pair residual GEMM (CPU).

The kernel (`SkWalk` / `ResidTiles` in csrc/gemm_sm100.cuh) gives pair c the
(tile, K block) units [c U / P, (c + 1) U / P) and walks them in reverse; the
dispatcher (kernels.cu) only picks it when tiles >= pairs and K blocks >= 36.
This restates the walk and checks what the kernel relies on: every unit is
computed exactly once; a tile is cut between at most two consecutive pairs;
the head piece of a cut tile is the LAST segment of pair c - 1 (so it is the
first one that pair walks, published before anything else) and its tail is
the FIRST segment of pair c (walked last, after the wait on c - 1's flag);
and each pair publishes at most one head partial (one workspace slot per CTA).
"""
import pytest


def walk(units_total, pairs, c, kblocks):
    u0 = units_total * c // pairs
    u = units_total * (c + 1) // pairs
    segs = []
    while u > u0:
        tile = (u - 1) // kblocks
        ts = tile * kblocks
        s = max(ts, u0)
        segs.append((tile, s - ts, u - ts))
        u = s
    return segs  # in walk order (reverse of the unit order)


@pytest.mark.parametrize("rows,N,K,pairs", [
    (4096, 1152, 4608, 74),    # C2 MLP-out (M = 1)
    (16384, 1152, 4608, 74),   # C3 MLP-out
    (4096, 1536, 6144, 74),    # SD3-medium MLP-out
    (16384 + 512, 3072, 12288, 74),  # Flux MLP-out rows rounded to pair tiles below
    (2048 * 9, 1152, 4608, 74),
])
def test_stream_k_walk_invariants(rows, N, K, pairs):
    rows -= rows % 256
    tiles = (rows // 256) * (N // 192)
    kblocks = (K + 63) // 64
    if not (kblocks >= 36 and tiles >= pairs):
        pytest.skip("dispatcher would not pick stream-K")
    U = tiles * kblocks
    covered = {}
    pieces = {}
    for c in range(pairs):
        segs = walk(U, pairs, c, kblocks)
        heads = [s for s in segs if s[2] < kblocks]
        assert len(heads) <= 1                      # one partial slot per CTA
        if heads:
            assert segs[0] == heads[0]              # published first
        tails = [s for s in segs if s[1] > 0]
        assert len(tails) <= 1
        if tails:
            assert segs[-1] == tails[0]             # finished last
        for tile, k0, k1 in segs:
            assert not (k0 > 0 and k1 < kblocks)    # no middle pieces
            pieces.setdefault(tile, []).append((c, k0, k1))
            for kb in range(k0, k1):
                assert (tile, kb) not in covered
                covered[(tile, kb)] = c
    assert len(covered) == U                        # every unit exactly once
    for tile, ps in pieces.items():
        assert len(ps) <= 2
        if len(ps) == 2:
            (c_tail, k0t, _), (c_head, _, k1h) = sorted(ps, key=lambda p: -p[1])
            assert c_head == c_tail - 1             # the flag the finisher waits on
            assert k1h == k0t                       # the pieces meet


def test_uniform_work_per_pair():
    U, pairs, kb = 96 * 72, 74, 72
    sizes = [sum(k1 - k0 for _, k0, k1 in walk(U, pairs, c, kb)) for c in range(pairs)]
    assert max(sizes) - min(sizes) <= 1
