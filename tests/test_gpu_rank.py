"""Rank mode (one context / process per stage) on the GPU.

Each rank owns one stage; boundary messages go straight into the receiver's
landing buffers over peer memory (same-process: UVA pointers; other
processes: CUDA IPC) with stream-ordered signal/ack counters
(pf_rank_plan). On the single GPU of the test box every rank lives on
device 0. The result must equal the single-context executor with the same
number of stages bit for bit (the reference's threads == inline property,
test_execute.cpp:151-164), and the summed staleness stats must match.
"""
import multiprocessing as mp
import socket

import numpy as np
import pytest

import paper_2405_14430_b200 as pf
from oracle import loader

pytestmark = pytest.mark.gpu


def _single(seed, L, hs, heads, p, N, S, M, W, x0, text=0):
    if text:
        m = pf.PixArtCuda(seed, L, hs, heads, 4.0, p, text, N)
    else:
        m = pf.ToyDiTCuda(seed, L, hs, heads, 4.0, p, N)
    with m:
        res = m.run_pipefusion(x0, S, M, W, 0.1)
    return res


def _same_process_ranks(seed, L, hs, heads, p, N, S, M, W, x0, text=0, runs=1, joint=None):
    import torch
    if joint is not None:
        ranks = [pf.JointDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, text, r, N, 0,
                                            double_layers=joint) for r in range(N)]
    elif text:
        ranks = [pf.PixArtCuda.rank_stage(seed, L, hs, heads, 4.0, p, text, r, N, 0)
                 for r in range(N)]
    else:
        ranks = [pf.ToyDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, r, N, 0) for r in range(N)]
    pf.connect_ranks(ranks)
    outs, stats = [], []
    # one caller stream per rank: a shared caller stream would chain the ranks'
    # joins and forks (rank 1 would wait for rank 0, which waits for rank 1)
    streams = [torch.cuda.Stream() for _ in ranks]
    for _ in range(runs):
        x = torch.from_numpy(x0.astype(np.float32)).cuda()
        torch.cuda.synchronize()
        st = []
        # enqueue every rank before waiting on any: the ranks depend on each other
        for r, m in enumerate(ranks):
            st.append(m.run_pipefusion_device(x.data_ptr() if r == 0 else 0, S, M, W, 0.1,
                                              streams[r].cuda_stream))
        for r, m in enumerate(ranks):
            m.synchronize(streams[r].cuda_stream)
        outs.append(x.double().cpu().numpy())
        stats.append((sum(s.fresh_patch_reads for s in st), sum(s.stale_patch_reads for s in st)))
    for m in ranks:
        m.close()
    return outs, stats


@pytest.mark.parametrize("N,S,M,W", [(2, 4, 4, 1), (3, 5, 2, 2), (4, 3, 4, 0), (2, 3, 1, 3)])
def test_same_process_ranks_equal_single_context(N, S, M, W):
    seed, L, hs, heads, p = 0, 4, 128, 4, 256
    x0 = pf.make_initial_latent(0, p, hs)
    ref = _single(seed, L, hs, heads, p, N, S, M, W, x0)
    outs, stats = _same_process_ranks(seed, L, hs, heads, p, N, S, M, W, x0, runs=2)
    for o in outs:  # second run: signal counters continue from the first
        assert np.array_equal(o, ref.final_x)
    assert stats[0] == (ref.stats.fresh_patch_reads, ref.stats.stale_patch_reads)


def test_same_process_ranks_pixart():
    seed, L, hs, heads, p, T = 3, 4, 64, 4, 128, 8
    x0 = pf.make_initial_latent(7, p, hs)
    ref = _single(seed, L, hs, heads, p, 2, 5, 4, 1, x0, text=T)
    outs, _ = _same_process_ranks(seed, L, hs, heads, p, 2, 5, 4, 1, x0, text=T)
    assert np.array_equal(outs[0], ref.final_x)
    o = loader.PixArtOracle(seed, L, hs, heads, 4.0, T)
    ora, _ = o.run_pipefusion(x0, 5, 2, 4, 1, 0.1)
    assert np.linalg.norm(outs[0] - ora) / np.linalg.norm(ora) <= 1e-2


# ----------------------------------------------------------------- one process per rank
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _proc_rank(rank, world, port, cfg, q):
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        seed, L, hs, heads, p, S, M, W = cfg
        m = pf.ToyDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, rank, world, 0)
        pf.connect_distributed(m)
        x0 = pf.make_initial_latent(0, p, hs)
        res = m.run_pipefusion(x0 if rank == 0 else None, S, M, W, 0.1)
        dist.barrier()
        m.close()
        q.put((rank, res.final_x, res.stats.fresh_patch_reads, res.stats.stale_patch_reads))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e), 0, 0))


def test_process_per_rank_over_cuda_ipc():
    seed, L, hs, heads, p, S, M, W = 0, 4, 128, 4, 256, 4, 4, 1
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cfg = (seed, L, hs, heads, p, S, M, W)
    procs = [ctx.Process(target=_proc_rank, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(world):
        r, x, fr, st = q.get(timeout=300)
        got[r] = (x, fr, st)
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert not isinstance(got[r][0], str), got[r][0]
    x0 = pf.make_initial_latent(0, p, hs)
    ref = _single(seed, L, hs, heads, p, world, S, M, W, x0)
    assert np.array_equal(got[0][0], ref.final_x)
    assert (sum(v[1] for v in got.values()), sum(v[2] for v in got.values())) == \
        (ref.stats.fresh_patch_reads, ref.stats.stale_patch_reads)


@pytest.mark.parametrize("D,N", [(4, 2), (2, 3)])
def test_same_process_ranks_joint(D, N):
    # SD3 / Flux-style joint rows: text rows travel with patch 0 between ranks
    seed, L, hs, heads, p, T = 2, 4, 64, 4, 256, 24
    x0 = pf.make_initial_latent(3, p, hs)
    with pf.JointDiTCuda(seed, L, hs, heads, 4.0, p, T, N, double_layers=D) as m:
        ref = m.run_pipefusion(x0, 4, 2, 1, 0.1)
    outs, stats = _same_process_ranks(seed, L, hs, heads, p, N, 4, 2, 1, x0, text=T, joint=D)
    assert np.array_equal(outs[0], ref.final_x)
    assert stats[0] == (ref.stats.fresh_patch_reads, ref.stats.stale_patch_reads)
