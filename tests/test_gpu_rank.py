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


def _same_process_ranks(seed, L, hs, heads, p, N, S, M, W, x0, text=0, runs=1, joint=None,
                        mmdit=None, precision=0):
    import torch
    if mmdit is not None:
        D, rope = mmdit
        ranks = [pf.MMDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, text, r, N, 0,
                                         double_layers=D, rope=rope) for r in range(N)]
    elif joint is not None:
        ranks = [pf.JointDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, text, r, N, 0,
                                            double_layers=joint) for r in range(N)]
    elif text:
        ranks = [pf.PixArtCuda.rank_stage(seed, L, hs, heads, 4.0, p, text, r, N, 0)
                 for r in range(N)]
    else:
        ranks = [pf.ToyDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, r, N, 0,
                                          precision=precision) for r in range(N)]
    pf.connect_ranks(ranks)
    outs, stats = [], []
    # one caller stream per rank: a shared caller stream would chain the ranks'
    # joins and forks (rank 1 would wait for rank 0, which waits for rank 1)
    streams = [torch.cuda.Stream() for _ in ranks]
    x = torch.from_numpy(x0.astype(np.float32)).cuda()
    # ranks sharing the device replay CUDA graphs only once all of them built
    # theirs (pf_prepare_pipefusion_device)
    for r, m in enumerate(ranks):
        m.prepare_pipefusion_device(x.data_ptr() if r == 0 else 0, S, M, W, 0.1,
                                    streams[r].cuda_stream)
    for _ in range(runs):
        x.copy_(torch.from_numpy(x0.astype(np.float32)))
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


@pytest.mark.parametrize("D,rope,N,M,W", [(4, False, 2, 4, 1), (2, True, 3, 2, 0),
                                          (1, True, 4, 4, 1)])
def test_same_process_ranks_mmdit(D, rope, N, M, W):
    """MMDiT blocks in rank mode: the LayerNorm statistics travel with the rows
    in the fused peer stores (text rows with patch 0); bitwise equal to the
    single-context engine with the same stage count."""
    seed, L, hs, heads, p, T, S = 4, 4, 128, 4, 256, 24, 4
    x0 = pf.make_initial_latent(5, p, hs)
    with pf.MMDiTCuda(seed, L, hs, heads, 4.0, p, T, N, double_layers=D, rope=rope) as m:
        ref = m.run_pipefusion(x0, S, M, W, 0.1)
    outs, stats = _same_process_ranks(seed, L, hs, heads, p, N, S, M, W, x0, text=T,
                                      mmdit=(D, rope))
    assert np.array_equal(outs[0], ref.final_x)
    assert stats[0] == (ref.stats.fresh_patch_reads, ref.stats.stale_patch_reads)


def test_same_process_ranks_fp32_parity_mode():
    """The fp32 parity mode in rank mode (fused sends write the fp32 rows)."""
    seed, L, hs, heads, p, N, S, M, W = 0, 4, 128, 4, 256, 2, 4, 4, 1
    x0 = pf.make_initial_latent(0, p, hs)
    with pf.ToyDiTCuda(seed, L, hs, heads, 4.0, p, N, precision=pf.PRECISION_FP32) as m:
        ref = m.run_pipefusion(x0, S, M, W, 0.1)
    outs, _ = _same_process_ranks(seed, L, hs, heads, p, N, S, M, W, x0,
                                  precision=pf.PRECISION_FP32)
    assert np.array_equal(outs[0], ref.final_x)
    o = loader.Restatement().build_toy_model(seed, L, hs, heads)
    ora, _ = o.run_pipefusion(x0, S, N, M, W, 0.1)
    assert np.linalg.norm(outs[0] - ora) / np.linalg.norm(ora) <= 1e-4


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


# ----------------------------------------------------------------- graph replay
def _proc_graphs(rank, world, port, cfg, q):
    """One rank per process (the deployment shape): three graph-less runs,
    then three CUDA-graph replays (prepared on every rank first)."""
    try:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        seed, L, hs, heads, p, S, M, W = cfg
        m = pf.ToyDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, rank, world, 0)
        pf.connect_distributed(m)
        x0 = pf.make_initial_latent(0, p, hs)
        x0t = torch.from_numpy(x0.astype(np.float32)).cuda()
        x = torch.empty_like(x0t)
        st = torch.cuda.Stream()
        outs = {}
        for graphs in (False, True):
            m.set_graphs(graphs)
            m.prepare_pipefusion_device(x.data_ptr() if rank == 0 else 0, S, M, W, 0.1,
                                        st.cuda_stream)
            dist.barrier()
            res = []
            for _ in range(3):
                x.copy_(x0t)
                torch.cuda.synchronize()
                m.run_pipefusion_device(x.data_ptr() if rank == 0 else 0, S, M, W, 0.1,
                                        st.cuda_stream)
                m.synchronize(st.cuda_stream)
                res.append(x.double().cpu().numpy())
                dist.barrier()
            outs[graphs] = res
        launches = m.last_launch_count()
        dist.barrier()
        m.close()
        q.put((rank, outs, launches))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "exception " + repr(e), 0))


@pytest.mark.parametrize("N,M", [(2, 4), (4, 8)])
def test_rank_graph_replay_equals_enqueue(N, M):
    """Each rank process captures its plan once; replays re-base the signal
    values. Three replays (bases R, 2R, 3R after three enqueued runs) equal
    the enqueued runs bit for bit (ranks share the test box's one GPU)."""
    cfg = (0, 4, 128, 4, 256, 4, M, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_proc_graphs, args=(r, N, port, cfg, q)) for r in range(N)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(N):
        r, outs, launches = q.get(timeout=600)
        got[r] = (outs, launches)
    for pr in procs:
        pr.join(timeout=60)
    assert not isinstance(got[0][0], str), got[0][0]
    enq, rep = got[0][0][False], got[0][0][True]
    for a, b in zip(enq, rep):
        assert np.array_equal(a, b)
    assert all(np.array_equal(enq[0], o) for o in enq[1:] + rep)
    x0 = pf.make_initial_latent(0, 256, 128)
    ref = _single(0, 4, 128, 4, 256, N, 4, M, 1, x0)
    assert np.array_equal(enq[0], ref.final_x)
    assert all(got[r][1] > 0 for r in range(N))


# ----------------------------------------------------------------- channel close
def _ranks(N, p=256, hs=128, L=4, heads=4):
    ranks = [pf.ToyDiTCuda.rank_stage(0, L, hs, heads, 4.0, p, r, N, 0) for r in range(N)]
    pf.connect_ranks(ranks)
    return ranks


def _run_all(ranks, x0, S, M, W, graphs=True):
    """Enqueue every rank, then wait on each; returns (x, per-rank error)."""
    import torch
    streams = [torch.cuda.Stream() for _ in ranks]
    x = torch.from_numpy(x0.astype(np.float32)).cuda()
    torch.cuda.synchronize()
    errs = [None] * len(ranks)
    for r, m in enumerate(ranks):
        m.set_graphs(graphs)
        try:
            m.run_pipefusion_device(x.data_ptr() if r == 0 else 0, S, M, W, 0.1,
                                    streams[r].cuda_stream)
        except (pf.NumericError, pf.ValidationError) as e:
            errs[r] = e
    for r, m in enumerate(ranks):
        try:
            m.synchronize(streams[r].cuda_stream)
        except pf.NumericError as e:
            errs[r] = errs[r] or e
    return x.double().cpu().numpy(), errs


@pytest.mark.parametrize("fail_rank,op", [(1, 5), (1, 40), (0, 12), (2, 25)])
def test_thrown_error_closes_every_channel(fail_rank, op):
    """A rank that throws mid-plan (execute.cpp:345-348 close_all) closes the
    run: every rank returns, the others report "channel closed mid-run", the
    root cause wins (execute.cpp:357-374), and the next run is bit-exact."""
    N, p, hs, S, M, W = 3, 256, 128, 4, 4, 1
    x0 = pf.make_initial_latent(0, p, hs)
    ref = _single(0, 4, hs, 4, p, N, S, M, W, x0)
    ranks = _ranks(N)
    ranks[fail_rank].debug_fail_at(op)
    _, errs = _run_all(ranks, x0, S, M, W)
    assert "injected failure" in str(errs[fail_rank])
    for r in range(N):
        if r != fail_rank:
            assert str(errs[r]) == "channel closed mid-run", (r, errs[r])
        assert not ranks[r].rank_broken
    assert "injected failure" in str(pf.root_cause(errs))
    # the failing rank played its message protocol to the end: the counters
    # agree and the next run (graphs on and off) is bit-exact, no reset needed
    ranks[fail_rank].debug_fail_at(-1)
    for graphs in (True, False):
        x, errs = _run_all(ranks, x0, S, M, W, graphs=graphs)
        assert errs == [None] * N
        assert np.array_equal(x, ref.final_x)
    for m in ranks:
        m.close()


def test_nan_root_cause_is_the_first_non_finite_layer():
    """A NaN born in rank 1's layer reaches rank 0 a step later; every rank
    returns, and the root cause is rank 1's (earliest timestep)."""
    N, p, hs, S, M, W = 2, 256, 128, 4, 4, 1
    x0 = pf.make_initial_latent(0, p, hs)
    ranks = _ranks(N)
    ranks[1].debug_poison_layer(3)
    _, errs = _run_all(ranks, x0, S, M, W)
    assert all(isinstance(e, pf.NumericError) for e in errs), errs
    assert str(errs[1]) == "non-finite activation at timestep 3, layer 3"
    assert str(pf.root_cause(errs)) == "non-finite activation at timestep 3, layer 3"
    for m in ranks:
        m.close()


def test_watchdog_releases_a_rank_whose_peer_never_runs(monkeypatch):
    monkeypatch.setenv("PF_RANK_TIMEOUT_S", "2")
    import torch
    N, p, hs, S, M, W = 2, 256, 128, 3, 2, 1
    x0 = pf.make_initial_latent(0, p, hs)
    ranks = _ranks(N)
    x = torch.from_numpy(x0.astype(np.float32)).cuda()
    st = torch.cuda.Stream()
    ranks[0].run_pipefusion_device(x.data_ptr(), S, M, W, 0.1, st.cuda_stream)  # rank 1 idle
    with pytest.raises(pf.NumericError, match="channel closed mid-run"):
        ranks[0].synchronize(st.cuda_stream)
    assert ranks[0].rank_broken
    with pytest.raises(pf.NumericError, match="channel closed mid-run"):
        ranks[0].run_pipefusion_device(x.data_ptr(), S, M, W, 0.1, st.cuda_stream)
    for m in ranks:
        m.rank_reset()
    ref = _single(0, 4, hs, 4, p, N, S, M, W, x0)
    x, errs = _run_all(ranks, x0, S, M, W)
    assert errs == [None] * N and np.array_equal(x, ref.final_x)
    for m in ranks:
        m.close()


def _proc_fail(rank, world, port, cfg, q):
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        seed, L, hs, heads, p, S, M, W = cfg
        m = pf.ToyDiTCuda.rank_stage(seed, L, hs, heads, 4.0, p, rank, world, 0)
        pf.connect_distributed(m)
        if rank == 1:
            m.debug_fail_at(9)
        x0 = pf.make_initial_latent(0, p, hs)
        try:
            m.run_pipefusion(x0 if rank == 0 else None, S, M, W, 0.1)
            out = "no error"
        except pf.NumericError as e:
            out = str(e)
        # the next run needs no reset: bitwise equal to a fresh single context
        m.debug_fail_at(-1)
        res = m.run_pipefusion(x0 if rank == 0 else None, S, M, W, 0.1)
        dist.barrier()
        m.close()
        q.put((rank, out, res.final_x))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "exception " + repr(e), None))


def test_process_per_rank_failure_reports_root_cause_everywhere():
    seed, L, hs, heads, p, S, M, W = 0, 4, 128, 4, 256, 4, 4, 1
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cfg = (seed, L, hs, heads, p, S, M, W)
    procs = [ctx.Process(target=_proc_fail, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(world):
        r, msg, x = q.get(timeout=300)
        got[r] = (msg, x)
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert got[r][0].startswith("injected failure at plan op 9 of rank 1"), got[r][0]
    x0 = pf.make_initial_latent(0, p, hs)
    ref = _single(seed, L, hs, heads, p, world, S, M, W, x0)
    assert np.array_equal(got[0][1], ref.final_x)
