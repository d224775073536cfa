"""One-process-per-stage PipeFusion: the per-rank plan (rank_plan.h), CPU only.

The GPU engine's rank mode executes pf_rank_plan's op list over peer memory.
Here the same op lists are (1) checked for protocol consistency (every send
has its matching receive with the same patch, rows and timestep tag; every
received message is acknowledged once, in order; a send never overwrites
rows the receiver has not acknowledged) and (2) executed by world_size 2 and
3 process groups over torch.distributed (gloo, 127.0.0.1) with the oracle's
layer arithmetic (oracle/pf_oracle.c, bit-exact with the reference). The
distributed result must equal the reference's single-process
run_pipefusion (execute.cpp:167-223) bit for bit, as the reference's own
threads backend does (test_execute.cpp:151-164).
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import paper_2405_14430_b200 as pf
from oracle import loader

KIND = {n: i for i, n in enumerate(pf.PLAN_KINDS)}


def plans(world, steps, patches, warmup, p):
    return [pf.rank_plan(r, world, steps, patches, warmup, p) for r in range(world)]


CASES = [(2, 4, 2, 1), (3, 5, 4, 2), (4, 3, 2, 0), (2, 3, 1, 3), (4, 6, 8, 1), (3, 4, 2, 4)]


@pytest.mark.parametrize("world,steps,patches,warmup", CASES)
def test_messages_match_across_each_boundary(world, steps, patches, warmup):
    p = 16 * patches
    pl = plans(world, steps, patches, warmup, p)
    for d in range(world):
        succ = (d + 1) % world
        sends = [tuple(o[[1, 2, 3, 4, 5]]) for o in pl[d] if o[0] == KIND["send"]]
        recvs = [tuple(o[[1, 2, 3, 4, 5]]) for o in pl[succ] if o[0] == KIND["recv"]]
        assert sends == recvs, (d, sends, recvs)
        assert [s[4] for s in sends] == list(range(1, len(sends) + 1))
        n_expected = warmup + (steps - warmup) * patches
        assert len(sends) == n_expected


@pytest.mark.parametrize("world,steps,patches,warmup", CASES)
def test_acks_and_overlaps(world, steps, patches, warmup):
    p = 16 * patches
    pl = plans(world, steps, patches, warmup, p)
    for d in range(world):
        ops = pl[d]
        recv_msgs = [o[5] for o in ops if o[0] == KIND["recv"]]
        acks = [o[5] for o in ops if o[0] == KIND["ack"]]
        # cumulative acknowledgements, increasing, ending at the last message
        assert acks == sorted(acks) and len(set(acks)) == len(acks)
        assert acks and acks[-1] == recv_msgs[-1]
        # an ack never precedes the receive of its message
        seen = set()
        for o in ops:
            if o[0] == KIND["recv"]:
                seen.add(o[5])
            if o[0] == KIND["ack"]:
                assert o[5] in seen
        # a send waits for the last earlier message on the same rows
        rows_of = {}
        for o in ops:
            if o[0] != KIND["send"]:
                continue
            msg, ov, r0, nr = o[5], o[6], o[3], o[4]
            prev = [m for m, (a, b) in rows_of.items() if a < r0 + nr and r0 < a + b]
            assert ov == (max(prev) if prev else 0)
            rows_of[msg] = (r0, nr)


def test_plan_rejects_invalid_arguments():
    with pytest.raises(pf.ValidationError):
        pf.rank_plan(0, 1, 4, 2, 1, 16)
    with pytest.raises(pf.ValidationError):
        pf.rank_plan(0, 2, 4, 3, 1, 16)


# ----------------------------------------------------------------- gloo execution
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, cfg, q):
    import torch
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        L, hs, heads, p, S, M, W, eta, seed = cfg
        model = loader.Restatement().build_toy_model(seed, L, hs, heads)
        x = loader.Restatement().make_initial_latent(seed + 1, p, hs) if rank == 0 else None
        cb = model.weights()[1]
        lo, hi = rank * L // world, (rank + 1) * L // world
        kv = {l: (np.zeros((p, hs)), np.zeros((p, hs))) for l in range(lo, hi)}
        h = np.zeros((p, hs))
        eps = np.zeros((p, hs))
        pending = []
        succ, pred = (rank + 1) % world, (rank - 1) % world
        for o in pf.rank_plan(rank, world, S, M, W, p):
            kind, t, patch, r0, nr, msg = (int(v) for v in o[:6])
            rows = slice(r0, r0 + nr)
            if kind == KIND["prepare"]:
                if o[7]:
                    x[rows] = x[rows] - eta * eps[rows]
                h[rows] = x[rows] + cb
            elif kind == KIND["compute"]:
                hr = np.ascontiguousarray(h[rows])
                for l in range(lo, hi):
                    hr, k, v = model.layer_forward(l, hr, kv[l][0], kv[l][1], r0)
                    kv[l] = (k, v)
                h[rows] = hr
            elif kind == KIND["send"]:
                tag = torch.tensor([patch, t, msg], dtype=torch.int64)
                buf = torch.from_numpy(np.ascontiguousarray(h[rows]).copy())
                pending += [dist.isend(tag, succ), dist.isend(buf, succ), tag, buf]
            elif kind == KIND["recv"]:
                tag = torch.empty(3, dtype=torch.int64)
                dist.recv(tag, pred)
                # the reference's protocol check (execute.cpp:257-265)
                assert tuple(tag.tolist()) == (patch, t, msg), (tag.tolist(), patch, t, msg)
                buf = torch.empty((nr, hs), dtype=torch.float64)
                dist.recv(buf, pred)
                (eps if rank == 0 else h)[rows] = buf.numpy()
            elif kind == KIND["latent_update"]:
                x = x - eta * eps
        for w in pending:
            if hasattr(w, "wait"):
                w.wait()
        dist.barrier()
        q.put((rank, x))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world,S,M,W", [(2, 4, 4, 1), (3, 5, 2, 2), (2, 3, 2, 0)])
def test_gloo_ranks_reproduce_the_reference_run(world, S, M, W):
    L, hs, heads, p, eta, seed = 6, 16, 4, 32, 0.1, 3
    cfg = (L, hs, heads, p, S, M, W, eta, seed)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    rs = loader.Restatement()
    model = rs.build_toy_model(seed, L, hs, heads)
    x0 = rs.make_initial_latent(seed + 1, p, hs)
    ref_x, _ = model.run_pipefusion(x0, S, 1, M, W, eta)
    assert np.array_equal(out[0], ref_x)
