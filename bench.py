#!/usr/bin/env python
"""Benchmark: seconds per image of PipeFusion DiT inference on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c1|cref] [--patches M]

Metric (BASELINE.json): "sec/image DiT latency at 1/2/4/8 B200 (PipeFusion
N,M); % of BF16 TC peak". One bench "step" = one image: the full 20-step
PipeFusion denoising loop (1 synchronous warmup step + 19 pipelined steps) of
the PixArt-alpha-shaped toy DiT (28 layers, hidden 1152, 16 heads, 4096
tokens = 1024 px), random-init weights from the reference's own RNG stream
(build_toy_model, seed 0) and the reference's synthetic latent.

* value  - device time per image with the latent already resident in HBM
           (CUDA events on the caller stream, which joins every stage stream).
* e2e    - the same through the C ABI the reference would bind
           (pf_run_pipefusion): fp64 host latent in, host->device copy, run,
           device->host copy, fp64 host latent out; wall clock per call.
* roofline - dominant kernel from a CUDA-event profile of one extra run
           (every kernel bracketed by events on its own stream), algorithmic
           FLOPs per SURVEY 8(d): QKV 6*r*hs^2, attention 4*r*p*hs, out-proj
           2*r*hs^2, MLP 2*2*r*hs*mlp per (patch, layer).
* cpu_baseline / --impl reference - the reference's own CPU code
           (oracle/_ref, compiled from /root/reference) timed on this host on
           sampled toy_layer_forward units at the true shape, extrapolated to
           a full image (a full C2 image is ~1e14 FLOP on an fp64 scalar loop).

Under torchrun with N > 1 ranks there is one process per GPU: rank d owns
pipeline stage d (its L/N layers) on GPU LOCAL_RANK, and stage-boundary
activations / the returned eps go straight into the neighbour's landing
buffers over peer memory (NVLink, CUDA IPC; rank_plan.h). Each rank times
its own stream with CUDA events; the reported time is the max over ranks.
Without torchrun, `--gpus N` (N > 1) launches the same N processes itself
(one per GPU, RANK/WORLD_SIZE/LOCAL_RANK set, rendezvous on 127.0.0.1) and
relays rank 0's line, so the plain command times the same rank-mode path
(per-rank CUDA-graph replay, patch lanes) as the torchrun launch.
`--single-process` keeps the older one-process multi-device engine (tests).
"""
from __future__ import annotations

import argparse
import json
import os

# Rank-mode patch lanes (stream-memory-op signal waits on several streams)
# need more than the default 8 hardware queues; set before CUDA initialises.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sec/image DiT latency at 1/2/4/8 B200 (PipeFusion N,M); % of BF16 TC peak"
UNIT = "s/image"

CONFIGS = {
    # name: (layers, hidden, heads, seq_len, diffusion steps, warmup steps)
    "c2": dict(name="PixArt-alpha-shaped DiT 1024px (28 layers, hidden 1152, 16 heads, "
                    "4096 tokens), 20 steps, 1 warmup",
               L=28, hs=1152, heads=16, p=4096, S=20, W=1),
    "c3": dict(name="PixArt-alpha-shaped DiT 2048px (28 layers, hidden 1152, 16 heads, "
                    "16384 tokens), 20 steps, 1 warmup",
               L=28, hs=1152, heads=16, p=16384, S=20, W=1),
    "c2px": dict(name="PixArt-alpha DiT block variant 1024px (28 layers, hidden 1152, 16 heads, "
                      "4096 tokens, 120 text tokens; adaLN-single + LayerNorm, cross-attention, "
                      "GELU MLP), 20 steps, 1 warmup",
                 L=28, hs=1152, heads=16, p=4096, S=20, W=1, block="pixart", T=120),
    "c3px": dict(name="PixArt-alpha DiT block variant 2048px (28 layers, hidden 1152, 16 heads, "
                      "16384 tokens, 120 text tokens), 20 steps, 1 warmup",
                 L=28, hs=1152, heads=16, p=16384, S=20, W=1, block="pixart", T=120),
    "c4": dict(name="SD3-medium-shaped MMDiT 1024px (24 double-stream joint blocks, hidden "
                    "1536, 24 heads, 4096 image + 333 text tokens in one K/V buffer; adaLN-Zero, "
                    "LayerNorm, QK RMSNorm, GELU MLP), 20 steps, 1 warmup",
               L=24, hs=1536, heads=24, p=4096, S=20, W=1, block="mmdit", T=333, D=24,
               rope=False),
    "c5": dict(name="Flux.1-shaped MMDiT 2048px (19 double-stream + 38 single-stream blocks, "
                    "hidden 3072, 24 heads, 16384 image + 512 text tokens, axial RoPE, QK "
                    "RMSNorm, ~11.8B parameters), 28 steps, 1 warmup",
               L=57, hs=3072, heads=24, p=16384, S=28, W=1, block="mmdit", T=512, D=19,
               rope=True),
    "c4toy": dict(name="SD3-medium-shaped joint-attention DiT 1024px (24 blocks, hidden 1536, "
                       "24 heads, 4096 image + 333 text tokens; toy arithmetic per stream), "
                       "20 steps, 1 warmup",
                  L=24, hs=1536, heads=24, p=4096, S=20, W=1, block="joint", T=333),
    "c1": dict(name="tiny DiT (4 layers, hidden 128, 4 heads, 256 tokens), 5 steps, 1 warmup",
               L=4, hs=128, heads=4, p=256, S=5, W=1),
    "cref": dict(name="reference_execute.cfg (4 layers, hidden 32, 4 heads, 64 tokens), 20 "
                      "steps, 1 warmup", L=4, hs=32, heads=4, p=64, S=20, W=1),
}


def config_of(c, n, M):
    """The `config` object of both arms (same keys and values)."""
    return {"workload": c["name"], "layers": c["L"], "hidden_size": c["hs"],
            "heads": c["heads"], "seq_len": c["p"], "diffusion_steps": c["S"],
            "warmup_steps": c["W"], "patches": M, "stages": n,
            "parallelism": f"pipefusion N={n} M={M}",
            "l2": "working set > L2 (0.9 GB bf16 weights + 0.6 GB K/V per image pass at "
                  "C2), no explicit flush"}


def flops_per_image(c, mlp):
    """The reference's ComputeModel (simulate.cpp:30-44) for mlp_ratio 4:
    S * L * (24 p hs^2 + 4 p^2 hs); generalised to mlp = 4 hs."""
    p, hs = c["p"], c["hs"]
    if c.get("block") in ("joint", "mmdit"):
        # both streams' GEMMs over their rows and joint attention over p + T
        # rows, per step and layer; the text rows run once per step
        pt = p + c["T"]
        return c["S"] * c["L"] * (8 * pt * hs * hs + 4 * pt * hs * mlp + 4 * pt * pt * hs)
    if c.get("block") == "pixart":
        # QKV 6, out 2, cross-q 2, cross-out 2 (x p hs^2), MLP 4 p hs mlp, self- and
        # cross-attention 4 p (p + T) hs per step and layer; text K/V once per image
        T = c["T"]
        return (c["S"] * c["L"] * (12 * p * hs * hs + 4 * p * hs * mlp + 4 * p * (p + T) * hs)
                + c["L"] * 4 * T * hs * hs)
    return c["S"] * c["L"] * (8 * p * hs * hs + 4 * p * hs * mlp + 4 * p * p * hs)


def load_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", ",".join(str(g) for g in self.gpus)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_port_baseline_pixart(c, budget_s=20.0, sample_rows=32):
    """PixArt block: the reference has no such block, so the CPU baseline is
    the fp64 oracle port (oracle/px_oracle.c, scalar, one layer unit per host
    thread) on sampled 32-row units at the true shape, extrapolated."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import loader
    if not loader.RESTATEMENT_LIB.exists():
        loader.build(reference=False)
    o = loader.PixArtOracle(0, 1, c["hs"], c["heads"], 4.0, c["T"])
    cores = min(os.cpu_count() or 1, 64)
    rng = np.random.default_rng(0)
    k = rng.uniform(-1, 1, (c["p"], c["hs"]))
    v = rng.uniform(-1, 1, (c["p"], c["hs"]))

    def one(i):
        h = np.random.default_rng(i).uniform(-1, 1, (sample_rows, c["hs"]))
        o.layer_forward(0, i % c["S"], c["S"], h, k, v, (i * sample_rows) % c["p"])
        return 1

    done, t0 = 0, time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        while True:
            done += sum(ex.map(one, range(done, done + cores)))
            if time.perf_counter() - t0 > budget_s * 0.5 or done >= 4 * cores:
                break
    wall = time.perf_counter() - t0
    samples_per_image = c["S"] * c["L"] * (c["p"] / sample_rows)
    return {"value": wall / done * samples_per_image, "unit": UNIT, "cores": cores,
            "kind": "port",
            "sample": (f"{done} PixArt-block layer units of {sample_rows} query rows x "
                       f"{c['p']}-row K/V (oracle/px_oracle.c fp64, {cores} threads in "
                       f"{wall:.1f}s); extrapolated x{samples_per_image:.0f} units/image")}


def cpu_port_baseline_mmdit(c, budget_s=20.0, sample_rows=32):
    """MMDiT blocks: no reference path exists, so the CPU baseline is the fp64
    spec (oracle/mmdit_oracle.py, numpy) on sampled 32-row units of one block
    of the true width (a double block for SD3, a single block for Flux's
    majority) against the full joint K/V buffer, extrapolated."""
    from oracle import mmdit_oracle as mo
    single = c["D"] < c["L"] - c["D"]
    m = mo.MMDiT(0, 1, c["hs"], c["heads"], 4 * c["hs"], c["T"], c["p"], 0 if single else 1,
                 rope=c["rope"])
    pt = c["p"] + c["T"]
    rng = np.random.default_rng(0)
    k = rng.uniform(-1, 1, (pt, c["hs"]))
    v = rng.uniform(-1, 1, (pt, c["hs"]))
    done, t0 = 0, time.perf_counter()
    while True:
        h = np.random.default_rng(done).uniform(-1, 1, (sample_rows, c["hs"]))
        row0 = c["T"] + (done * sample_rows) % c["p"]
        mo.layer_forward(m, 0, c["S"] - 1, c["S"], h, k, v, row0)
        done += 1
        if time.perf_counter() - t0 > budget_s * 0.5 or done >= 64:
            break
    wall = time.perf_counter() - t0
    units = c["S"] * c["L"] * (pt / sample_rows)
    cores = os.cpu_count() or 1
    return {"value": wall / done * units, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"{done} {'single' if single else 'double'}-stream block units of "
                       f"{sample_rows} rows x {pt}-row joint K/V (oracle/mmdit_oracle.py, "
                       f"numpy fp64, BLAS threads up to {cores}) in {wall:.1f}s; extrapolated "
                       f"x{units:.0f} units/image")}


def cpu_reference_baseline(c, budget_s=20.0, sample_rows=32, run_shape=(1, 1)):
    """Time the reference's own toy_layer_forward (oracle/_ref, built from
    /root/reference) at the true shape on `sample_rows` query rows against a
    full p-row K/V buffer, one sample per host core in parallel, and
    extrapolate to one image: S * L * (p / sample_rows) samples."""
    if c.get("block") == "pixart":
        return cpu_port_baseline_pixart(c, budget_s, sample_rows)
    if c.get("block") == "mmdit":
        return cpu_port_baseline_mmdit(c, budget_s, sample_rows)
    from concurrent.futures import ThreadPoolExecutor
    from oracle import loader
    if not loader.REFERENCE_LIB.exists():
        loader.build(reference=True)
    ref = loader.Reference()
    model = ref.build_toy_model(0, 1, c["hs"], c["heads"], 4.0)
    cores = min(os.cpu_count() or 1, 64)
    rng = np.random.default_rng(0)
    # joint block: each stream's rows run the toy block against all p + T rows
    kvp = c["p"] + (c["T"] if c.get("block") == "joint" else 0)
    k = rng.uniform(-1, 1, (kvp, c["hs"]))
    v = rng.uniform(-1, 1, (kvp, c["hs"]))

    def one(i):
        h = np.random.default_rng(i).uniform(-1, 1, (sample_rows, c["hs"]))
        row0 = (i * sample_rows) % kvp
        model.layer_forward(0, h, k, v, row0)
        return 1

    done, t0 = 0, time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        while True:
            done += sum(ex.map(one, range(done, done + cores)))
            if time.perf_counter() - t0 > budget_s * 0.5 or done >= 8 * cores:
                break
    wall = time.perf_counter() - t0
    per_sample = wall / done  # throughput-equivalent seconds per sample
    samples_per_image = c["S"] * c["L"] * (kvp / sample_rows)
    if c.get("block") is None and per_sample * cores * samples_per_image < budget_s:
        # small enough for the real thing: one full run_pipefusion image through the
        # reference's own executor (Threads backend, the CLI default), timed
        full = ref.build_toy_model(0, c["L"], c["hs"], c["heads"], 4.0)
        x0 = ref.make_initial_latent(0, c["p"], c["hs"])
        n, M = run_shape
        t1 = time.perf_counter()
        full.run_pipefusion(x0, c["S"], n, M, c["W"], 0.1)
        dt = time.perf_counter() - t1
        return {"value": dt, "unit": UNIT, "cores": n, "kind": "reference",
                "sample": (f"one full image: the reference's run_pipefusion (toy_model.cpp / "
                           f"execute.cpp, Threads backend, {n} worker threads, M={M}), timed "
                           f"end to end")}
    return {
        "value": per_sample * samples_per_image, "unit": UNIT, "cores": cores,
        "kind": "reference",
        # the reference's own N=1 path (Backend::Inline, execute.cpp:694) is
        # one host thread; spreading sampled units over `cores` threads makes
        # `value` a throughput-equivalent figure about `cores` x kinder to the CPU
        "single_thread_value": per_sample * cores * samples_per_image,
        "semantics": (f"units spread over {cores} host threads (throughput-equivalent); the "
                      "reference's own N=1 run is single-threaded (execute.cpp:694), see "
                      "single_thread_value"),
        "sample": (f"{done} toy_layer_forward units of {sample_rows} query rows x "
                   f"{kvp}-row K/V at hs={c['hs']} heads={c['heads']} (reference "
                   f"toy_model.cpp, fp64, {cores} threads in {wall:.1f}s); extrapolated "
                   f"x{samples_per_image:.0f} units/image (linear in rows)"),
    }


# ----------------------------------------------------------------------------- ours
def run_ours(args, c, world, rank):
    import torch
    import paper_2405_14430_b200 as pf

    n = args.gpus
    M = args.patches or n
    peaks, peak_kind = load_peaks()
    px = c.get("block") == "pixart"
    t_build = time.perf_counter()
    if world > 1:
        # one process per GPU: this rank owns stage `rank` (rank mode); stage
        # boundaries go over peer memory (NVLink / CUDA IPC), see rank_plan.h
        if world != n:
            raise SystemExit(f"--gpus {n} must equal the torchrun world size {world}")
        # (on a box with fewer GPUs than ranks, ranks share devices round-robin:
        # correctness runs of the multi-process path on one GPU)
        local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if px:
            model = pf.PixArtCuda.rank_stage(0, c["L"], c["hs"], c["heads"], 4.0, c["p"],
                                             c["T"], rank, world, local)
        elif c.get("block") == "joint":
            model = pf.JointDiTCuda.rank_stage(0, c["L"], c["hs"], c["heads"], 4.0, c["p"],
                                               c["T"], rank, world, local,
                                               double_layers=c.get("D"))
        elif c.get("block") == "mmdit":
            model = pf.MMDiTCuda.rank_stage(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], c["T"],
                                            rank, world, local, double_layers=c["D"],
                                            rope=c["rope"])
        else:
            model = pf.ToyDiTCuda.rank_stage(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], rank,
                                             world, local)
        pf.connect_distributed(model)
        devices = [local]
    else:
        torch.cuda.set_device(0)
        devices = list(range(n))
        if px:
            model = pf.PixArtCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], c["T"], n,
                                  devices)
        elif c.get("block") == "joint":
            model = pf.JointDiTCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], c["T"], n,
                                    devices, double_layers=c.get("D"))
        elif c.get("block") == "mmdit":
            model = pf.MMDiTCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], c["T"], n,
                                 devices, double_layers=c["D"], rope=c["rope"])
        else:
            model = pf.ToyDiTCuda(0, c["L"], c["hs"], c["heads"], 4.0, c["p"], n, devices)
    t_build = time.perf_counter() - t_build
    mlp = model.mlp_hidden
    x0 = pf.make_initial_latent(0, c["p"], c["hs"])
    holds_x = rank == 0
    x0_dev = torch.from_numpy(x0.astype(np.float32)).cuda() if holds_x else None
    x_dev = torch.empty_like(x0_dev) if holds_x else None
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream

    def one_image():
        if holds_x:
            x_dev.copy_(x0_dev)
        model.run_pipefusion_device(x_dev.data_ptr() if holds_x else 0, c["S"], M, c["W"], 0.1,
                                    sp)

    # rank mode: every rank builds its CUDA graph before any rank replays one
    # (pf_prepare_pipefusion_device), then the ranks start together
    model.prepare_pipefusion_device(x_dev.data_ptr() if holds_x else 0, c["S"], M, c["W"], 0.1,
                                    sp)
    barrier(world)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one_image()
        model.synchronize(sp)
        launches = model.last_launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(devices if world == 1 else [devices[0]]) as clocks:
        with torch.cuda.stream(stream):
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            h0 = time.perf_counter()
            for _ in range(args.steps):
                one_image()
            host_ms = (time.perf_counter() - h0) * 1e3
            ev1.record(stream)
            model.synchronize(sp)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    clock_info = clocks.summary()
    # host time to enqueue (or replay) one image vs its device time, per rank
    enqueue = {"host_ms_per_image": gather_ranks(host_ms / args.steps, world),
               "device_ms_per_image": gather_ranks(ms / args.steps, world)}
    ms = max_over_ranks(ms, world)
    barrier(world)

    sec_per_image = ms / 1e3 / args.steps
    # ---- e2e through the C ABI with host buffers (all ranks call it together)
    # host buffers in pinned memory (the fp64 latent in, the fp64 result out),
    # allocated once and reused across calls as a serving loop would
    x_host = out_host = None
    if holds_x:
        x_host = torch.empty(x0.shape, dtype=torch.float64, pin_memory=True).numpy()
        x_host[...] = x0
        out_host = torch.empty(x0.shape, dtype=torch.float64, pin_memory=True).numpy()
    e2e_times = []
    out = None
    for i in range(max(2, args.steps) + 1):
        barrier(world)
        t0 = time.perf_counter()
        out = model.run_pipefusion(x_host, c["S"], M, c["W"], 0.1, out=out_host)
        dt = max_over_ranks(time.perf_counter() - t0, world)
        if i > 0:
            e2e_times.append(dt)
    e2e = statistics.mean(e2e_times)
    # ---- per-kernel CUDA-event profile of one extra image (every rank profiles
    # its own stage; rank 0's is reported)
    model.set_profiling(True)
    barrier(world)
    with torch.cuda.stream(stream):
        one_image()
        model.synchronize(sp)
    prof = model.kernel_profile()
    model.set_profiling(False)
    barrier(world)
    all_launches = gather_ranks(launches, world)
    mem = {"param_bytes_per_stage": gather_ranks(model.param_bytes(), world),
           "kv_bytes_per_stage": gather_ranks(model.kv_bytes(), world)}
    if rank != 0:
        return None
    finite = bool(np.isfinite(out.final_x).all())
    nvlink = None
    bb = boundary_bytes(c, world, M)
    if bb is not None:
        # the boundary stores are fused into the last MLP-out GEMM of each
        # stage, so the link is timed per image: bytes on the busiest boundary
        # over the image time, against one direction of one GPU's NVLink 5
        link_peak = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal
        busiest = max(bb)
        gbs = busiest / sec_per_image / 1e9
        nvlink = {"bytes_per_image_per_boundary": bb, "achieved_gbs": gbs,
                  "peak_gbs": link_peak, "frac": gbs / link_peak,
                  "ideal_ms_per_image": busiest / (link_peak * 1e9) * 1e3,
                  "note": "fp32 + bf16 activation rows per message, fp32 eps back to "
                          "rank 0; peak = measured peer copy per direction (770 GB/s, "
                          "900 nominal); the stores are fused into the last MLP-out GEMM of "
                          "each stage, so achieved = bytes on the busiest boundary / image time"}
    # ---- per-kernel CUDA-event profile of one extra image
    gemm_kinds = ["gemm_qkv", "gemm_out_proj", "gemm_mlp_in", "gemm_mlp_out", "gemm_cross_q",
                  "gemm_cross_out"]
    dom = max((k for k in prof if k not in ("sampler", "conditioning")),
              key=lambda k: prof[k]["ms"])
    peak_tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    kernels = {}
    for k, d in prof.items():
        if d["launches"] == 0:
            continue
        e = {"ms_per_image": d["ms"], "launches": d["launches"],
             "avg_us": 1e3 * d["ms"] / d["launches"]}
        if d["flops"]:
            e["tflops"] = d["flops"] / (d["ms"] * 1e-3) / 1e12
            e["frac_bf16"] = e["tflops"] / peak_tf
        if d["bytes"]:
            e["gbs"] = d["bytes"] / (d["ms"] * 1e-3) / 1e9
            e["frac_hbm"] = e["gbs"] / peaks["hbm_gbs"]
        kernels[k] = e
    gemm_ms = sum(prof[k]["ms"] for k in gemm_kinds)
    gemm_fl = sum(prof[k]["flops"] for k in gemm_kinds)
    d = prof[dom]
    achieved = d["flops"] / d["launches"] / (d["ms"] / d["launches"] * 1e-3) / 1e12
    traffic, traffic_src = None, None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        # dram__bytes_read + dram__bytes_write per launch of this config's
        # dominant kernel, from an ncu --set full capture of the same config
        # and patch count (null when that capture does not exist)
        try:
            t = json.loads(tf.read_text())
            ent = t.get("configs", {}).get(f"{args.config}_m{M}", {})
            traffic = ent.get(dom)
            traffic_src = ent.get("source") if traffic is not None else None
        except Exception:
            traffic = None
    total_flops = flops_per_image(c, mlp)
    line = {
        "metric": METRIC, "value": sec_per_image, "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "processes": ("one per GPU (rank mode, peer-memory stage boundaries)" if world > 1
                      else "one"),
        "dtype": "bf16", "data": "synthetic (reference RNG: build_toy_model seed 0, "
                                  "make_initial_latent seed 0)",
        "config": config_of(c, n, M),
        "tc_frac_image": total_flops / sec_per_image / 1e12 / peak_tf,
        "block": c.get("block", "toy"),
        # the C ABI moves the fp64 host latent both ways (converted on the GPU)
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": c["p"] * c["hs"] * 8,
                "d2h_bytes_per_step": c["p"] * c["hs"] * 8,
                "api": "pf_run_pipefusion (C ABI, fp64 host latent in/out, pinned host "
                       "buffers reused across calls)"},
        "roofline": {"bound": "tensor", "kernel": dom, "achieved": achieved,
                     "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved / peak_tf,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": f"{peak_kind} bf16 sustained",
                     "measured_in": ("a separate profiled image: every kernel bracketed by "
                                     "CUDA events on its stream, one lane, no graph replay "
                                     "(value runs graphs" + (" and patch lanes" if M > 1
                                                             else "") + ")"),
                     "gemm_all_frac": (gemm_fl / (gemm_ms * 1e-3) / 1e12) / peak_tf},
        "kernels": kernels,
        "gpu_launches": sum(all_launches) * args.steps,
        "gpu_launches_note": ("summed over the ranks" if world > 1 else "all stages"),
        "enqueue": enqueue,
        "nvlink": nvlink,
        "clocks": clock_info,
        "finite": finite,
        "model_build_s": t_build,
        "memory": mem,
    }
    return line


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def gather_ranks(v, world):
    """[v of rank 0, v of rank 1, ...] (every rank gets the list)."""
    if world <= 1:
        return [v]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, v)
    return out


def boundary_bytes(c, world, M):
    """Bytes one image moves over each stage boundary (rank d -> d+1) and
    from the last rank back to rank 0, from the rank plans (pf_rank_plan):
    activations travel as fp32 rows plus their bf16 copy (the next stage's
    GEMM operand), PixArt adds per-row LayerNorm partial stats (hs/32 float2),
    the returned eps is fp32 only. Per SURVEY 8(d) / costmodel.cpp:117-123."""
    if world <= 1:
        return None
    import paper_2405_14430_b200 as pf
    hs, p = c["hs"], c["p"]
    per_rank = []
    for d in range(world):
        plan = pf.rank_plan(d, world, c["S"], M, c["W"], p)
        sends = plan[plan[:, 0] == 2]  # kind 2 = send
        rows = int(sends[:, 4].sum())
        last = d == world - 1
        if c.get("block") == "joint" and not last:
            # the text rows ride along with the full sequence and patch 0
            rows += c["T"] * int((sends[:, 2] <= 0).sum())
        b = rows * hs * 4 + (0 if last else rows * hs * 2)
        if c.get("block") == "pixart" and not last:
            b += rows * (hs // 32) * 8
        per_rank.append(b)
    return per_rank


def max_over_ranks(v, world):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def spawn_ranks(args):
    """`--gpus N` without torchrun: start one bench process per GPU (the same
    environment torchrun would give them) and relay rank 0's JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    n = args.gpus
    import tempfile
    procs = []
    out = tempfile.TemporaryFile()
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), GROUP_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_DEVICE_MAX_CONNECTIONS="32")
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve())]
                                      + sys.argv[1:], env=env,
                                      stdout=out if r == 0 else subprocess.DEVNULL))
    rc = 0
    while any(pr.poll() is None for pr in procs):
        failed = [pr for pr in procs if pr.poll() not in (None, 0)]
        if failed:  # one rank died: the others would wait for it forever
            rc = failed[0].returncode
            for pr in procs:
                if pr.poll() is None:
                    pr.kill()
            break
        time.sleep(0.2)
    for pr in procs:
        rc = rc or pr.wait()
    out.seek(0)
    sys.stdout.write(out.read().decode(errors="replace"))
    sys.stdout.flush()
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--patches", type=int, default=0, help="M (default: N)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--single-process", action="store_true",
                    help="--gpus N from one process (multi-device engine, no rank mode)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world == 1 and args.gpus > 1 and args.impl == "ours" and not args.single_process:
        sys.exit(spawn_ranks(args))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    c = CONFIGS[args.config]

    if args.impl == "reference":
        if rank == 0:
            base = cpu_reference_baseline(c, budget_s=args.cpu_budget,
                                          run_shape=(args.gpus, args.patches or args.gpus))
            line = {"metric": METRIC, "value": base["value"], "unit": UNIT,
                    "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                    "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
                    "dtype": "f64", "data": "synthetic", "impl": "reference",
                    "config": config_of(c, args.gpus, args.patches or args.gpus),
                    "cpu_baseline": base,
                    "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    line = run_ours(args, c, world, rank)
    if rank == 0:
        if not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_reference_baseline(
                    c, budget_s=args.cpu_budget, run_shape=(args.gpus, args.patches or args.gpus))
            except Exception as e:  # the checker must not sink the GPU number
                line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
