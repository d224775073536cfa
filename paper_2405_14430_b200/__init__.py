"""B200-native PipeFusion executor (host-side Python mirror of the C ABI).

The product is the sm_100a shared library `libpipefusion_b200.so` (C ABI in
include/pipefusion_b200.h). This module binds it with ctypes and mirrors the
reference's executor interface (/root/reference/proj/include/ditsim/execute.hpp)
so tests read like the reference's own:

    ctx = ToyDiTCuda(seed, layers, hidden_size, heads, mlp_ratio, seq_len, workers)
    res = ctx.run_pipefusion(x_init, steps, patches, warmup, eta)
    res.final_x, res.stats.fresh_patch_reads, ...

There is no CPU fallback: importing works without a GPU, but every compute
call goes through the CUDA library and raises if it is missing or fails.
"""
from __future__ import annotations

import ctypes
import math
import sys
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "LIB_PATH", "load_library", "ValidationError", "NumericError", "CudaError",
    "StalenessStats", "ParallelRunResult", "ToyDiTCuda", "EXPORTED_SYMBOLS",
    "mlp_hidden_of", "make_initial_latent", "KERNEL_KINDS", "PixArtCuda", "rank_plan",
    "PLAN_KINDS", "connect_ranks", "connect_distributed", "trace_json", "JointDiTCuda",
    "SerialResult", "AutoWarmupResult", "root_cause", "reset_distributed", "MMDiTCuda",
    "PRECISION_BF16", "PRECISION_FP32",
]

LIB_PATH = Path(__file__).resolve().parent / "libpipefusion_b200.so"

# Every symbol declared in include/pipefusion_b200.h and pipefusion_b200_debug.h.
EXPORTED_SYMBOLS = [
    "pf_create_toy", "pf_create", "pf_create_pixart", "pf_set_text", "pf_block_kind",
    "pf_layer_forward_t", "pf_destroy", "pf_last_error", "pf_create_toy_rank",
    "pf_create_pixart_rank", "pf_peer_blob_size", "pf_export_peer", "pf_connect_peers",
    "pf_rank", "pf_world", "pf_rank_plan", "pf_set_timeline", "pf_timeline",
    "pf_run_distrifusion", "pf_run_distrifusion_device", "pf_create_joint",
    "pf_create_joint_rank",
    "pf_run_pipefusion", "pf_run_pipefusion_device", "pf_synchronize",
    "pf_serial_reference", "pf_layer_forward", "pf_stage_count",
    "pf_stage_first_layer", "pf_stage_layer_count", "pf_last_launch_count",
    "pf_version", "pf_make_initial_latent", "pf_set_graphs", "pf_set_profiling", "pf_kernel_profile",
    "pf_debug_gemm", "pf_debug_attention", "pf_debug_attention_trace", "pf_debug_gemm_trace",
    "pf_debug_attention_ex",
    "pf_debug_attn_schedule", "pf_serial_reference_ex", "pf_auto_warmup", "pf_divergence",
    "pf_rank_reset", "pf_rank_broken", "pf_connect_world", "pf_device_count", "pf_debug_fail_at",
    "pf_debug_poison_layer", "pf_create_toy_ex", "pf_create_toy_rank_ex", "pf_precision_of",
    "pf_create_mmdit", "pf_create_mmdit_rank", "pf_stage_param_bytes", "pf_stage_kv_bytes",
    "pf_prepare_pipefusion_device",
]

KERNEL_KINDS = ["gemm_qkv", "attention", "gemm_out_proj", "gemm_mlp_in", "gemm_mlp_out",
                "sampler", "gemm_cross_q", "cross_attention", "gemm_cross_out", "conditioning"]

PF_OK, PF_NUMERIC, PF_VALIDATION, PF_CUDA = 0, 1, 2, 3
PF_ROW_MAJOR, PF_COL_MAJOR = 0, 1


PRECISION_BF16 = 0  # pf_precision (include/pipefusion_b200.h)
PRECISION_FP32 = 1


class ValidationError(ValueError):
    """ditsim::ValidationError (model.hpp:27-30); CLI exit code 2."""


class NumericError(ArithmeticError):
    """ditsim::NumericError (model.hpp:32-36); CLI exit code 1."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the library."""


class _Desc(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int), ("hidden_size", ctypes.c_int),
                ("heads", ctypes.c_int), ("mlp_hidden", ctypes.c_int),
                ("seq_len", ctypes.c_int64)]


class _Stats(ctypes.Structure):
    _fields_ = [("fresh_patch_reads", ctypes.c_int64),
                ("stale_patch_reads", ctypes.c_int64),
                ("fresh_fraction", ctypes.POINTER(ctypes.c_double)),
                ("fresh_fraction_capacity", ctypes.c_int64)]


_lib: Optional[ctypes.CDLL] = None


def load_library(path: Optional[Path] = None) -> ctypes.CDLL:
    """Load (once) and type the C ABI. Raises if the library is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise CudaError(f"{p} not built: run `python __graft_entry__.py build` "
                        "(or paper_2405_14430_b200/_build.py)")
    lib = ctypes.CDLL(str(p))
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    dptr = ctypes.POINTER(ctypes.c_double)
    lib.pf_create_toy.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc),
                                  ctypes.POINTER(i32), i32, ctypes.POINTER(vp)]
    lib.pf_create.argtypes = [ctypes.POINTER(_Desc), ctypes.POINTER(dptr), dptr, i32,
                              ctypes.POINTER(i32), i32, ctypes.POINTER(vp)]
    lib.pf_create_pixart.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32,
                                     ctypes.POINTER(i32), i32, ctypes.POINTER(vp)]
    lib.pf_set_text.argtypes = [vp, dptr, i64, i32]
    lib.pf_create_joint.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32, i32,
                                    ctypes.POINTER(i32), i32, ctypes.POINTER(vp)]
    lib.pf_create_joint_rank.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32, i32, i32,
                                         i32, i32, ctypes.POINTER(vp)]
    lib.pf_block_kind.argtypes = [vp]
    lib.pf_create_mmdit.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32, i32, i32,
                                    ctypes.POINTER(i32), i32, ctypes.POINTER(vp)]
    lib.pf_create_mmdit_rank.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32, i32, i32,
                                         i32, i32, i32, ctypes.POINTER(vp)]
    lib.pf_stage_param_bytes.argtypes = [vp]
    lib.pf_stage_param_bytes.restype = ctypes.c_size_t
    lib.pf_stage_kv_bytes.argtypes = [vp]
    lib.pf_stage_kv_bytes.restype = ctypes.c_size_t
    lib.pf_layer_forward_t.argtypes = [vp, i32, i32, i32, dptr, i64, i64, dptr, dptr, i32]
    lib.pf_create_toy_rank.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32, i32, i32,
                                       ctypes.POINTER(vp)]
    lib.pf_create_toy_ex.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32,
                                     ctypes.POINTER(i32), i32, ctypes.POINTER(vp)]
    lib.pf_create_toy_rank_ex.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32, i32,
                                          i32, i32, ctypes.POINTER(vp)]
    lib.pf_precision_of.argtypes = [vp]
    lib.pf_create_pixart_rank.argtypes = [ctypes.c_uint64, ctypes.POINTER(_Desc), i32, i32,
                                          i32, i32, ctypes.POINTER(vp)]
    lib.pf_serial_reference_ex.argtypes = [vp, dptr, i32, i32, dbl, dptr, dptr]
    lib.pf_auto_warmup.argtypes = [vp, dptr, i32, i32, dbl, dbl, ctypes.POINTER(i32),
                                   ctypes.POINTER(i32)]
    lib.pf_divergence.argtypes = [vp, dptr, i64, i64, dptr, i64, i64, dptr]
    lib.pf_rank_reset.argtypes = [vp]
    lib.pf_rank_broken.argtypes = [vp]
    lib.pf_debug_fail_at.argtypes = [vp, i32]
    lib.pf_debug_poison_layer.argtypes = [vp, i32]
    lib.pf_peer_blob_size.restype = ctypes.c_size_t
    lib.pf_export_peer.argtypes = [vp, vp, ctypes.c_size_t]
    lib.pf_connect_peers.argtypes = [vp, vp, vp]
    lib.pf_connect_world.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p), i32]
    lib.pf_rank.argtypes = [vp]
    lib.pf_world.argtypes = [vp]
    lib.pf_rank_plan.argtypes = [i32, i32, i32, i32, i32, i64, ctypes.POINTER(ctypes.c_int32),
                                 i64]
    lib.pf_rank_plan.restype = i64
    lib.pf_run_distrifusion.argtypes = [vp, dptr, i32, i32, i32, i32, dbl, dptr,
                                        ctypes.POINTER(_Stats)]
    lib.pf_run_distrifusion_device.argtypes = [vp, vp, i32, i32, i32, dbl, vp,
                                               ctypes.POINTER(_Stats)]
    lib.pf_set_timeline.argtypes = [vp, i32]
    lib.pf_timeline.argtypes = [vp, dptr, i64]
    lib.pf_timeline.restype = i64
    lib.pf_destroy.argtypes = [vp]
    lib.pf_destroy.restype = None
    lib.pf_last_error.argtypes = [vp]
    lib.pf_last_error.restype = ctypes.c_char_p
    lib.pf_run_pipefusion.argtypes = [vp, dptr, i32, i32, i32, i32, dbl, dptr,
                                      ctypes.POINTER(_Stats)]
    lib.pf_run_pipefusion_device.argtypes = [vp, vp, i32, i32, i32, dbl, vp,
                                             ctypes.POINTER(_Stats)]
    lib.pf_synchronize.argtypes = [vp, vp]
    lib.pf_prepare_pipefusion_device.argtypes = [vp, vp, i32, i32, i32, dbl, vp]
    lib.pf_serial_reference.argtypes = [vp, dptr, i32, i32, dbl, dptr]
    lib.pf_layer_forward.argtypes = [vp, i32, dptr, i64, i64, dptr, dptr, i32]
    for name in ("pf_stage_count",):
        getattr(lib, name).argtypes = [vp]
    lib.pf_stage_first_layer.argtypes = [vp, i32]
    lib.pf_stage_layer_count.argtypes = [vp, i32]
    lib.pf_last_launch_count.argtypes = [vp]
    lib.pf_last_launch_count.restype = i64
    lib.pf_version.restype = ctypes.c_char_p
    lib.pf_make_initial_latent.argtypes = [ctypes.c_uint64, i64, i32, dptr]
    lib.pf_set_profiling.argtypes = [vp, i32]
    lib.pf_set_graphs.argtypes = [vp, i32]
    lib.pf_kernel_profile.argtypes = [vp, i32, dptr, ctypes.POINTER(i64), dptr, dptr]
    lib.pf_debug_gemm.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp]
    lib.pf_debug_attention.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp]
    lib.pf_debug_attention_trace.argtypes = [i32, vp]
    lib.pf_debug_attention_ex.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, i32]
    lib.pf_debug_gemm_trace.argtypes = [i32, vp]
    lib.pf_debug_attn_schedule.argtypes = [i32, i32, i32, i32, i32, ctypes.POINTER(ctypes.c_longlong)]
    if path is None:
        _lib = lib
    return lib


def _raise(status: int, msg: str) -> None:
    if status == PF_OK:
        return
    if status == PF_VALIDATION:
        raise ValidationError(msg)
    if status == PF_NUMERIC:
        raise NumericError(msg)
    raise CudaError(msg)


def mlp_hidden_of(hidden_size: int, mlp_ratio: float) -> int:
    """int(std::lround(mlp_ratio * hidden_size)) as in toy_model.cpp:56."""
    v = mlp_ratio * hidden_size
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def make_initial_latent(seed: int, seq_len: int, hidden_size: int) -> np.ndarray:
    """ditsim::make_initial_latent (execute.hpp:56-57), host, bit-exact."""
    lib = load_library()
    out = np.empty((seq_len, hidden_size), dtype=np.float64)
    _raise(lib.pf_make_initial_latent(ctypes.c_uint64(seed), seq_len, hidden_size,
                                      _dptr(out)), lib.pf_last_error(None).decode())
    return out


@dataclass
class StalenessStats:
    """ditsim::StalenessStats (execute.hpp:108-114)."""
    fresh_patch_reads: int = 0
    stale_patch_reads: int = 0
    per_worker_fresh_fraction: List[List[float]] = field(default_factory=list)


@dataclass
class SerialResult:
    """ditsim::SerialResult (execute.hpp:93-98): trajectory[0] is the initial
    latent, trajectory[k] the latent after k update steps."""
    final_x: np.ndarray
    trajectory: List[np.ndarray] = field(default_factory=list)
    timestep: int = -1


@dataclass
class AutoWarmupResult:
    """ditsim::AutoWarmupResult (execute.hpp:139-142)."""
    warmup: int = 0
    threshold_met: bool = False


_NONFINITE = "non-finite activation at timestep "
_CLOSED = "channel closed mid-run"


def root_cause(errors: Sequence[Optional[BaseException]]) -> Optional[BaseException]:
    """The error a failed multi-rank run reports, given each rank's error in
    rank order (None = that rank succeeded): the reference prefers a root
    cause over the "channel closed mid-run" cascade (execute.cpp:357-374).
    Ranks here detect non-finite activations after the run, so a NaN that
    travelled on to later stages is reported by several ranks: the earliest
    in execution order (highest timestep, then lowest layer) is the root."""
    first = next((e for e in errors if e is not None), None)
    roots = [e for e in errors if e is not None and not str(e).startswith(_CLOSED)]
    if not roots:
        return first
    nonfinite = []
    for e in roots:
        m = str(e)
        if isinstance(e, NumericError) and m.startswith(_NONFINITE):
            try:
                t, layer = m[len(_NONFINITE):].split(", layer ")
                nonfinite.append((-int(t), int(layer), e))
            except ValueError:
                pass
    parsed = {id(v[2]) for v in nonfinite}
    others = [e for e in roots if id(e) not in parsed]
    if others:  # a failure other than a travelling NaN: first in rank order
        return others[0]
    return min(nonfinite, key=lambda v: v[:2])[2]


@dataclass
class ParallelRunResult:
    """ditsim::ParallelRunResult (execute.hpp:116-119); final timestep is -1."""
    final_x: np.ndarray
    stats: StalenessStats
    timestep: int = -1


def _f64c(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _out_buffer(x: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
    """Result latent for a host-buffer run: the caller's `out` (float64,
    C-contiguous, x's shape; reusing one array across runs avoids the
    first-touch page faults of a fresh 37 MB array, ~5 ms at C2) or a new
    array. The library never keeps or reuses a returned array itself."""
    if out is None:
        return np.empty_like(x)
    if (not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != x.shape
            or not out.flags.c_contiguous or not out.flags.writeable):
        raise ValidationError("out must be a writeable C-contiguous float64 array of the "
                              "latent's shape")
    return out


class ToyDiTCuda:
    """A toy DiT resident on B200 stage devices, split into `workers` stages.

    Weights come from `seed` exactly as build_toy_model does
    (toy_model.cpp:44-82), or from explicit fp64 matrices via `from_weights`.
    """

    def __init__(self, seed: int, layers: int, hidden_size: int, heads: int,
                 mlp_ratio: float, seq_len: int, workers: int = 1,
                 devices: Optional[Sequence[int]] = None, _weights=None, _text_tokens=0,
                 _rank=None, _joint=None, precision: int = 0, _mmdit=None):
        """precision: PRECISION_BF16 (the product path) or PRECISION_FP32
        (parity mode: fp32 CUDA-core kernels, same executor; toy block)."""
        self._lib = load_library()
        self._ctx = ctypes.c_void_p()
        self.layers, self.hidden_size, self.heads = layers, hidden_size, heads
        self.mlp_hidden = mlp_hidden_of(hidden_size, mlp_ratio)
        self.seq_len, self.workers = seq_len, workers
        desc = _Desc(layers, hidden_size, heads, self.mlp_hidden, seq_len)
        self.rank, self.world = 0, 1
        if _rank is not None:
            # rank mode: this context holds stage `rank` of `workers` on `device`
            rank, device = _rank
            self.rank, self.world = rank, workers
            if _mmdit is not None:
                st = self._lib.pf_create_mmdit_rank(ctypes.c_uint64(seed), ctypes.byref(desc),
                                                    _text_tokens, _mmdit[0], _mmdit[1], rank,
                                                    workers, device, ctypes.byref(self._ctx))
            elif _joint is not None:
                st = self._lib.pf_create_joint_rank(ctypes.c_uint64(seed), ctypes.byref(desc),
                                                    _text_tokens, _joint, rank, workers, device,
                                                    ctypes.byref(self._ctx))
            elif _text_tokens:
                st = self._lib.pf_create_pixart_rank(ctypes.c_uint64(seed), ctypes.byref(desc),
                                                     _text_tokens, rank, workers, device,
                                                     ctypes.byref(self._ctx))
            else:
                st = self._lib.pf_create_toy_rank_ex(ctypes.c_uint64(seed), ctypes.byref(desc),
                                                     precision, rank, workers, device,
                                                     ctypes.byref(self._ctx))
            if st != PF_OK:
                _raise(st, self._lib.pf_last_error(None).decode())
            return
        devs = list(devices) if devices is not None else [0] * workers
        if len(devs) != workers:
            raise ValidationError("devices must list one CUDA device per worker")
        dev_arr = (ctypes.c_int * max(1, workers))(*devs)
        if _mmdit is not None:
            st = self._lib.pf_create_mmdit(ctypes.c_uint64(seed), ctypes.byref(desc),
                                           _text_tokens, _mmdit[0], _mmdit[1], dev_arr, workers,
                                           ctypes.byref(self._ctx))
        elif _joint is not None:
            st = self._lib.pf_create_joint(ctypes.c_uint64(seed), ctypes.byref(desc),
                                           _text_tokens, _joint, dev_arr, workers,
                                           ctypes.byref(self._ctx))
        elif _text_tokens:
            st = self._lib.pf_create_pixart(ctypes.c_uint64(seed), ctypes.byref(desc),
                                            _text_tokens, dev_arr, workers,
                                            ctypes.byref(self._ctx))
        elif _weights is None:
            st = self._lib.pf_create_toy_ex(ctypes.c_uint64(seed), ctypes.byref(desc),
                                            precision, dev_arr, workers,
                                            ctypes.byref(self._ctx))
        else:
            mats, cb = _weights
            keep = [_f64c(m) for m in mats]
            ptrs = (ctypes.POINTER(ctypes.c_double) * len(keep))(*[_dptr(m) for m in keep])
            cbc = _f64c(cb)
            st = self._lib.pf_create(ctypes.byref(desc), ptrs, _dptr(cbc), PF_ROW_MAJOR,
                                     dev_arr, workers, ctypes.byref(self._ctx))
        if st != PF_OK:
            _raise(st, self._lib.pf_last_error(None).decode())

    @classmethod
    def rank_stage(cls, seed: int, layers: int, hidden_size: int, heads: int, mlp_ratio: float,
                   seq_len: int, rank: int, world: int, device: int = 0,
                   precision: int = 0) -> "ToyDiTCuda":
        """One process (or context) per stage: stage `rank` of `world` on
        `device` (the reference's worker thread d of run_pipefusion_threads).
        Connect the ranks with connect_ranks / connect_distributed."""
        obj = cls.__new__(cls)
        ToyDiTCuda.__init__(obj, seed, layers, hidden_size, heads, mlp_ratio, seq_len, world,
                            None, _rank=(rank, device), precision=precision)
        return obj

    def export_peer(self) -> bytes:
        buf = ctypes.create_string_buffer(int(self._lib.pf_peer_blob_size()))
        _raise(self._lib.pf_export_peer(self._ctx, buf, len(buf)), self._err())
        return buf.raw

    def connect_peers(self, pred: bytes, succ: bytes) -> None:
        _raise(self._lib.pf_connect_peers(self._ctx, pred, succ), self._err())

    def connect_world(self, blobs: Sequence[bytes]) -> None:
        """Connect to the neighbours and open every rank's signal page
        (pf_connect_world): a failing rank then closes the run for all."""
        arr = (ctypes.c_char_p * len(blobs))(*blobs)
        _raise(self._lib.pf_connect_world(self._ctx, arr, len(blobs)), self._err())

    @classmethod
    def from_weights(cls, layer_mats, condition_bias, heads: int, seq_len: int,
                     workers: int = 1, devices=None) -> "ToyDiTCuda":
        """layer_mats: per layer (w_q, w_k, w_v, w_o, w_mlp_in, w_mlp_out) fp64."""
        flat = [m for layer in layer_mats for m in layer]
        hs = int(np.asarray(flat[0]).shape[0])
        mlp = int(np.asarray(flat[4]).shape[1])
        obj = cls.__new__(cls)
        cls.__init__(obj, 0, len(layer_mats), hs, heads, mlp / hs, seq_len, workers,
                     devices, _weights=(flat, condition_bias))
        return obj

    # ---------------------------------------------------------------- lifecycle
    def close(self) -> None:
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.pf_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _err(self) -> str:
        return self._lib.pf_last_error(self._ctx).decode()

    # ---------------------------------------------------------------- stages
    def stage_layers(self) -> List[range]:
        n = self._lib.pf_stage_count(self._ctx)
        out = []
        for d in range(n):
            f = self._lib.pf_stage_first_layer(self._ctx, d)
            c = self._lib.pf_stage_layer_count(self._ctx, d)
            out.append(range(f, f + c))
        return out

    def param_bytes(self) -> int:
        """Device bytes of this context's parameters (pf_stage_param_bytes)."""
        return int(self._lib.pf_stage_param_bytes(self._ctx))

    def kv_bytes(self) -> int:
        """Device bytes of this context's K/V buffers (pf_stage_kv_bytes)."""
        return int(self._lib.pf_stage_kv_bytes(self._ctx))

    @property
    def precision(self) -> int:
        """PRECISION_BF16 or PRECISION_FP32 (pf_precision_of)."""
        return int(self._lib.pf_precision_of(self._ctx))

    def last_launch_count(self) -> int:
        return int(self._lib.pf_last_launch_count(self._ctx))

    # ---------------------------------------------------------------- runs
    def _rank_status(self, status: int) -> None:
        """Raise this rank's error; with a process group attached
        (connect_distributed), every rank raises the run's root cause
        (root_cause) so all ranks report the same failure."""
        group = getattr(self, "_group", False)  # set by connect_distributed
        if self.world <= 1 or group is False:
            _raise(status, self._err())
            return
        import torch.distributed as dist
        mine = None if status == PF_OK else (status, self._err())
        allv = [None] * self.world
        dist.all_gather_object(allv, mine, group=group)
        errs = []
        for v in allv:
            if v is None:
                errs.append(None)
                continue
            try:
                _raise(*v)
            except Exception as e:  # noqa: BLE001 - rebuilt per rank
                errs.append(e)
        err = root_cause(errs)
        if err is not None:
            raise err

    def run_pipefusion(self, x_init, steps: int, patches: int, warmup: int,
                       eta: float, out: Optional[np.ndarray] = None) -> ParallelRunResult:
        """ditsim::run_pipefusion (execute.hpp:124-127) on the GPU stages.
        `out`: optional float64 array receiving the final latent."""
        per = max(0, patches * (steps - warmup))
        stages = 1 if self.world > 1 else self.workers
        cap = stages * per
        ff = (ctypes.c_double * max(1, cap))()
        st = _Stats(0, 0, ff, cap)
        if self.rank > 0:
            # rank mode, not rank 0: the latent lives on rank 0
            status = self._lib.pf_run_pipefusion(self._ctx, None, PF_ROW_MAJOR, steps, patches,
                                                 warmup, ctypes.c_double(eta), None,
                                                 ctypes.byref(st))
            self._rank_status(status)
            return ParallelRunResult(None, StalenessStats(st.fresh_patch_reads,
                                                          st.stale_patch_reads,
                                                          [list(ff[:per])]))
        x = _f64c(x_init)
        if x.shape != (self.seq_len, self.hidden_size):
            raise ValidationError("latent width does not match the model hidden size")
        out = _out_buffer(x, out)
        status = self._lib.pf_run_pipefusion(self._ctx, _dptr(x), PF_ROW_MAJOR, steps,
                                             patches, warmup, ctypes.c_double(eta),
                                             _dptr(out), ctypes.byref(st))
        self._rank_status(status)
        fr = [list(ff[d * per:(d + 1) * per]) for d in range(stages)]
        return ParallelRunResult(out, StalenessStats(st.fresh_patch_reads,
                                                     st.stale_patch_reads, fr))

    def run_distrifusion(self, x_init, steps: int, workers: int, warmup: int,
                         eta: float) -> ParallelRunResult:
        """ditsim::run_distrifusion (execute.hpp:131-133) on this context's GPU."""
        x = _f64c(x_init)
        out = _out_buffer(x)
        per = max(0, steps - warmup)
        cap = workers * per
        ff = (ctypes.c_double * max(1, cap))()
        st = _Stats(0, 0, ff, cap)
        status = self._lib.pf_run_distrifusion(self._ctx, _dptr(x), PF_ROW_MAJOR, steps,
                                               workers, warmup, ctypes.c_double(eta),
                                               _dptr(out), ctypes.byref(st))
        _raise(status, self._err())
        fr = [list(ff[w * per:(w + 1) * per]) for w in range(workers)]
        return ParallelRunResult(out, StalenessStats(st.fresh_patch_reads,
                                                     st.stale_patch_reads, fr))

    def serial_reference(self, x_init, steps: int, eta: float, keep_trajectory: bool = False):
        """ditsim::serial_reference (execute.hpp:102-104) on the GPU: the final
        latent, or with keep_trajectory a SerialResult holding the S + 1
        latents of the trajectory (pf_serial_reference_ex)."""
        x = _f64c(x_init)
        out = _out_buffer(x)
        if not keep_trajectory:
            status = self._lib.pf_serial_reference(self._ctx, _dptr(x), PF_ROW_MAJOR, steps,
                                                   ctypes.c_double(eta), _dptr(out))
            _raise(status, self._err())
            return out
        traj = np.empty((max(steps, 0) + 1,) + x.shape)
        status = self._lib.pf_serial_reference_ex(self._ctx, _dptr(x), PF_ROW_MAJOR, steps,
                                                  ctypes.c_double(eta), _dptr(out),
                                                  _dptr(traj))
        _raise(status, self._err())
        return SerialResult(out, list(traj))

    def auto_warmup(self, x_init, steps: int, eta: float, threshold: float) -> AutoWarmupResult:
        """ditsim::auto_warmup (execute.hpp:141-147) on the GPU."""
        x = _f64c(x_init)
        w, met = ctypes.c_int(0), ctypes.c_int(0)
        status = self._lib.pf_auto_warmup(self._ctx, _dptr(x), PF_ROW_MAJOR, steps,
                                          ctypes.c_double(eta), ctypes.c_double(threshold),
                                          ctypes.byref(w), ctypes.byref(met))
        _raise(status, self._err())
        return AutoWarmupResult(w.value, bool(met.value))

    def divergence(self, a, b) -> float:
        """ditsim::divergence (execute.hpp:136-137): ||a - b|| / ||b||, fp64 on the GPU."""
        a, b = _f64c(a), _f64c(b)
        a2 = a.reshape(a.shape[0], -1) if a.ndim else a.reshape(1, 1)
        b2 = b.reshape(b.shape[0], -1) if b.ndim else b.reshape(1, 1)
        out = ctypes.c_double()
        status = self._lib.pf_divergence(self._ctx, _dptr(a2), a2.shape[0], a2.shape[1],
                                         _dptr(b2), b2.shape[0], b2.shape[1], ctypes.byref(out))
        _raise(status, self._err())
        return out.value

    # ---------------------------------------------------------------- rank mode
    def rank_reset(self) -> None:
        """Reopen a pipeline the watchdog closed (pf_rank_reset); call on every
        rank between two host barriers (reset_distributed does that)."""
        _raise(self._lib.pf_rank_reset(self._ctx), self._err())

    @property
    def rank_broken(self) -> bool:
        return bool(self._lib.pf_rank_broken(self._ctx))

    def debug_fail_at(self, op: int) -> None:
        """Test hook: this rank's next runs throw at plan op `op` (-1: off)."""
        _raise(self._lib.pf_debug_fail_at(self._ctx, op), self._err())

    def debug_poison_layer(self, layer: int) -> None:
        """Test hook: layer `layer`'s out-projection produces NaN."""
        _raise(self._lib.pf_debug_poison_layer(self._ctx, layer), self._err())

    def layer_forward(self, layer: int, h, k_buf, v_buf, row0: int):
        """ditsim::toy_layer_forward (execute.hpp:75-77); returns (h, k, v)."""
        h = _f64c(h).copy()
        k = _f64c(k_buf).copy()
        v = _f64c(v_buf).copy()
        status = self._lib.pf_layer_forward(self._ctx, layer, _dptr(h), h.shape[0], row0,
                                            _dptr(k), _dptr(v), PF_ROW_MAJOR)
        _raise(status, self._err())
        return h, k, v

    def run_distrifusion_device(self, x_dev_ptr: int, steps: int, workers: int,
                                warmup: int, eta: float, stream_ptr: int = 0) -> StalenessStats:
        """Enqueue a DistriFusion run on a device fp32 latent (in place); asynchronous."""
        st = _Stats(0, 0, None, 0)
        status = self._lib.pf_run_distrifusion_device(
            self._ctx, ctypes.c_void_p(x_dev_ptr), steps, workers, warmup,
            ctypes.c_double(eta), ctypes.c_void_p(stream_ptr), ctypes.byref(st))
        _raise(status, self._err())
        return StalenessStats(st.fresh_patch_reads, st.stale_patch_reads, [])

    def run_pipefusion_device(self, x_dev_ptr: int, steps: int, patches: int,
                              warmup: int, eta: float, stream_ptr: int = 0) -> StalenessStats:
        """Enqueue a run on a device fp32 latent (in place); asynchronous."""
        st = _Stats(0, 0, None, 0)
        status = self._lib.pf_run_pipefusion_device(
            self._ctx, ctypes.c_void_p(x_dev_ptr), steps, patches, warmup,
            ctypes.c_double(eta), ctypes.c_void_p(stream_ptr), ctypes.byref(st))
        _raise(status, self._err())
        return StalenessStats(st.fresh_patch_reads, st.stale_patch_reads, [])

    def prepare_pipefusion_device(self, x_dev_ptr: int, steps: int, patches: int, warmup: int,
                                  eta: float, stream_ptr: int = 0) -> None:
        """Rank mode: build this rank's CUDA graph for these arguments without
        running it (pf_prepare_pipefusion_device); call on every rank before
        the first run when ranks share a device in one process."""
        _raise(self._lib.pf_prepare_pipefusion_device(
            self._ctx, ctypes.c_void_p(x_dev_ptr or None), steps, patches, warmup,
            ctypes.c_double(eta), ctypes.c_void_p(stream_ptr or None)), self._err())

    def set_graphs(self, enabled: bool) -> None:
        self._lib.pf_set_graphs(self._ctx, 1 if enabled else 0)

    def set_profiling(self, enabled: bool) -> None:
        self._lib.pf_set_profiling(self._ctx, 1 if enabled else 0)

    def kernel_profile(self) -> dict:
        """Per kernel kind of the last profiled run: ms, launches, flops, bytes."""
        out = {}
        for kind, name in enumerate(KERNEL_KINDS):
            ms, fl, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            n = ctypes.c_int64()
            _raise(self._lib.pf_kernel_profile(self._ctx, kind, ctypes.byref(ms),
                                               ctypes.byref(n), ctypes.byref(fl),
                                               ctypes.byref(by)), self._err())
            out[name] = dict(ms=ms.value, launches=n.value, flops=fl.value, bytes=by.value)
        return out

    def set_timeline(self, enabled: bool) -> None:
        self._lib.pf_set_timeline(self._ctx, 1 if enabled else 0)

    def timeline(self) -> List[dict]:
        """Spans of the last run with the timeline enabled (pf_timeline)."""
        n = self._lib.pf_timeline(self._ctx, None, 0)
        if n < 0:
            raise CudaError(self._err())
        buf = np.zeros((max(n, 1), 6))
        self._lib.pf_timeline(self._ctx, _dptr(buf), n)
        return [dict(device=int(r[0]), stream="compute" if r[1] == 0 else "comm",
                     patch=None if r[2] < 0 else int(r[2]),
                     timestep=None if r[3] < 0 else int(r[3]), start_us=float(r[4]),
                     dur_us=float(r[5])) for r in buf[:n]]

    def synchronize(self, stream_ptr: int = 0) -> None:
        _raise(self._lib.pf_synchronize(self._ctx, ctypes.c_void_p(stream_ptr)), self._err())


class PixArtCuda(ToyDiTCuda):
    """The PixArt-alpha block variant under the same
    PipeFusion executor: adaLN-single modulation, LayerNorm folded through the
    GEMMs, self-attention over the stale/fresh K/V buffer, cross-attention over
    `text_tokens` text tokens, GELU(tanh) MLP. Parameters and text come from
    `seed` as oracle/px_oracle.c (pxo_build) specifies."""

    def __init__(self, seed: int, layers: int, hidden_size: int, heads: int,
                 mlp_ratio: float, seq_len: int, text_tokens: int, workers: int = 1,
                 devices: Optional[Sequence[int]] = None):
        if text_tokens < 1:
            raise ValidationError("PixArt block needs at least one text token")
        self.text_tokens = text_tokens
        super().__init__(seed, layers, hidden_size, heads, mlp_ratio, seq_len, workers,
                         devices, _text_tokens=text_tokens)

    @classmethod
    def rank_stage(cls, seed: int, layers: int, hidden_size: int, heads: int, mlp_ratio: float,
                   seq_len: int, text_tokens: int, rank: int, world: int,
                   device: int = 0) -> "PixArtCuda":
        obj = cls.__new__(cls)
        obj.text_tokens = text_tokens
        ToyDiTCuda.__init__(obj, seed, layers, hidden_size, heads, mlp_ratio, seq_len, world,
                            None, _text_tokens=text_tokens, _rank=(rank, device))
        return obj

    def set_text(self, y) -> None:
        y = _f64c(y)
        _raise(self._lib.pf_set_text(self._ctx, _dptr(y), y.shape[0], PF_ROW_MAJOR),
               self._err())

    def layer_forward_t(self, layer: int, t: int, steps: int, h, k_buf, v_buf, row0: int):
        """One PixArt block at timestep index t of a `steps`-step run; (h, k, v)."""
        h = _f64c(h).copy()
        k = _f64c(k_buf).copy()
        v = _f64c(v_buf).copy()
        status = self._lib.pf_layer_forward_t(self._ctx, layer, t, steps, _dptr(h), h.shape[0],
                                              row0, _dptr(k), _dptr(v), PF_ROW_MAJOR)
        _raise(status, self._err())
        return h, k, v


PLAN_KINDS = ["prepare", "compute", "send", "recv", "ack", "latent_update"]


def rank_plan(rank: int, world: int, steps: int, patches: int, warmup: int,
              seq_len: int) -> np.ndarray:
    """Op list of `rank` (include/pipefusion_b200.h pf_rank_plan): int32
    [n_ops x 8] = kind, t, patch, row0, rows, msg, overlap, flag. Host only."""
    lib = load_library()
    n = lib.pf_rank_plan(rank, world, steps, patches, warmup, seq_len, None, 0)
    if n < 0:
        raise ValidationError("invalid rank plan arguments")
    out = np.zeros((max(n, 1), 8), dtype=np.int32)
    lib.pf_rank_plan(rank, world, steps, patches, warmup, seq_len,
                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n)
    return out[:n]


def connect_ranks(stages: Sequence[ToyDiTCuda]) -> None:
    """Connect the rank-mode contexts of one process (stages[d] = rank d)."""
    blobs = [s.export_peer() for s in stages]
    for s in stages:
        s.connect_world(blobs)


def connect_distributed(stage: ToyDiTCuda, group=None, agree_on_errors: bool = True) -> None:
    """Connect this process's rank-mode context to its neighbours, exchanging
    peer blobs over torch.distributed (any backend; gloo is enough). With
    agree_on_errors, host-buffer runs (run_pipefusion) all-gather each rank's
    status afterwards and every rank raises the run's root cause."""
    import torch.distributed as dist
    blobs = [None] * stage.world
    dist.all_gather_object(blobs, stage.export_peer(), group=group)
    stage.connect_world(blobs)
    stage._group = group if agree_on_errors else False


def reset_distributed(stage: ToyDiTCuda, group=None) -> None:
    """Reopen a pipeline closed by a failed run: barrier, pf_rank_reset on
    every rank, barrier."""
    import torch.distributed as dist
    dist.barrier(group=group)
    stage.rank_reset()
    dist.barrier(group=group)


def trace_json(spans: Sequence[dict]) -> dict:
    """A measured timeline in the reference's trace format
    (timeline_to_trace_json, simulate.cpp:607-645): events sorted by start,
    device, stream, label; labels as simulate_pipefusion names them
    ("warmup t<t>", "stage t<t> p<j>", "send t<t>[ p<j>]")."""
    events = []
    for e in spans:
        t, j = e["timestep"], e["patch"]
        if e["stream"] == "compute":
            name = f"warmup t{t}" if j is None else f"stage t{t} p{j}"
        else:
            name = f"send t{t}" if j is None else f"send t{t} p{j}"
        events.append({"name": name, "device": e["device"], "stream": e["stream"],
                       "start_us": e["start_us"], "dur_us": e["dur_us"], "patch": j,
                       "timestep": t})
    events.sort(key=lambda ev: (ev["start_us"], ev["device"], ev["stream"] != "compute",
                                ev["name"]))
    makespan = max((ev["start_us"] + ev["dur_us"] for ev in events), default=0.0)
    return {"makespan_us": makespan, "events": events}


class JointDiTCuda(ToyDiTCuda):
    """SD3-style joint-attention (MMDiT double-stream) block with the toy
    block's arithmetic per stream: `text_tokens` text
    rows with their own weights share the K/V buffer with the image rows;
    under PipeFusion they re-enter every step with patch 0 (always fresh)."""

    def __init__(self, seed: int, layers: int, hidden_size: int, heads: int,
                 mlp_ratio: float, seq_len: int, text_tokens: int, workers: int = 1,
                 devices: Optional[Sequence[int]] = None, double_layers: Optional[int] = None):
        """double_layers: leading double-stream layers (default: all); the rest
        are Flux-style single-stream blocks."""
        if text_tokens < 1:
            raise ValidationError("joint block needs at least one text token")
        self.text_tokens = text_tokens
        self.double_layers = layers if double_layers is None else double_layers
        super().__init__(seed, layers, hidden_size, heads, mlp_ratio, seq_len, workers,
                         devices, _text_tokens=text_tokens, _joint=self.double_layers)

    @classmethod
    def rank_stage(cls, seed: int, layers: int, hidden_size: int, heads: int, mlp_ratio: float,
                   seq_len: int, text_tokens: int, rank: int, world: int, device: int = 0,
                   double_layers: Optional[int] = None) -> "JointDiTCuda":
        obj = cls.__new__(cls)
        obj.text_tokens = text_tokens
        obj.double_layers = layers if double_layers is None else double_layers
        ToyDiTCuda.__init__(obj, seed, layers, hidden_size, heads, mlp_ratio, seq_len, world,
                            None, _text_tokens=text_tokens, _rank=(rank, device),
                            _joint=obj.double_layers)
        return obj

    def set_text(self, y) -> None:
        y = _f64c(y)
        _raise(self._lib.pf_set_text(self._ctx, _dptr(y), y.shape[0], PF_ROW_MAJOR),
               self._err())


class MMDiTCuda(ToyDiTCuda):
    """MMDiT blocks (pf_create_mmdit): `double_layers` SD3 / Flux double-stream
    joint blocks, then Flux single-stream blocks; `rope` adds the Flux axial
    RoPE. Parameters and text tokens are generated on the device from `seed`
    (oracle/mmdit_oracle.py MMDiT holds the same values)."""

    def __init__(self, seed: int, layers: int, hidden_size: int, heads: int, mlp_ratio: float,
                 seq_len: int, text_tokens: int, workers: int = 1,
                 devices: Optional[Sequence[int]] = None, double_layers: Optional[int] = None,
                 rope: bool = False):
        self.text_tokens = text_tokens
        self.double_layers = layers if double_layers is None else double_layers
        self.rope = bool(rope)
        super().__init__(seed, layers, hidden_size, heads, mlp_ratio, seq_len, workers,
                         devices, _text_tokens=text_tokens,
                         _mmdit=(self.double_layers, int(self.rope)))

    @classmethod
    def rank_stage(cls, seed: int, layers: int, hidden_size: int, heads: int, mlp_ratio: float,
                   seq_len: int, text_tokens: int, rank: int, world: int, device: int = 0,
                   double_layers: Optional[int] = None, rope: bool = False) -> "MMDiTCuda":
        obj = cls.__new__(cls)
        obj.text_tokens = text_tokens
        obj.double_layers = layers if double_layers is None else double_layers
        obj.rope = bool(rope)
        ToyDiTCuda.__init__(obj, seed, layers, hidden_size, heads, mlp_ratio, seq_len, world,
                            None, _text_tokens=text_tokens, _rank=(rank, device),
                            _mmdit=(obj.double_layers, int(obj.rope)))
        return obj

    def set_text(self, y) -> None:
        """Replace the text tokens [text_tokens x hidden] (pf_set_text)."""
        y = _f64c(y)
        _raise(self._lib.pf_set_text(self._ctx, _dptr(y), y.shape[0], PF_ROW_MAJOR),
               self._err())
