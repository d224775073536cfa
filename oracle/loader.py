"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

* `Restatement`  -> oracle/libpf_oracle.so   (oracle/pf_oracle.c, plain C)
* `Reference`    -> oracle/_ref/libditsim_ref.so (the reference's own sources,
                    compiled by oracle/Makefile against oracle/shim/)

Both expose the same Pythonic surface (row-major float64 numpy arrays), so
tests can pin one against the other bit for bit. Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may use this module.
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path
from typing import List, Optional, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
RESTATEMENT_LIB = HERE / "libpf_oracle.so"
REFERENCE_LIB = HERE / "_ref" / "libditsim_ref.so"
REFERENCE_SRC = Path("/root/reference/proj")

_d = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_ip = ctypes.POINTER(ctypes.c_int)


def build(reference: bool = True, quiet: bool = True) -> None:
    """Compile the restatement, and the reference when its sources exist."""
    out = subprocess.DEVNULL if quiet else None
    subprocess.run(["make", "-C", str(HERE), "all"], check=True, stdout=out)
    if reference and REFERENCE_SRC.exists():
        subprocess.run(["make", "-C", str(HERE), "ref"], check=True, stdout=out)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_d)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # 1 numeric, 2 validation


class _Base:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (and `make -C oracle ref`)")
        self.lib = ctypes.CDLL(str(path))

    # model handles
    def build_toy_model(self, seed, layers, hs, heads, mlp_ratio=4.0) -> "Model":
        return Model(self, seed, layers, hs, heads, mlp_ratio)


class Model:
    """A ToyDiT held by one of the oracle libraries."""

    def __init__(self, owner: "_Base", seed, layers, hs, heads, mlp_ratio):
        self.o = owner
        err = ctypes.create_string_buffer(256)
        fn = getattr(owner.lib, owner.prefix + "build")
        fn.restype = ctypes.c_void_p
        fn.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                       ctypes.c_double, ctypes.c_char_p, ctypes.c_int]
        self.h = fn(seed, layers, hs, heads, mlp_ratio, err, 256)
        if not self.h:
            raise OracleError(2, err.value.decode())
        self.layers, self.hs, self.heads = layers, hs, heads
        mh = getattr(owner.lib, owner.prefix + "mlp_hidden")
        mh.argtypes = [ctypes.c_void_p]
        self.mlp = mh(self.h)

    def __del__(self):
        try:
            fn = getattr(self.o.lib, self.o.prefix + "free")
            fn.argtypes = [ctypes.c_void_p]
            fn(self.h)
        except Exception:
            pass

    def weights(self) -> Tuple[List[tuple], np.ndarray]:
        """Per layer (w_q, w_k, w_v, w_o, w_mlp_in, w_mlp_out) + condition_bias."""
        shapes = [(self.hs, self.hs)] * 4 + [(self.hs, self.mlp), (self.mlp, self.hs)]
        out = []
        for l in range(self.layers):
            mats = []
            for i, sh in enumerate(shapes):
                mats.append(self.o._weight(self.h, l, i, sh))
            out.append(tuple(mats))
        return out, self.o._cb(self.h, self.hs)

    def serial_reference(self, x, steps, eta):
        return self.o._serial(self, x, steps, eta)

    def run_pipefusion(self, x, steps, workers, patches, warmup, eta, **kw):
        return self.o._pipefusion(self, x, steps, workers, patches, warmup, eta, **kw)

    def layer_forward(self, layer, h, k, v, row0):
        return self.o._layer(self, layer, h, k, v, row0)

    def auto_warmup(self, x, steps, eta, threshold):
        return self.o._auto_warmup(self, x, steps, eta, threshold)


class _Impl(_Base):
    def _weight(self, h, l, i, shape):
        if self.prefix == "pfo_":
            fn = self.lib.pfo_weight
            fn.restype = _d
            fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
            ptr = fn(h, l, i)
            return np.ctypeslib.as_array(ptr, shape=shape).copy()
        out = np.empty(shape)
        self.lib.ref_weight.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _d]
        self.lib.ref_weight(h, l, i, _p(out))
        return out

    def _cb(self, h, hs):
        if self.prefix == "pfo_":
            fn = self.lib.pfo_condition_bias
            fn.restype = _d
            fn.argtypes = [ctypes.c_void_p]
            return np.ctypeslib.as_array(fn(h), shape=(hs,)).copy()
        out = np.empty(hs)
        self.lib.ref_condition_bias.argtypes = [ctypes.c_void_p, _d]
        self.lib.ref_condition_bias(h, _p(out))
        return out

    def make_initial_latent(self, seed, p, hs):
        out = np.empty((p, hs))
        if self.prefix == "pfo_":
            self.lib.pfo_latent.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, _d]
            self.lib.pfo_latent(seed, p, hs, _p(out))
        else:
            err = ctypes.create_string_buffer(256)
            self.lib.ref_latent.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, _d,
                                            ctypes.c_char_p, ctypes.c_int]
            rc = self.lib.ref_latent(seed, p, hs, _p(out), err, 256)
            if rc:
                raise OracleError(rc, err.value.decode())
        return out

    def _serial(self, m, x, steps, eta):
        x = _c(x)
        out = np.empty_like(x)
        err = ctypes.create_string_buffer(256)
        fn = getattr(self.lib, self.prefix + "serial")
        fn.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int, ctypes.c_double, _d,
                       ctypes.c_char_p, ctypes.c_int]
        rc = fn(m.h, _p(x), x.shape[0], steps, eta, _p(out), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def _pipefusion(self, m, x, steps, workers, patches, warmup, eta, backend="threads"):
        x = _c(x)
        out = np.empty_like(x)
        fresh = ctypes.c_int64()
        stale = ctypes.c_int64()
        per = max(0, patches * (steps - warmup))
        cap = workers * per
        ff = np.zeros(max(1, cap))
        err = ctypes.create_string_buffer(256)
        if self.prefix == "pfo_":
            fn = self.lib.pfo_pipefusion
            fn.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_double, _d, _i64p, _i64p, _d,
                           ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
            rc = fn(m.h, _p(x), x.shape[0], steps, workers, patches, warmup, eta, _p(out),
                    ctypes.byref(fresh), ctypes.byref(stale), _p(ff), cap, err, 256)
        else:
            fn = self.lib.ref_pipefusion
            fn.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, _d,
                           _i64p, _i64p, _d, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
            rc = fn(m.h, _p(x), x.shape[0], steps, workers, patches, warmup, eta,
                    1 if backend == "inline" else 0, _p(out), ctypes.byref(fresh),
                    ctypes.byref(stale), _p(ff), cap, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        fr = [list(ff[d * per:(d + 1) * per]) for d in range(workers)]
        return out, (fresh.value, stale.value, fr)

    def _layer(self, m, layer, h, k, v, row0):
        h, k, v = _c(h).copy(), _c(k).copy(), _c(v).copy()
        fn = getattr(self.lib, self.prefix + "layer_forward")
        fn.argtypes = [ctypes.c_void_p, ctypes.c_int, _d, ctypes.c_int64, _d, _d,
                       ctypes.c_int64, ctypes.c_int64]
        fn(m.h, layer, _p(h), h.shape[0], _p(k), _p(v), k.shape[0], row0)
        return h, k, v

    def _auto_warmup(self, m, x, steps, eta, threshold):
        x = _c(x)
        w = ctypes.c_int()
        met = ctypes.c_int()
        fn = getattr(self.lib, self.prefix + "auto_warmup")
        fn.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                       ctypes.c_double, _ip, _ip]
        fn(m.h, _p(x), x.shape[0], steps, eta, threshold, ctypes.byref(w), ctypes.byref(met))
        return w.value, bool(met.value)

    def divergence(self, a, b) -> float:
        a, b = _c(a), _c(b)
        fn = getattr(self.lib, self.prefix + "divergence")
        fn.restype = ctypes.c_double
        fn.argtypes = [_d, _d, ctypes.c_int64, ctypes.c_int64]
        return fn(_p(a), _p(b), a.shape[0], a.shape[1])

    def schedule(self, n, m, steps, warmup):
        """Grid as (patch, timestep, kind) arrays of shape [slots, devices]."""
        cap = (warmup * n * m + (steps - warmup) * max(m, n) + m + n) * n + 1
        pa = np.zeros(cap, dtype=np.int32)
        ts = np.zeros(cap, dtype=np.int32)
        kd = np.zeros(cap, dtype=np.int32)
        ws = ctypes.c_int()
        ss = ctypes.c_int()
        fn = getattr(self.lib, self.prefix + "schedule")
        fn.argtypes = [ctypes.c_int] * 4 + [_ip, _ip, _ip, ctypes.c_int, _ip, _ip]
        ip = lambda a: a.ctypes.data_as(_ip)
        cells = fn(n, m, steps, warmup, ip(pa), ip(ts), ip(kd), cap, ctypes.byref(ws),
                   ctypes.byref(ss))
        slots = cells // n
        sh = (slots, n)
        return (pa[:cells].reshape(sh), ts[:cells].reshape(sh), kd[:cells].reshape(sh),
                ws.value, ss.value)

    def fresh_series(self, n, m, steps, warmup):
        cap = (warmup * n * m + (steps - warmup) * max(m, n) + m + n) + 1
        out = np.zeros(cap)
        fn = getattr(self.lib, self.prefix + "fresh_series")
        fn.argtypes = [ctypes.c_int] * 4 + [_d, ctypes.c_int]
        k = fn(n, m, steps, warmup, _p(out), cap)
        return out[:k]


class Restatement(_Impl):
    prefix = "pfo_"

    def __init__(self, path: Optional[Path] = None):
        super().__init__(path or RESTATEMENT_LIB)


def simulate_pipefusion(layers, hs, heads, seq_len, steps, warmup, devices, patches,
                        device_flops, link_bandwidth, link_latency=0.0, mlp_ratio=4.0,
                        bytes_per_element=2, per_message_overhead_s=50e-6):
    """The reference's own PipeFusion cost model (simulate.cpp:263-342) and
    trace JSON (timeline_to_trace_json): (makespan_s, trace dict)."""
    import json
    lib = ctypes.CDLL(str(REFERENCE_LIB))
    fn = lib.ref_simulate_pipefusion
    fn.restype = ctypes.c_longlong
    fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                   ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                   ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, _d,
                   ctypes.c_char_p, ctypes.c_longlong, ctypes.c_char_p, ctypes.c_int]
    mk = ctypes.c_double()
    err = ctypes.create_string_buffer(256)
    args = (layers, hs, heads, mlp_ratio, bytes_per_element, seq_len, steps, warmup, devices,
            patches, device_flops, link_bandwidth, link_latency, per_message_overhead_s)
    n = fn(*args, ctypes.byref(mk), None, 0, err, 256)
    if n < 0:
        raise OracleError(int(-n), err.value.decode())
    buf = ctypes.create_string_buffer(int(n) + 1)
    fn(*args, ctypes.byref(mk), buf, n + 1, err, 256)
    return mk.value, json.loads(buf.value.decode())


class Reference(_Impl):
    prefix = "ref_"

    def __init__(self, path: Optional[Path] = None):
        super().__init__(path or REFERENCE_LIB)

    def run_distrifusion(self, m, x, steps, workers, warmup, eta, backend="threads",
                         with_stats=False):
        x = _c(x)
        out = np.empty_like(x)
        err = ctypes.create_string_buffer(256)
        if with_stats:
            per = max(0, steps - warmup)
            ff = np.zeros(max(1, workers * per))
            fresh, stale = ctypes.c_int64(), ctypes.c_int64()
            fn = self.lib.ref_distrifusion_stats
            fn.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_double, ctypes.c_int, _d, _i64p, _i64p, _d,
                           ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
            rc = fn(m.h, _p(x), x.shape[0], steps, workers, warmup, eta,
                    1 if backend == "inline" else 0, _p(out), ctypes.byref(fresh),
                    ctypes.byref(stale), _p(ff), workers * per, err, 256)
            if rc:
                raise OracleError(rc, err.value.decode())
            return out, (fresh.value, stale.value,
                         [list(ff[w * per:(w + 1) * per]) for w in range(workers)])
        fn = self.lib.ref_distrifusion
        fn.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                       ctypes.c_int, ctypes.c_double, ctypes.c_int, _d, ctypes.c_char_p,
                       ctypes.c_int]
        rc = fn(m.h, _p(x), x.shape[0], steps, workers, warmup, eta,
                1 if backend == "inline" else 0, _p(out), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out


# ---------------------------------------------------------------- PixArt block
PXO_PARAMS = ["wqkv", "bqkv", "wo", "bo", "wqc", "bqc", "wkc", "bkc", "wvc", "bvc", "woc",
              "boc", "w1", "b1", "w2", "b2", "sst"]
PXO_GLOBALS = ["wt1", "bt1", "wt2", "bt2", "wt0", "bt0", "cb", "y"]


class PixArtOracle:
    """fp64 PixArt-alpha block variant under the reference schedule
    (oracle/px_oracle.c). Row-major float64 numpy in and out."""

    def __init__(self, seed, layers, hs, heads, mlp_ratio, text_tokens,
                 path: Optional[Path] = None):
        p = path or RESTATEMENT_LIB
        if not p.exists():
            raise FileNotFoundError(f"{p} missing: run `make -C oracle`")
        self.lib = lib = ctypes.CDLL(str(p))
        lib.pxo_build.restype = ctypes.c_void_p
        lib.pxo_build.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_int]
        lib.pxo_free.argtypes = [ctypes.c_void_p]
        lib.pxo_mlp_hidden.argtypes = [ctypes.c_void_p]
        lib.pxo_param.restype = _d
        lib.pxo_param.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.pxo_global.restype = _d
        lib.pxo_global.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.pxo_set_text.argtypes = [ctypes.c_void_p, _d]
        lib.pxo_tvec.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _d]
        lib.pxo_layer_forward.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, _d, ctypes.c_int64, _d, _d,
                                          ctypes.c_int64, ctypes.c_int64]
        lib.pxo_serial.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int,
                                   ctypes.c_double, _d, ctypes.c_char_p, ctypes.c_int]
        lib.pxo_pipefusion.argtypes = [ctypes.c_void_p, _d, ctypes.c_int64, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       _d, _i64p, _i64p, ctypes.c_char_p, ctypes.c_int]
        self.h = lib.pxo_build(seed, layers, hs, heads, mlp_ratio, text_tokens)
        if not self.h:
            raise OracleError(2, "invalid PixArt model shape")
        self.layers, self.hs, self.heads, self.T = layers, hs, heads, text_tokens
        self.mlp = lib.pxo_mlp_hidden(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.pxo_free(self.h)
            self.h = None

    def _shape(self, name):
        hs, mlp, T = self.hs, self.mlp, self.T
        return {"wqkv": (hs, 3 * hs), "bqkv": (3 * hs,), "w1": (hs, mlp), "b1": (mlp,),
                "w2": (mlp, hs), "sst": (6, hs), "wt1": (256, hs), "wt2": (hs, hs),
                "wt0": (hs, 6 * hs), "bt0": (6 * hs,), "y": (T, hs)}.get(
                    name, (hs, hs) if name.startswith("w") else (hs,))

    def param(self, layer: int, name: str) -> np.ndarray:
        shp = self._shape(name)
        ptr = self.lib.pxo_param(self.h, layer, PXO_PARAMS.index(name))
        return np.ctypeslib.as_array(ptr, shape=shp).copy()

    def glob(self, name: str) -> np.ndarray:
        shp = self._shape(name)
        ptr = self.lib.pxo_global(self.h, PXO_GLOBALS.index(name))
        return np.ctypeslib.as_array(ptr, shape=shp).copy()

    def set_text(self, y):
        y = _c(y)
        self.lib.pxo_set_text(self.h, _p(y))

    def tvec(self, t: int, steps: int) -> np.ndarray:
        out = np.empty(6 * self.hs)
        self.lib.pxo_tvec(self.h, t, steps, _p(out))
        return out

    def layer_forward(self, layer, t, steps, h, k, v, row0):
        h, k, v = _c(h).copy(), _c(k).copy(), _c(v).copy()
        self.lib.pxo_layer_forward(self.h, layer, t, steps, _p(h), h.shape[0], _p(k), _p(v),
                                   k.shape[0], row0)
        return h, k, v

    def serial_reference(self, x, steps, eta):
        x = _c(x)
        out = np.empty_like(x)
        err = ctypes.create_string_buffer(256)
        rc = self.lib.pxo_serial(self.h, _p(x), x.shape[0], steps, eta, _p(out), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def run_pipefusion(self, x, steps, workers, patches, warmup, eta):
        x = _c(x)
        out = np.empty_like(x)
        fresh, stale = ctypes.c_int64(), ctypes.c_int64()
        err = ctypes.create_string_buffer(256)
        rc = self.lib.pxo_pipefusion(self.h, _p(x), x.shape[0], steps, workers, patches,
                                     warmup, eta, _p(out), ctypes.byref(fresh),
                                     ctypes.byref(stale), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out, (fresh.value, stale.value)


def uniform_stream(seed: int, n: int) -> np.ndarray:
    """n next_uniform values of mt19937_64(seed) (pf_oracle.c pfo_uniform_stream)."""
    lib = ctypes.CDLL(str(RESTATEMENT_LIB))
    lib.pfo_uniform_stream.argtypes = [ctypes.c_uint64, ctypes.c_int64, _d]
    out = np.empty(n)
    lib.pfo_uniform_stream(ctypes.c_uint64(seed), n, _p(out))
    return out


def joint_model(seed, layers, hs, mlp, text_tokens, double_layers=None):
    """Parameters of pf_create_joint(seed, ...) (include/pipefusion_b200.h):
    per layer (image six, text six | None for single-stream layers) toy
    matrices, condition bias, text y."""
    D = layers if double_layers is None else double_layers
    sizes = [(hs, hs)] * 4 + [(hs, mlp), (mlp, hs)]
    per_stream = sum(a * b for a, b in sizes)
    total = (D * 2 + (layers - D)) * per_stream + hs
    u = uniform_stream(seed ^ 0x4a4f494e542d4449, total)
    scale = 1.0 / np.sqrt(hs)
    rscale = scale / np.sqrt(2.0 * layers)  # w_o, w_mlp_out: depth-scaled
    out, k = [], 0
    for l in range(layers):
        streams = []
        for _st in range(2 if l < D else 1):
            mats = []
            for i, (a, b) in enumerate(sizes):
                mats.append(u[k:k + a * b].reshape(a, b) * (rscale if i in (3, 5) else scale))
                k += a * b
            streams.append(tuple(mats))
        out.append((streams[0], streams[1] if l < D else None))
    cb = u[k:k + hs] * 1.0
    y = uniform_stream(seed ^ 0x5458542d544f4b53, text_tokens * hs).reshape(text_tokens, hs)
    return out, cb, y
