"""TEST INFRASTRUCTURE ONLY — numpy front end for the CPU oracle.

Two back ends with one calling convention:

* ``Oracle("port")`` loads ``oracle/liboracle.so``: our plain-C restatement of
  the reference hot path (``oracle/csd_oracle.c``).
* ``Oracle("reference")`` loads ``oracle/_ref/libcsd_ref.so``: the unmodified
  reference library compiled from ``/root/reference/proj/src`` (``oracle/Makefile``)
  behind the ``oracle/ref_capi.cpp`` shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcsd_ref.so")

_F = C.POINTER(C.c_float)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_L = C.c_int64


class OracleError(RuntimeError):
    """Raised with the reference exception class name the oracle mapped."""

    NAMES = {-1: "ShapeError", -2: "IndexError", -3: "NumericError", -4: "StateError",
             -5: "ValueError", -6: "ConfigError", -100: "Error"}

    def __init__(self, code: int):
        self.code = code
        self.kind = self.NAMES.get(code, f"code{code}")
        super().__init__(self.kind)


def _f(a):
    return a.ctypes.data_as(_F) if a is not None else None


def _i32(a):
    return a.ctypes.data_as(_I32) if a is not None else None


def _chk(rc):
    if rc != 0:
        raise OracleError(rc)


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle{' ref' if kind != 'port' else ''}`)")
        self.lib = C.CDLL(path)
        self.p = "csdo_" if kind == "port" else "ref_"
        for name in ("expf", "tanhf", "gelu"):
            if kind == "port":
                fn = getattr(self.lib, "csdo_" + name)
                fn.restype = C.c_float
                fn.argtypes = [C.c_float]

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    # -- seeded inputs (rng.hpp:12-44; bit-identical to the reference stream) --
    def gaussian(self, seed: int, shape, std: float = 1.0) -> np.ndarray:
        n = int(np.prod(shape))
        out = np.empty(n, np.float32)
        fn = self.lib.csdo_gaussian if self.kind == "port" else self.lib.ref_gaussian
        fn(C.c_uint64(seed), _L(n), C.c_float(std), _f(out))
        return out.reshape(shape)

    def libm_mismatches(self, start: int, stop: int, step: int, which: int) -> int:
        fn = self.lib.csdo_libm_mismatches
        fn.restype = C.c_int64
        fn.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]
        return int(fn(start, stop, step, which))

    # -- scalar transcendentals (port only) --------------------------------
    def expf(self, x: float) -> float:
        return self.lib.csdo_expf(C.c_float(x))

    def tanhf(self, x: float) -> float:
        return self.lib.csdo_tanhf(C.c_float(x))

    # -- voxel --------------------------------------------------------------
    def voxel_permutation(self, grid, voxel):
        t, h, w = grid
        perm = np.zeros(t * h * w, dtype=np.int64)
        _chk(self._fn("voxel_permutation")(_L(t), _L(h), _L(w), _L(voxel[0]), _L(voxel[1]),
                                           _L(voxel[2]), perm.ctypes.data_as(_I64)))
        return perm

    def voxel_order(self, x, voxel):
        x = f32(x)
        b, t, h, w, d = x.shape
        out = np.empty((b, t * h * w, d), np.float32)
        _chk(self._fn("voxel_order")(_f(x), _L(b), _L(t), _L(h), _L(w), _L(d), _L(voxel[0]),
                                     _L(voxel[1]), _L(voxel[2]), _f(out)))
        return out

    def reverse_voxel_order(self, x, grid, voxel):
        x = f32(x)
        b, n, d = x.shape
        t, h, w = grid
        out = np.empty((b, t, h, w, d), np.float32)
        _chk(self._fn("reverse_voxel_order")(_f(x), _L(b), _L(t), _L(h), _L(w), _L(d),
                                             _L(voxel[0]), _L(voxel[1]), _L(voxel[2]), _f(out)))
        return out

    # -- projections (port only; model.cpp:107-120) --------------------------
    def project(self, x, w):
        """x [B, N, D] @ w [D, Dout] with the reference's accumulation order."""
        x, w = f32(x), f32(w)
        b, n, d = x.shape
        out = np.empty((b, n, w.shape[1]), np.float32)
        self.lib.csdo_project(_f(x), _f(w), _L(b), _L(n), _L(d), _L(w.shape[1]), _f(out))
        return out

    # -- selection ----------------------------------------------------------
    def select_top_k(self, scores, k):
        s = f32(scores)
        m = s.shape[-1]
        rows = s.size // m
        idx = np.empty(rows * k, np.int32)
        _chk(self._fn("select_top_k")(_f(s), _L(rows), _L(m), _L(k), _i32(idx)))
        return idx.reshape(s.shape[:-1] + (k,))

    # -- attention ----------------------------------------------------------
    def dense_attention(self, q, k, v):
        q, k, v = f32(q), f32(k), f32(v)
        out = np.empty_like(q)
        _chk(self._fn("dense_attention")(_f(q), _f(k), _f(v), *map(_L, q.shape), _f(out)))
        return out

    def column_sum_attention(self, q, k, v, prev_stats, chunk):
        q, k, v = f32(q), f32(k), f32(v)
        b, h, n, e = q.shape
        out = np.empty_like(q)
        m = np.empty((b, h, n), np.float32)
        l = np.empty((b, h, n), np.float32)
        cs = np.empty((b, h, n // chunk, n), np.float32) if chunk > 0 and n % chunk == 0 else np.empty(1, np.float32)
        pm = f32(prev_stats[0]) if prev_stats is not None else None
        pl = f32(prev_stats[1]) if prev_stats is not None else None
        _chk(self._fn("column_sum_attention")(_f(q), _f(k), _f(v), _f(pm), _f(pl), _L(b), _L(h),
                                              _L(n), _L(e), _L(chunk), _f(out), _f(m), _f(l), _f(cs)))
        return out, cs, (m, l)

    def sparse_delta_attention(self, q, k, v, idx, counts, chunk, base, scale):
        q, k, v, base = f32(q), f32(k), f32(v), f32(base)
        idx, counts = i32(idx), i32(counts)
        b, h, n, e = q.shape
        k_max = idx.shape[-1]
        out = np.empty_like(q)
        _chk(self._fn("sparse_delta_attention")(_f(q), _f(k), _f(v), _i32(idx), _i32(counts),
                                                _L(k_max), _L(chunk), _f(base), C.c_float(scale),
                                                _L(b), _L(h), _L(n), _L(e), _f(out)))
        return out

    # -- mlp ----------------------------------------------------------------
    def dense_mlp(self, x, w1, b1, w2, b2):
        x = f32(x)
        b, n, d = x.shape
        f = w1.shape[0]
        out = np.empty_like(x)
        pre = np.empty((b, n, f), np.float32)
        act = np.empty((b, n, f), np.float32)
        _chk(self._fn("dense_mlp")(_f(x), _f(f32(w1)), _f(f32(b1)), _f(f32(w2)), _f(f32(b2)),
                                   _L(b), _L(n), _L(d), _L(f), _f(out), _f(pre), _f(act)))
        return out, pre, act

    def mlp_tile_means(self, x, w1, chunk):
        x = f32(x)
        b, n, d = x.shape
        f = w1.shape[0]
        out = np.empty((b, n // chunk, f), np.float32)
        _chk(self._fn("mlp_tile_means")(_f(x), _f(f32(w1)), _L(b), _L(n), _L(d), _L(f),
                                        _L(chunk), _f(out)))
        return out

    def mlp_change_indices(self, x, w1, tile_means, k, chunk):
        x = f32(x)
        b, n, d = x.shape
        f = w1.shape[0]
        idx = np.empty((b, 1, n // chunk, k), np.int32)
        _chk(self._fn("mlp_change_indices")(_f(x), _f(f32(w1)), _f(f32(tile_means)), _L(b), _L(n),
                                            _L(d), _L(f), _L(k), _L(chunk), _i32(idx)))
        return idx

    def sparse_delta_mlp(self, x, w1, b1, w2, b2, idx, counts, chunk, act_cache, out_cache):
        """Returns (new_out, new_act_cache); inputs are not modified."""
        x = f32(x)
        b, n, d = x.shape
        f = w1.shape[0]
        idx, counts = i32(idx), i32(counts)
        act = f32(act_cache).copy()
        out = f32(out_cache).copy()
        args = [_f(x), _f(f32(w1)), _f(f32(b1)), _f(f32(w2))]
        if self.kind != "port":
            args.append(_f(f32(b2)))
        _chk(self._fn("sparse_delta_mlp")(*args, _i32(idx), _i32(counts), _L(idx.shape[-1]),
                                          _L(chunk), _L(b), _L(n), _L(d), _L(f), _f(act), _f(out)))
        return out, act


class RefModel:
    """Handle on the reference toy block stack (model.cpp) — reference backend only."""

    def __init__(self, cfg: dict):
        self.lib = C.CDLL(REF_LIB)
        self.lib.ref_model_create.restype = C.c_void_p
        self.cfg = dict(cfg)
        c = self.cfg
        self.h = self.lib.ref_model_create(
            _L(c["batch"]), _L(c["grid"][0]), _L(c["grid"][1]), _L(c["grid"][2]), _L(c["dim"]),
            _L(c["head_dim"]), _L(c["heads"]), _L(c["hidden"]), _L(c["layers"]),
            _L(c["voxel"][0]), _L(c["voxel"][1]), _L(c["voxel"][2]), _L(c["chunk"]),
            C.c_uint64(c["seed"]))
        if not self.h:
            raise OracleError(-6)
        self.n = c["grid"][0] * c["grid"][1] * c["grid"][2]

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_model_destroy(C.c_void_p(self.h))
            self.h = None

    def weights(self, layer):
        c = self.cfg
        d, f = c["dim"], c["hidden"]
        shapes = [(d, d)] * 4 + [(f, d), (f,), (f, d), (d,)]
        names = ["wq", "wk", "wv", "wo", "w1", "b1", "w2", "b2"]
        out = {}
        for i, (nm, shp) in enumerate(zip(names, shapes)):
            a = np.empty(shp, np.float32)
            self.lib.ref_model_weight(C.c_void_p(self.h), _L(layer), C.c_int(i), _f(a))
            out[nm] = a
        return out

    def step(self, x, dense, attn_k, mlp_k):
        x = f32(x)
        out = np.empty_like(x)
        _chk(self.lib.ref_model_step(C.c_void_p(self.h), _f(x), C.c_int(int(dense)), _L(attn_k),
                                     _L(mlp_k), _f(out)))
        return out

    def step_static(self, x, dense, attn_k, mlp_k, idx, counts):
        """model_forward_step with a static attention pattern (model.hpp:97-99)."""
        x = f32(x)
        out = np.empty_like(x)
        idx = np.ascontiguousarray(idx, np.int32)
        counts = np.ascontiguousarray(counts, np.int32)
        _chk(self.lib.ref_model_step_static(C.c_void_p(self.h), _f(x), C.c_int(int(dense)),
                                            _L(attn_k), _L(mlp_k), _i32(idx), _i32(counts),
                                            _L(idx.shape[-1]), _f(out)))
        return out

    def dense(self, x):
        x = f32(x)
        out = np.empty_like(x)
        _chk(self.lib.ref_model_dense(C.c_void_p(self.h), _f(x), _f(out)))
        return out

    def indices(self, layer, mlp, k_max):
        c = self.cfg
        nc = self.n // c["chunk"]
        heads = 1 if mlp else c["heads"]
        idx = np.zeros((c["batch"], heads, nc, k_max), np.int32)
        cnt = np.zeros((c["batch"], heads, nc), np.int32)
        self.lib.ref_model_indices(C.c_void_p(self.h), _L(layer), C.c_int(int(mlp)), _i32(idx), _i32(cnt))
        return idx, cnt


def resolve_schedule(total_steps, dense_interval, step_cache=False, window=0, stride=1):
    """schedule.cpp:44-87 through the reference library: modes (0 dense, 1 sparse, 2 skipped)."""
    lib = C.CDLL(REF_LIB)
    modes = np.zeros(max(int(total_steps), 1), np.int32)
    _chk(lib.ref_resolve_schedule(_L(total_steps), _L(dense_interval), C.c_int(int(step_cache)),
                                  _L(window), _L(stride), _i32(modes)))
    return modes


def run_generation(cfg: dict, sched: dict):
    """harness.cpp:123-224 (run_generation, sparse-delta mode) through the reference library.

    Returns (modes, per-step latent R^2, end-to-end R^2, decoded final latent [B,T,H,W,D])."""
    lib = C.CDLL(REF_LIB)
    c = cfg
    cv = np.array([c["batch"], *c["grid"], c["dim"], c["head_dim"], c["heads"], c["hidden"],
                   c["layers"], *c["voxel"], c["chunk"], c["seed"]], np.int64)
    sv = np.array([sched["total_steps"], sched["dense_interval"], int(sched["step_cache"]),
                   sched["window"], sched["stride"], sched["attn_k"], sched["mlp_k"]], np.int64)
    t = int(sched["total_steps"])
    modes = np.zeros(t, np.int32)
    r2 = np.zeros(t, np.float64)
    e2e = np.zeros(1, np.float64)
    out = np.zeros((c["batch"], *c["grid"], c["dim"]), np.float32)
    p64 = C.POINTER(C.c_int64)
    pd = C.POINTER(C.c_double)
    _chk(lib.ref_run_generation(cv.ctypes.data_as(p64), sv.ctypes.data_as(p64), _i32(modes),
                                r2.ctypes.data_as(pd), e2e.ctypes.data_as(pd), _f(out)))
    return modes, r2, float(e2e[0]), out


def gaussian(seed: int, shape, std: float = 1.0) -> np.ndarray:
    """tests/test_util.hpp:50-55 random_tensor, bit-identical (needs the reference lib)."""
    lib = C.CDLL(REF_LIB)
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    lib.ref_gaussian(C.c_uint64(seed), _L(n), C.c_float(std), _f(out))
    return out.reshape(shape)
