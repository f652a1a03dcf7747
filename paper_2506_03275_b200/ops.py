"""Python mirror of the reference's ``csd::`` operator API over the C ABI.

Same names, argument meaning and error behaviour as
``/root/reference/proj/include/csd/{voxel,sparse_index,attention,mlp}.hpp``,
operating on CUDA tensors.  The tensor dtype selects the mode:

* ``torch.float32`` -> ``CSD_MODE_CHECK`` (bit-exact reference arithmetic),
* ``torch.bfloat16`` -> ``CSD_MODE_PROD`` (tcgen05 tensor-core path).

Every call goes through ``libcsd_b200.so``; nothing here computes on the CPU.
Errors raise the reference's exception classes (``paper_2506_03275_b200.errors``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _capi as capi
from .errors import raise_for


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise TypeError("csd ops take CUDA tensors (host data goes through .to('cuda'))")
    if not t.is_contiguous():
        raise ValueError("csd ops take contiguous tensors")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _mode(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return capi.MODE_CHECK
    if t.dtype == torch.bfloat16:
        return capi.MODE_PROD
    raise TypeError(f"unsupported dtype {t.dtype}: float32 (check) or bfloat16 (production)")


class Context:
    """Owns a ``csd_ctx`` (workspaces, cuBLAS handle, device error flags)."""

    def __init__(self, device: int = 0):
        self.lib = capi.lib()
        h = C.c_void_p()
        raise_for(self.lib, self.lib.csd_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.csd_ctx_destroy(self.h)
            self.h = None

    __del__ = close

    def sync(self):
        raise_for(self.lib, self.lib.csd_ctx_sync(self.h, _stream()))

    def set_validation(self, enabled: bool):
        """PROD-mode per-call index-set validation (CHECK mode always validates)."""
        raise_for(self.lib, self.lib.csd_ctx_set_validation(self.h, int(bool(enabled))))

    def set_sorted_topk(self, sorted_: bool):
        """select_top_k order: descending (reference) or the same set in index order."""
        raise_for(self.lib, self.lib.csd_ctx_set_sorted_topk(self.h, int(bool(sorted_))))

    @property
    def launches(self) -> int:
        return int(self.lib.csd_ctx_launch_count(self.h))


_default: Optional[Context] = None


def context() -> Context:
    global _default
    if _default is None:
        _default = Context(torch.cuda.current_device())
    return _default


def _call(name, *args):
    ctx = context()
    rc = getattr(ctx.lib, name)(ctx.h, *args)
    raise_for(ctx.lib, rc)


# ------------------------------------------------------------------ voxel
@dataclass
class VoxelLayout:
    """voxel.hpp:13-20"""
    t: int = 1
    h: int = 1
    w: int = 1
    vt: int = 1
    vh: int = 1
    vw: int = 1

    def tokens(self) -> int:
        return self.t * self.h * self.w

    def voxel_volume(self) -> int:
        return self.vt * self.vh * self.vw


def voxel_permutation(layout: VoxelLayout) -> torch.Tensor:
    """voxel.cpp:18-42 -> int64 host tensor (new position -> original raster index)."""
    lib = capi.lib()
    perm = torch.empty(max(layout.tokens(), 1), dtype=torch.int64)
    raise_for(lib, lib.csd_voxel_permutation(layout.t, layout.h, layout.w, layout.vt, layout.vh,
                                             layout.vw, C.c_void_p(perm.data_ptr())))
    return perm


def voxel_order(x: torch.Tensor, layout: VoxelLayout):
    """voxel.cpp:44-73: [B,T,H,W,D] -> ([B,N,D], permutation)."""
    from .errors import ShapeError
    if x.dim() != 5:
        raise ShapeError(f"voxel_order expects [B x T x H x W x D], got {list(x.shape)}")
    if tuple(x.shape[1:4]) != (layout.t, layout.h, layout.w):
        raise ShapeError(f"voxel_order: tensor grid {list(x.shape)} does not match layout")
    b, d = x.shape[0], x.shape[4]
    out = torch.empty((b, layout.tokens(), d), dtype=x.dtype, device=x.device)
    _call("csd_voxel_reorder", _ptr(x), _ptr(out), b, layout.t, layout.h, layout.w, layout.vt,
          layout.vh, layout.vw, d * x.element_size(), 0, _stream())
    return out, voxel_permutation(layout)


def reverse_voxel_order(x: torch.Tensor, layout: VoxelLayout) -> torch.Tensor:
    """voxel.cpp:75-102: [B,N,D] -> [B,T,H,W,D]."""
    from .errors import ShapeError
    if x.dim() != 3:
        raise ShapeError(f"reverse_voxel_order expects [B x N x D], got {list(x.shape)}")
    if x.shape[1] != layout.tokens():
        raise ShapeError("reverse_voxel_order: sequence length does not match layout token count")
    b, d = x.shape[0], x.shape[2]
    out = torch.empty((b, layout.t, layout.h, layout.w, d), dtype=x.dtype, device=x.device)
    _call("csd_voxel_reorder", _ptr(x), _ptr(out), b, layout.t, layout.h, layout.w, layout.vt,
          layout.vh, layout.vw, d * x.element_size(), 1, _stream())
    return out


# ------------------------------------------------------------------ index sets
@dataclass
class SparseIndexSet:
    """sparse_index.hpp:15-40 with device storage: indices [B,H,C,k_max], counts [B,H,C]."""
    batch: int
    heads: int
    chunks: int
    chunk_size: int
    k_max: int
    domain: int
    indices: torch.Tensor
    counts: torch.Tensor

    @staticmethod
    def empty(batch, heads, chunks, chunk_size, k_max, domain, device="cuda"):
        return SparseIndexSet(batch, heads, chunks, chunk_size, k_max, domain,
                              torch.zeros((batch, heads, chunks, max(k_max, 0)), dtype=torch.int32,
                                          device=device),
                              torch.zeros((batch, heads, chunks), dtype=torch.int32, device=device))

    def validate(self):
        _call("csd_validate_index_set", _ptr(self.indices), _ptr(self.counts),
              self.batch * self.heads * self.chunks, self.k_max, self.domain, _stream())
        context().sync()


def index_set_to_masks(idx: SparseIndexSet, n: int) -> torch.Tensor:
    """bitmask.cpp:55-85 on the device: uint8 [B, H, C, ceil(n / 8)], one LSB-first bitpacked
    mask per (b, h, chunk) (bitmask.hpp:13-17); popcount of each row equals its count."""
    from . import errors
    if n < idx.domain:
        raise errors.ValueError(f"mask length {n} smaller than index domain {idx.domain}")
    out = torch.empty((idx.batch, idx.heads, idx.chunks, (n + 7) // 8), dtype=torch.uint8,
                      device=idx.indices.device)
    _call("csd_index_set_to_masks", _ptr(idx.indices), _ptr(idx.counts),
          idx.batch * idx.heads * idx.chunks, idx.k_max, n, _ptr(out), _stream())
    return out


def select_top_k(scores: torch.Tensor, k: int, chunk_size: int) -> SparseIndexSet:
    """sparse_index.cpp:64-96 on a [B,H,C,M] float32 tensor."""
    from .errors import ShapeError
    if scores.dim() != 4:
        raise ShapeError(f"select_top_k expects [B x H x C x M] scores, got {list(scores.shape)}")
    if scores.dtype != torch.float32:
        raise TypeError("select_top_k scores must be float32")
    b, h, c, m = scores.shape
    s = SparseIndexSet.empty(b, h, c, chunk_size, k, m, scores.device) if 1 <= k <= m else None
    if s is None:
        idx = torch.empty(1, dtype=torch.int32, device=scores.device)
        _call("csd_select_top_k", _ptr(scores), b * h * c, m, k, _ptr(idx), _ptr(idx), _stream())
    _call("csd_select_top_k", _ptr(scores), b * h * c, m, k, _ptr(s.indices), _ptr(s.counts),
          _stream())
    return s


# ------------------------------------------------------------------ attention
@dataclass
class SoftmaxStats:
    row_max: torch.Tensor
    exp_sum: torch.Tensor


def _layout_of(q: torch.Tensor, layout: int):
    if q.dim() != 4:
        from .errors import ShapeError
        raise ShapeError(f"attention expects [B x H x N x E] tensors, got q={list(q.shape)}")
    if layout == capi.LAYOUT_BHNE:
        b, h, n, e = q.shape
    else:
        b, n, h, e = q.shape
    return b, h, n, e


def _check_qkv(q, k, v):
    from .errors import ShapeError
    if q.shape != k.shape or q.shape != v.shape:
        raise ShapeError(f"attention q/k/v shapes disagree: q={list(q.shape)} k={list(k.shape)} "
                         f"v={list(v.shape)}")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise TypeError("attention q/k/v dtypes disagree")


def dense_attention(q, k, v, layout: int = capi.LAYOUT_BHNE) -> torch.Tensor:
    """attention.cpp:59-74"""
    _check_qkv(q, k, v)
    b, h, n, e = _layout_of(q, layout)
    out = torch.empty_like(q)
    _call("csd_dense_attention", _mode(q), layout, _ptr(q), _ptr(k), _ptr(v), b, h, n, e, _ptr(out),
          _stream())
    return out


@dataclass
class ColumnSumAttentionResult:
    output: torch.Tensor
    column_sums: torch.Tensor
    stats: SoftmaxStats


def column_sum_attention(q, k, v, prev_stats: Optional[SoftmaxStats], chunk: int,
                         layout: int = capi.LAYOUT_BHNE) -> ColumnSumAttentionResult:
    """attention.cpp:76-145"""
    from .errors import ShapeError
    _check_qkv(q, k, v)
    b, h, n, e = _layout_of(q, layout)
    if chunk < 1 or n % chunk:
        raise ShapeError(f"column_sum_attention: sequence length {n} not divisible by chunk {chunk}")
    if prev_stats is not None and (tuple(prev_stats.row_max.shape) != (b, h, n)
                                   or tuple(prev_stats.exp_sum.shape) != (b, h, n)):
        raise ShapeError("column_sum_attention: previous stats shape does not match")
    dev = q.device
    out = torch.empty_like(q)
    m = torch.empty((b, h, n), dtype=torch.float32, device=dev)
    l = torch.empty((b, h, n), dtype=torch.float32, device=dev)
    cs = torch.empty((b, h, n // chunk, n), dtype=torch.float32, device=dev)
    _call("csd_column_sum_attention", _mode(q), layout, _ptr(q), _ptr(k), _ptr(v),
          _ptr(prev_stats.row_max) if prev_stats else None,
          _ptr(prev_stats.exp_sum) if prev_stats else None, b, h, n, e, chunk, _ptr(out), _ptr(m),
          _ptr(l), _ptr(cs), _stream())
    return ColumnSumAttentionResult(out, cs, SoftmaxStats(m, l))


def _check_index_set(idx: SparseIndexSet, b, h, n):
    from .errors import ShapeError
    if idx.batch != b or idx.heads != h:
        raise ShapeError(f"sparse index set dims ({idx.batch},{idx.heads}) do not match q")
    if idx.domain != n or idx.chunks * idx.chunk_size != n:
        raise ShapeError(f"sparse index set chunking does not cover the sequence length {n}")


def sparse_delta_attention(q, k, v, indices: SparseIndexSet, base: torch.Tensor, scale: float,
                           layout: int = capi.LAYOUT_BHNE, out: Optional[torch.Tensor] = None):
    """attention.cpp:147-194"""
    from .errors import ShapeError
    _check_qkv(q, k, v)
    if base.shape != q.shape:
        raise ShapeError(f"sparse_delta_attention: base shape {list(base.shape)} does not match q")
    b, h, n, e = _layout_of(q, layout)
    _check_index_set(indices, b, h, n)
    if out is None:
        out = torch.empty_like(base)
    _call("csd_sparse_delta_attention", _mode(q), layout, _ptr(q), _ptr(k), _ptr(v),
          _ptr(indices.indices), _ptr(indices.counts), indices.k_max, indices.chunk_size,
          _ptr(base), float(scale), b, h, n, e, _ptr(out), _stream())
    return out


@dataclass
class AttentionCache:
    """attention.hpp:13-19"""
    residual_output: Optional[torch.Tensor] = None
    stats: Optional[SoftmaxStats] = None
    indices: Optional[SparseIndexSet] = None
    age: int = 0
    initialized: bool = False


def attention_step(q, k, v, cache: AttentionCache, dense_step: bool, top_k: int, chunk: int,
                   static_indices: Optional[SparseIndexSet] = None,
                   layout: int = capi.LAYOUT_BHNE) -> torch.Tensor:
    """attention.cpp:196-219"""
    from .errors import StateError
    if not dense_step and not cache.initialized:
        raise StateError("sparse attention step requested before any dense step")
    if dense_step:
        prev = cache.stats if cache.initialized else None
        res = column_sum_attention(q, k, v, prev, chunk, layout)
        idx = static_indices if static_indices is not None else select_top_k(res.column_sums,
                                                                              top_k, chunk)
        b, h, n, _ = _layout_of(q, layout)
        _check_index_set(idx, b, h, n)
        cache.residual_output = sparse_delta_attention(q, k, v, idx, res.output, -1.0, layout)
        cache.stats = res.stats
        cache.indices = idx
        cache.age = 0
        cache.initialized = True
        return res.output
    cache.age += 1
    return sparse_delta_attention(q, k, v, cache.indices, cache.residual_output, 1.0, layout)


# ------------------------------------------------------------------ MLP
@dataclass
class MlpWeights:
    """mlp.hpp:12-21: w1 [F,D], b1 [F], w2 [F,D], b2 [D] (biases always float32)."""
    w1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    b2: torch.Tensor

    def hidden(self):
        return self.w1.shape[0]

    def model_dim(self):
        return self.w1.shape[1]


@dataclass
class MlpCache:
    """mlp.hpp:29-36.  ``activations`` is in the mode's cache layout: [B,N,F] float32 (check) or
    chunk-major [B,C,F,c] bfloat16 (production); ``activations_ref()`` gives [B,N,F] float32."""
    tile_means: Optional[torch.Tensor] = None
    activations: Optional[torch.Tensor] = None
    outputs: Optional[torch.Tensor] = None
    indices: Optional[SparseIndexSet] = None
    age: int = 0
    initialized: bool = False
    chunk: int = 0

    def activations_ref(self) -> torch.Tensor:
        b, n, _ = self.outputs.shape
        f = self.tile_means.shape[-1]
        out = torch.empty((b, n, f), dtype=torch.float32, device=self.outputs.device)
        _call("csd_mlp_act_cache_to_ref", _mode(self.activations), _ptr(self.activations), b, n, f,
              self.chunk, _ptr(out), _stream())
        return out


def _check_x(x, w: MlpWeights):
    from .errors import ShapeError
    if x.dim() != 3:
        raise ShapeError(f"mlp expects [B x N x D] input, got {list(x.shape)}")
    if x.shape[2] != w.model_dim():
        raise ShapeError(f"mlp input dim {x.shape[2]} does not match weights' model dim {w.model_dim()}")


def dense_mlp(x, w: MlpWeights, chunk: int = 0):
    """mlp.cpp:49-81 -> (output float32 [B,N,D], activations in the mode's cache layout)."""
    _check_x(x, w)
    b, n, d = x.shape
    f = w.hidden()
    out = torch.empty((b, n, d), dtype=torch.float32, device=x.device)
    mode = _mode(x)
    if mode == capi.MODE_PROD:
        c = chunk if chunk else n
        act = torch.empty((b, n // c, f, c), dtype=torch.bfloat16, device=x.device)
    else:
        c = chunk if chunk else n
        act = torch.empty((b, n, f), dtype=torch.float32, device=x.device)
    _call("csd_dense_mlp", mode, _ptr(x), _ptr(w.w1), _ptr(w.b1), _ptr(w.w2), _ptr(w.b2), b, n, d, f,
          c, _ptr(out), _ptr(act), _stream())
    return out, act


def project(x, w) -> torch.Tensor:
    """model.cpp:107-120: [B, N, D] @ [D, Dout] -> [B, N, Dout] (PROD: the tcgen05 GEMM of
    gemm_tc.cu, bf16 out; CHECK: float32, the reference's loop order)."""
    from .errors import ShapeError
    if x.dim() != 3:
        raise ShapeError(f"project expects [B x N x D] input, got {list(x.shape)}")
    if w.dim() != 2 or w.shape[0] != x.shape[2]:
        raise ShapeError(f"project weight {list(w.shape)} does not match input dim {x.shape[2]}")
    b, n, d = x.shape
    out = torch.empty((b, n, w.shape[1]), dtype=x.dtype, device=x.device)
    _call("csd_project", _mode(x), _ptr(x), _ptr(w), b, n, d, w.shape[1], _ptr(out), _stream())
    return out


def mlp_tile_means(x, w1, chunk: int) -> torch.Tensor:
    """mlp.cpp:83-96"""
    from .errors import ShapeError
    if x.dim() != 3:
        raise ShapeError(f"mlp_tile_means expects [B x N x D] input, got {list(x.shape)}")
    b, n, d = x.shape
    f = w1.shape[0]
    if chunk < 1 or n % chunk:
        raise ShapeError(f"mlp_tile_means: sequence length {n} not divisible by chunk {chunk}")
    out = torch.empty((b, n // chunk, f), dtype=torch.float32, device=x.device)
    _call("csd_mlp_tile_means", _mode(x), _ptr(x), _ptr(w1), b, n, d, f, chunk, _ptr(out), _stream())
    return out


def mlp_change_indices(x, w1, tile_means, k: int, chunk: int) -> SparseIndexSet:
    """mlp.cpp:98-118"""
    from .errors import ShapeError
    b, n, d = x.shape
    f = w1.shape[0]
    if chunk < 1 or n % chunk:
        raise ShapeError(f"mlp_change_indices: sequence length {n} not divisible by chunk {chunk}")
    if tuple(tile_means.shape) != (b, n // chunk, f):
        raise ShapeError("mlp_change_indices: cached tile means do not match fresh")
    s = SparseIndexSet.empty(b, 1, n // chunk, chunk, max(k, 0), f, x.device)
    _call("csd_mlp_change_indices", _mode(x), _ptr(x), _ptr(w1), _ptr(tile_means), b, n, d, f, k,
          chunk, _ptr(s.indices), _ptr(s.counts), _stream())
    return s


def sparse_delta_mlp(x, w: MlpWeights, indices: SparseIndexSet, cache: MlpCache) -> torch.Tensor:
    """mlp.cpp:120-182: updates cache.activations / cache.outputs in place, returns outputs."""
    from .errors import ShapeError, StateError
    _check_x(x, w)
    if not cache.initialized:
        raise StateError("sparse MLP step requested before any dense step")
    b, n, d = x.shape
    f = w.hidden()
    if (indices.batch != b or indices.heads != 1 or indices.domain != f
            or indices.chunks * indices.chunk_size != n):
        raise ShapeError(f"mlp sparse index set does not match (B={b}, N={n}, F={f})")
    _call("csd_sparse_delta_mlp", _mode(x), _ptr(x), _ptr(w.w1), _ptr(w.b1), _ptr(w.w2),
          _ptr(indices.indices), _ptr(indices.counts), indices.k_max, indices.chunk_size, b, n, d,
          f, _ptr(cache.activations), _ptr(cache.outputs), _stream())
    return cache.outputs


def mlp_step(x, w: MlpWeights, cache: MlpCache, dense_step: bool, top_k: int,
             chunk: int) -> torch.Tensor:
    """mlp.cpp:184-211"""
    from .errors import ShapeError, StateError
    if not dense_step and not cache.initialized:
        raise StateError("sparse MLP step requested before any dense step")
    if x.dim() != 3:
        raise ShapeError(f"mlp_step expects [B x N x D] input, got {list(x.shape)}")
    if chunk < 1 or x.shape[1] % chunk:
        raise ShapeError(f"mlp_step: sequence length {x.shape[1]} not divisible by chunk {chunk}")
    if dense_step:
        out, act = dense_mlp(x, w, chunk)
        cache.tile_means = mlp_tile_means(x, w.w1, chunk)
        cache.activations = act
        cache.outputs = out.clone()
        cache.indices = None
        cache.age = 0
        cache.initialized = True
        cache.chunk = chunk
        return out
    idx = mlp_change_indices(x, w.w1, cache.tile_means, top_k, chunk)
    cache.age += 1
    out = sparse_delta_mlp(x, w, idx, cache).clone()
    cache.indices = idx
    return out


# ------------------------------------------------------------------ block
@dataclass
class BlockConfig:
    """ModelConfig (model.hpp:16-41) restricted to one block, plus the per-chunk k's."""
    batch: int
    seq: int
    dim: int
    heads: int
    head_dim: int
    hidden: int
    chunk: int
    attn_k: int
    mlp_k: int
    head0: int = 0
    heads_local: int = 0
    f0: int = 0
    f_local: int = 0
    t0: int = 0       # token-sharded execution: Wo + MLP on rows [t0, t0 + t_local)
    t_local: int = 0


class Block:
    """Device-resident DiT block (model_forward_step for one layer, model.cpp:178-216)."""

    def __init__(self, cfg: BlockConfig, weights: dict, production: bool = True):
        self.cfg = cfg
        self.mode = capi.MODE_PROD if production else capi.MODE_CHECK
        self.dtype = torch.bfloat16 if production else torch.float32
        ctx = context()
        self.ctx = ctx
        c = capi.BlockConfig(*[getattr(cfg, f) for f, _ in capi.BlockConfig._fields_])
        hw = {k: torch.as_tensor(weights[k], dtype=torch.float32).contiguous().cpu()
              for k in ("wq", "wk", "wv", "wo", "w1", "b1", "w2", "b2")}
        self._host = hw
        h = C.c_void_p()
        raise_for(ctx.lib, ctx.lib.csd_block_create(
            ctx.h, self.mode, C.byref(c), *[C.c_void_p(hw[k].data_ptr()) for k in
                                            ("wq", "wk", "wv", "wo", "w1", "b1", "w2", "b2")],
            C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.csd_block_destroy(self.h)
            self.h = None

    __del__ = close

    def step(self, x: torch.Tensor, dense: bool, out: Optional[torch.Tensor] = None,
             static: Optional[SparseIndexSet] = None) -> torch.Tensor:
        if x.dtype != self.dtype:
            raise TypeError(f"block expects {self.dtype} activations")
        if out is None:
            out = torch.empty_like(x)
        if static is not None:
            from .errors import ShapeError
            c = self.cfg
            hl = c.heads_local or c.heads
            want = (c.batch, hl, c.seq // c.chunk, c.chunk, c.seq)
            got = (static.batch, static.heads, static.chunks, static.chunk_size, static.domain)
            if got != want or tuple(static.indices.shape) != (*want[:3], static.k_max):
                raise ShapeError(f"static attention pattern (batch, heads, chunks, chunk, domain)"
                                 f" = {got} does not match the block {want}")
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_step(
            self.h, _ptr(x), _ptr(out), int(bool(dense)),
            _ptr(static.indices) if static else None, _ptr(static.counts) if static else None,
            static.k_max if static else 0, _stream()))
        return out

    def forward_dense(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """model_forward_dense for this layer (model.cpp:167-176): exact attention + dense MLP,
        no cache touched (the reference's dense baseline)."""
        if x.dtype != self.dtype:
            raise TypeError(f"block expects {self.dtype} activations")
        if out is None:
            out = torch.empty_like(x)
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_step(self.h, _ptr(x), _ptr(out), 2, None, None, 0,
                                                             _stream()))
        return out

    def reset(self):
        """A fresh ModelState for this layer (model.cpp:101-105): the next step must be dense."""
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_reset(self.h))

    def cache_arena(self):
        """(device pointer, bytes) of the one allocation holding this layer's persistent caches."""
        ptr, n = C.c_void_p(), C.c_size_t()
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_cache_arena(self.h, C.byref(ptr), C.byref(n)))
        return ptr.value, n.value

    def bind_cache_arena(self, storage: torch.Tensor):
        """Re-point this layer's caches into `storage` (a device uint8 tensor of at least
        cache_arena() bytes, same layout; contents not copied).  The block keeps a reference."""
        if not storage.is_cuda or storage.dtype != torch.uint8:
            raise TypeError("cache storage is a device uint8 tensor")
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_bind_cache_arena(
            self.h, C.c_void_p(storage.data_ptr()), storage.numel()))
        self._arena_storage = storage

    def attn_heads(self, x: torch.Tensor, dense: bool, out: Optional[torch.Tensor] = None):
        """Token-sharded step, part 1: this block's heads over every token -> [B*N, Dl] bf16."""
        c = self.cfg
        hl = c.heads_local or c.heads
        if out is None:
            out = torch.empty((c.batch * c.seq, hl * c.head_dim), dtype=self.dtype, device=x.device)
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_attn_heads(self.h, _ptr(x), int(bool(dense)),
                                                                  _ptr(out), _stream()))
        return out

    def rows_step(self, x_rows: torch.Tensor, attn_rows: torch.Tensor, world: int, dense: bool,
                  out: Optional[torch.Tensor] = None):
        """Token-sharded step, part 2: x_out rows = MLP(x + O Wo) on this block's token rows;
        attn_rows = [world][t_local][Dl] (the all-to-all of every rank's attn_heads)."""
        if out is None:
            out = torch.empty_like(x_rows)
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_rows_step(
            self.h, _ptr(x_rows), _ptr(attn_rows.contiguous()), int(world), int(bool(dense)),
            _ptr(out), _stream()))
        return out

    def cache(self, which: int) -> torch.Tensor:
        c = self.cfg
        hl = c.heads_local or c.heads
        fl = c.f_local or c.hidden
        nc = c.seq // c.chunk
        mb, mn = (1, c.t_local) if c.t_local else (c.batch, c.seq)  # the MLP caches' rows
        shapes = {0: (c.batch, hl, c.seq, c.head_dim), 1: (c.batch, hl, c.seq),
                  2: (c.batch, hl, c.seq), 3: (mb, mn, fl), 4: (mb, mn, c.dim),
                  5: (mb, mn // c.chunk, fl)}
        t = torch.empty(shapes[which], dtype=torch.float32, device="cuda")
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_cache(self.h, which, _ptr(t), None, _stream()))
        return t

    def indices(self, mlp: bool):
        c = self.cfg
        hl = 1 if mlp else (c.heads_local or c.heads)
        k = (c.mlp_k or (c.f_local or c.hidden)) if mlp else (c.attn_k or c.seq)
        b, nc = c.batch, c.seq // c.chunk
        if mlp and c.t_local:  # a token shard's MLP chunks
            b, nc = 1, c.t_local // c.chunk
        idx = torch.empty((b, hl, nc, k), dtype=torch.int32, device="cuda")
        cnt = torch.empty((b, hl, nc), dtype=torch.int32, device="cuda")
        raise_for(self.ctx.lib, self.ctx.lib.csd_block_cache(self.h, 7 if mlp else 6, _ptr(idx),
                                                             _ptr(cnt), _stream()))
        return idx, cnt
