"""Head + hidden-column sharding of one block over ranks.

The reference runs a block on one CPU (model_forward_step, model.cpp:178-216).  Over g
GPUs, one process per GPU:

  attention  rank r owns heads [h0, h0 + H_r): q/k/v, column sums, the per-head top-k and
             the attention caches are all per head, so nothing crosses ranks until
             O_r . Wo[rows of those heads] — a partial [B, N, D] fp32 sum that is
             all-reduced (NCCL), then x1 = x + sum.
  MLP        rank r owns neurons [f0, f0 + F_r) (rows of W1 / W2, entries of b1; b2 lives
             on rank 0).  Dense step: partial M_r, all-reduced, x2 = x1 + sum.
             Sparse step: mlp_change_indices (mlp.cpp:98-118) is a GLOBAL per-chunk top-k
             over all F neurons.  Each rank all-gathers its local top-k candidates (k per
             chunk row, sorted by global id), every rank merges them identically on the GPU
             (csrc/shard.cu) and keeps its own neurons; the delta update is then local and
             its partial is all-reduced.

The per-head / per-neuron values do not depend on the shard (the tile-means split-K
depends on D only), so the selected neuron sets equal the single-GPU ones for the same
x1.  Only the Wo / W2 partial-sum order differs from one GPU (fp32, well inside the PROD
tolerance).
"""
from __future__ import annotations

from dataclasses import replace
from typing import Optional, Sequence

import torch

from .errors import raise_for
from .ops import Block, BlockConfig, _ptr, _stream


def split_range(total: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Balanced split of `total` items into `world` parts in units of `align`: (start, count)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if total % align:
        raise ValueError(f"{total} is not a multiple of the shard alignment {align}")
    units = total // align
    if units < world:
        raise ValueError(f"cannot split {total} into {world} shards of >= {align}")
    base, extra = divmod(units, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start * align, count * align


def shard_config(cfg: BlockConfig, world: int, rank: int, f_align: int = 128) -> BlockConfig:
    """This rank's slice of the block: its heads and its hidden columns."""
    h0, hl = split_range(cfg.heads, world, rank)
    f0, fl = split_range(cfg.hidden, world, rank, f_align)
    return replace(cfg, head0=h0, heads_local=hl, f0=f0, f_local=fl)


class Comm:
    """The collectives the sharded steps need."""

    world = 1
    rank = 0

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:  # in place, sum
        return t

    def all_gather(self, t: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """-> [world, *t.shape] in rank order (into `out` when given)."""
        if out is None:
            return t.unsqueeze(0)
        out.view(1, *t.shape).copy_(t)
        return out

    def all_to_all(self, t: torch.Tensor) -> torch.Tensor:
        """t = [world * rows, cols]: block s goes to rank s; returns [world, rows, cols] with
        the block received from rank s at index s."""
        return t.view(1, *t.shape)


class TorchComm(Comm):
    """torch.distributed process group (NCCL on GPUs, gloo in the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def all_reduce(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def all_gather(self, t, out=None):
        t = t.contiguous()
        if out is None:
            out = t.new_empty((self.world,) + tuple(t.shape))
        if self.nccl:
            self.dist.all_gather_into_tensor(out, t, group=self.group)
        else:
            self.dist.all_gather(list(out.unbind(0)), t, group=self.group)
        return out

    def all_to_all(self, t):
        t = t.contiguous()
        g = self.world
        out = t.new_empty((g, t.shape[0] // g) + tuple(t.shape[1:]))
        self.dist.all_to_all_single(out, t, group=self.group)  # NCCL and gloo
        return out


class BlockShard:
    """One rank's slice of a block on its GPU, driven through the csd_block_*_partial ABI."""

    def __init__(self, cfg: BlockConfig, weights: dict, world: int, rank: int,
                 f_align: int = 128):
        self.full = cfg
        self.cfg = shard_config(cfg, world, rank, f_align)
        self.block = Block(self.cfg, weights, production=True)
        self.lib = self.block.ctx.lib
        self.ctx = self.block.ctx
        c = cfg
        self.k = c.mlp_k or c.hidden
        self.rows = c.batch * (c.seq // c.chunk)
        dev = torch.device("cuda", torch.cuda.current_device())
        self._bufs = {
            "attn": torch.empty((c.batch, c.seq, c.dim), dtype=torch.float32, device=dev),
            "mlp": torch.empty((c.batch, c.seq, c.dim), dtype=torch.float32, device=dev),
            "cs": torch.empty((self.rows, self.k), dtype=torch.float32, device=dev),
            "ci": torch.empty((self.rows, self.k), dtype=torch.int32, device=dev),
        }

    def _chk(self, rc):
        raise_for(self.lib, rc)

    def attn_partial(self, x: torch.Tensor, dense: bool) -> torch.Tensor:
        out = self._bufs["attn"]
        self._chk(self.lib.csd_block_attn_partial(self.block.h, _ptr(x), int(bool(dense)),
                                                  _ptr(out), _stream()))
        return out

    def mlp_dense_partial(self, x_mid: torch.Tensor) -> torch.Tensor:
        out = self._bufs["mlp"]
        self._chk(self.lib.csd_block_mlp_dense_partial(self.block.h, _ptr(x_mid), _ptr(out),
                                                       _stream()))
        return out

    def mlp_candidates(self, x_mid: torch.Tensor):
        s, i = self._bufs["cs"], self._bufs["ci"]
        self._chk(self.lib.csd_block_mlp_candidates(self.block.h, _ptr(x_mid), _ptr(s), _ptr(i),
                                                    _stream()))
        return s, i

    def mlp_sparse_partial(self, x_mid, all_scores, all_ids) -> torch.Tensor:
        if all_scores.shape[1:] != (self.rows, self.k) or all_ids.shape != all_scores.shape:
            raise ValueError("candidate lists must be [world, rows, k]")
        out = self._bufs["mlp"]
        self._chk(self.lib.csd_block_mlp_sparse_partial(
            self.block.h, _ptr(x_mid), _ptr(all_scores.contiguous()), _ptr(all_ids.contiguous()),
            all_scores.shape[0], _ptr(out), _stream()))
        return out

    def residual_add(self, x: torch.Tensor, partial: torch.Tensor,
                     out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(x)
        self._chk(self.lib.csd_residual_add(self.ctx.h, _ptr(x), _ptr(partial), x.numel(),
                                            _ptr(out), _stream()))
        return out

    def indices(self, mlp: bool):
        """This shard's current index set (MLP ids are local: global id = f0 + id)."""
        return self.block.indices(mlp)

    def close(self):
        self.block.close()


class ShardedBlock:
    """model_forward_step for one block over a process group (one rank per GPU)."""

    def __init__(self, cfg: BlockConfig, weights: dict, comm: Comm, shard=None):
        self.cfg = cfg
        self.comm = comm
        self.shard = shard if shard is not None else BlockShard(cfg, weights, comm.world, comm.rank)

    def step(self, x: torch.Tensor, dense: bool, out: Optional[torch.Tensor] = None):
        sh, comm = self.shard, self.comm
        p = comm.all_reduce(sh.attn_partial(x, dense))
        x1 = sh.residual_add(x, p)
        if dense:
            m = sh.mlp_dense_partial(x1)
        else:
            s, i = sh.mlp_candidates(x1)
            m = sh.mlp_sparse_partial(x1, comm.all_gather(s), comm.all_gather(i))
        comm.all_reduce(m)
        return sh.residual_add(x1, m, out)


def token_shard_config(cfg: BlockConfig, world: int, rank: int) -> BlockConfig:
    """Token-sharded slice: heads split evenly for attention, the B*N token rows
    split into equal chunk-aligned ranges for Wo and the MLP (every hidden neuron)."""
    if cfg.heads % world:
        raise ValueError(f"{cfg.heads} heads do not split evenly over {world} ranks")
    rows = cfg.batch * cfg.seq
    if rows % (world * cfg.chunk):
        raise ValueError(f"{rows} token rows do not split into {world} equal chunk-aligned ranges")
    hl = cfg.heads // world
    tl = rows // world
    return replace(cfg, head0=rank * hl, heads_local=hl, f0=0, f_local=cfg.hidden,
                   t0=rank * tl, t_local=tl)


class TokenShardedBlock:
    """model_forward_step for one block over a process group, token-sharded: attention by
    heads (no communication), ONE bf16 all-to-all to token rows, Wo + the MLP on this rank's
    rows (exact: the MLP selection is per chunk), ONE bf16 all-gather of the output rows."""

    def __init__(self, cfg: BlockConfig, weights: dict, comm: Comm, block=None):
        self.full = cfg
        self.comm = comm
        self.cfg = token_shard_config(cfg, comm.world, comm.rank)
        self.block = block if block is not None else Block(self.cfg, weights, production=True)
        c = self.cfg
        self.rows = slice(c.t0, c.t0 + c.t_local)
        self._attn = self._y = None  # per-step buffers, allocated on the first step (x's dtype)

    def step(self, x: torch.Tensor, dense: bool, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        c, comm = self.cfg, self.comm
        if self._attn is None or self._attn.dtype != x.dtype or self._attn.device != x.device:
            self._attn = torch.empty((c.batch * c.seq, c.heads_local * c.head_dim), dtype=x.dtype,
                                     device=x.device)
            self._y = torch.empty((c.t_local, c.dim), dtype=x.dtype, device=x.device)
        xf = x.reshape(c.batch * c.seq, c.dim)
        a = self.block.attn_heads(xf, dense, out=self._attn)
        a_rows = comm.all_to_all(a)  # [world, t_local, Dl]
        y = self.block.rows_step(xf[self.rows], a_rows, comm.world, dense, out=self._y)
        if out is None:
            out = torch.empty_like(x)
        comm.all_gather(y, out=out.view(comm.world, c.t_local, c.dim))
        return out

    def close(self):
        self.block.close()


def simulate_token_step(blocks: Sequence[Block], x: torch.Tensor, dense: bool) -> torch.Tensor:
    """All token shards in ONE process (tests): the all-to-all / all-gather become slices and
    concatenations in rank order; every kernel call is exactly what each rank runs."""
    g = len(blocks)
    c0 = blocks[0].cfg
    xf = x.reshape(c0.batch * c0.seq, c0.dim)
    attn = [b.attn_heads(xf, dense).clone() for b in blocks]
    ys = []
    for r, b in enumerate(blocks):
        c = b.cfg
        a_rows = torch.stack([attn[s][c.t0:c.t0 + c.t_local] for s in range(g)])
        ys.append(b.rows_step(xf[c.t0:c.t0 + c.t_local].contiguous(), a_rows, g, dense).clone())
    return torch.cat(ys).reshape(x.shape)


def simulate_step(shards: Sequence, x: torch.Tensor, dense: bool) -> torch.Tensor:
    """All shards of one block in ONE process (tests): the collectives become sums / stacks
    in rank order, everything else is exactly what each rank runs."""
    ps = [s.attn_partial(x, dense).clone() for s in shards]
    p = ps[0]
    for q in ps[1:]:
        p = p + q
    x1 = shards[0].residual_add(x, p)
    if dense:
        ms = [s.mlp_dense_partial(x1).clone() for s in shards]
    else:
        cands = [tuple(t.clone() for t in s.mlp_candidates(x1)) for s in shards]
        all_s = torch.stack([c[0] for c in cands])
        all_i = torch.stack([c[1] for c in cands])
        ms = [s.mlp_sparse_partial(x1, all_s, all_i).clone() for s in shards]
    m = ms[0]
    for q in ms[1:]:
        m = m + q
    return shards[0].residual_add(x1, m)


__all__ = ["split_range", "shard_config", "Comm", "TorchComm", "BlockShard", "ShardedBlock",
           "simulate_step", "token_shard_config", "TokenShardedBlock", "simulate_token_step"]
