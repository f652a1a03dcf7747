"""Test-side shard backed by the CPU oracle (test infrastructure, never shipped).

Implements the same five calls as `paper_2506_03275_b200.shard.BlockShard` with the oracle
ops on this rank's heads / neurons, so `ShardedBlock`'s collective sequence can run over
gloo on CPU (world_size 2) and be checked against the single-process reference results.
The merge follows csrc/shard.cu: local top-k -> ascending global id -> pad to k ->
all-gather (rank-major) -> top-k over positions -> keep own ids.
"""
import os
import pickle
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

import oracle as O  # noqa: E402
from paper_2506_03275_b200.shard import shard_config  # noqa: E402


def candidates(port, scores_rows, k, f0):
    """[rows, F_r] scores -> ([rows, k] scores, [rows, k] global ids), ascending id, padded."""
    rows, fl = scores_rows.shape
    k_loc = min(k, fl)
    ids = port.select_top_k(scores_rows, k_loc)
    ids = np.sort(ids, axis=1)
    cs = np.full((rows, k), -1.0, np.float32)
    ci = np.full((rows, k), np.iinfo(np.int32).max, np.int32)
    cs[:, :k_loc] = np.take_along_axis(scores_rows, ids, axis=1)
    ci[:, :k_loc] = ids + f0
    return cs, ci


def merge(port, all_s, all_i, k, f0, fl):
    """[g, rows, k] candidates -> this rank's (local idx [rows, k], counts [rows])."""
    g, rows, _ = all_s.shape
    s = np.ascontiguousarray(all_s.transpose(1, 0, 2).reshape(rows, g * k))
    i = np.ascontiguousarray(all_i.transpose(1, 0, 2).reshape(rows, g * k))
    pos = port.select_top_k(s, k)
    gids = np.take_along_axis(i, pos, axis=1)
    idx = np.zeros((rows, k), np.int32)
    cnt = np.zeros(rows, np.int32)
    for r in range(rows):
        mine = [int(x) - f0 for x in gids[r] if f0 <= x < f0 + fl]
        idx[r, :len(mine)] = mine
        cnt[r] = len(mine)
    return idx, cnt


class OracleShard:
    def __init__(self, cfg, w, world, rank, f_align=32):
        self.port = O.Oracle("port")
        self.full = cfg
        self.cfg = c = shard_config(cfg, world, rank, f_align)
        e = c.head_dim
        cols = slice(c.head0 * e, (c.head0 + c.heads_local) * e)
        f = slice(c.f0, c.f0 + c.f_local)
        self.wq, self.wk, self.wv = (np.ascontiguousarray(w[n][:, cols]) for n in ("wq", "wk", "wv"))
        self.wo = np.ascontiguousarray(w["wo"][cols, :])
        self.w1, self.b1, self.w2 = (np.ascontiguousarray(w[n][f]) for n in ("w1", "b1", "w2"))
        self.b2 = w["b2"] if c.f0 == 0 else np.zeros_like(w["b2"])
        self.k = cfg.mlp_k or cfg.hidden
        self.stats = None
        self.aidx = None
        self.midx = None

    def _heads(self, t):
        c = self.cfg
        return np.ascontiguousarray(
            t.reshape(c.batch, c.seq, c.heads_local, c.head_dim).transpose(0, 2, 1, 3))

    def attn_partial(self, x, dense):
        P, c = self.port, self.cfg
        x = x.numpy()
        q, k, v = (self._heads(P.project(x, w)) for w in (self.wq, self.wk, self.wv))
        if dense:
            o, cs, self.stats = P.column_sum_attention(q, k, v, self.stats, c.chunk)
            self.aidx = P.select_top_k(cs, c.attn_k)
            self.acnt = np.full(self.aidx.shape[:-1], c.attn_k, np.int32)
            self.resid = P.sparse_delta_attention(q, k, v, self.aidx, self.acnt, c.chunk, o, -1.0)
        else:
            if self.aidx is None:
                raise RuntimeError("sparse attention step requested before any dense step")
            o = P.sparse_delta_attention(q, k, v, self.aidx, self.acnt, c.chunk, self.resid, 1.0)
        merged = np.ascontiguousarray(o.transpose(0, 2, 1, 3)).reshape(c.batch, c.seq, -1)
        return torch.from_numpy(P.project(merged, self.wo))

    def residual_add(self, x, partial, out=None):
        r = x + partial
        if out is not None:
            out.copy_(r)
            return out
        return r

    def mlp_dense_partial(self, x1):
        P, c = self.port, self.cfg
        x1 = x1.numpy()
        self.out, _, self.act = P.dense_mlp(x1, self.w1, self.b1, self.w2, self.b2)
        self.tm = P.mlp_tile_means(x1, self.w1, c.chunk)
        return torch.from_numpy(self.out.copy())

    def mlp_candidates(self, x1):
        c = self.cfg
        t = self.port.mlp_tile_means(x1.numpy(), self.w1, c.chunk)
        s = np.abs(t - self.tm).reshape(-1, c.f_local)  # mlp.cpp:116
        cs, ci = candidates(self.port, s, self.k, c.f0)
        return torch.from_numpy(cs), torch.from_numpy(ci)

    def mlp_sparse_partial(self, x1, all_s, all_i):
        c = self.cfg
        idx, cnt = merge(self.port, all_s.numpy(), all_i.numpy(), self.k, c.f0, c.f_local)
        nc = c.seq // c.chunk
        self.midx = (idx.reshape(c.batch, 1, nc, self.k), cnt.reshape(c.batch, 1, nc))
        self.out, self.act = self.port.sparse_delta_mlp(
            x1.numpy(), self.w1, self.b1, self.w2, self.b2, self.midx[0], self.midx[1], c.chunk,
            self.act, self.out)
        return torch.from_numpy(self.out.copy())


def golden_setup(g):
    from paper_2506_03275_b200.ops import BlockConfig
    misc, grid = g["cfg_misc"], g["cfg_grid"]
    cfg = BlockConfig(batch=int(misc[0]), seq=int(np.prod(grid)), dim=int(misc[1]),
                      heads=int(misc[3]), head_dim=int(misc[2]), hidden=int(misc[4]),
                      chunk=int(misc[5]), attn_k=int(g["ks"][0]), mlp_k=int(g["ks"][1]))
    w = {k[2:]: g[k] for k in g if k.startswith("w_")}
    return cfg, w


def run_schedule(block, shard, g):
    """Drive a ShardedBlock over the golden schedule; returns outputs and global MLP ids."""
    ys, mids = [], []
    for t, dense in enumerate(g["sched"]):
        y = block.step(torch.from_numpy(g[f"x{t}"]), bool(dense))
        ys.append(y.numpy().copy())
        if not dense:
            idx, cnt = shard.midx
            mids.append([sorted(int(a) + shard.cfg.f0 for a in idx.reshape(-1, idx.shape[-1])[r][:n])
                         for r, n in enumerate(cnt.reshape(-1))])
        else:
            mids.append(None)
    return ys, mids


def gloo_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    from paper_2506_03275_b200.shard import ShardedBlock, TorchComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        g = dict(np.load(os.path.join(HERE, "golden", "block.npz")))
        cfg, w = golden_setup(g)
        shard = OracleShard(cfg, w, world, rank)
        blk = ShardedBlock(cfg, w, TorchComm(), shard=shard)
        ys, mids = run_schedule(blk, shard, g)
        with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as fh:
            pickle.dump((ys, mids), fh)
    finally:
        dist.destroy_process_group()
