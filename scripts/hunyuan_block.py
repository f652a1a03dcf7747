"""HunyuanVideo-shaped block (BASELINE.json configs[3]) end to end on one B200.

    python scripts/hunyuan_block.py [--world 1] [--out profiles/r02_hunyuan_block.json]

Latent grid 32 x 42 x 88 = 118 272 tokens, voxel 4 x 6 x 8 reorder (voxel.cpp), D 3072,
24 x 128 heads, MLP 12 288, chunk 192, 95 % sparsity (attn k 5914, MLP k 614), random-init
weights.  Runs the schedule D, S, S, D, S through the device-resident block (or, with
--world g, the token-sharded path: g shards simulated on this GPU), timing each
step with CUDA events.  Parity on the dense steps is a CHECK sub-sample: the block output of
sampled query chunks against a float32 PyTorch restatement of model.cpp:178-216 for those
rows (full-length keys, all heads, the block's bf16-rounded weights), relative L2 over the
block's branch (y - x).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03275_b200 import ops  # noqa: E402

HUNYUAN = dict(batch=1, grid=(32, 42, 88), voxel=(4, 6, 8), dim=3072, heads=24, head_dim=128,
               hidden=12288, chunk=192, sparsity=0.95)


def gelu(v):
    return 0.5 * v * (1.0 + torch.tanh(0.7978845608028654 * (v + 0.044715 * v ** 3)))


def reference_rows(x, w, rows, heads, e):
    """model.cpp:178-216 for the given token rows, float32 (dense attention over all keys)."""
    xf = x[0].float()
    k = xf @ w["wk"]
    v = xf @ w["wv"]
    q = xf[rows] @ w["wq"]
    outs = []
    for h in range(heads):
        sl = slice(h * e, (h + 1) * e)
        s = (q[:, sl] @ k[:, sl].t()) / np.sqrt(e)
        p = torch.softmax(s, dim=-1)
        outs.append(p @ v[:, sl])
    attn = torch.cat(outs, dim=1)
    x_mid = xf[rows] + attn @ w["wo"]
    m = gelu(x_mid @ w["w1"].t() + w["b1"]) @ w["w2"] + w["b2"]
    return x_mid + m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_hunyuan_block.json"))
    ap.add_argument("--sample-chunks", type=int, nargs="*", default=[0, 307, 615])
    args = ap.parse_args()
    cfg = dict(HUNYUAN)
    t_, hh, ww = cfg["grid"]
    n = t_ * hh * ww
    ak, mk = bench.k_of(n, cfg["sparsity"]), bench.k_of(cfg["hidden"], cfg["sparsity"])
    bc = ops.BlockConfig(batch=1, seq=n, dim=cfg["dim"], heads=cfg["heads"],
                         head_dim=cfg["head_dim"], hidden=cfg["hidden"], chunk=cfg["chunk"],
                         attn_k=ak, mlp_k=mk)
    weights = bench.make_weights(cfg)
    dev = torch.device("cuda")
    # the block's bf16-rounded weights, float32 on the device (the reference restatement's)
    wref = {k: (torch.as_tensor(v).to(dev).to(torch.bfloat16).float() if k not in ("b1", "b2")
                else torch.as_tensor(v).to(dev)) for k, v in weights.items()}
    if args.world > 1:
        from paper_2506_03275_b200.shard import simulate_token_step, token_shard_config
        blocks = [ops.Block(token_shard_config(bc, args.world, r), weights, production=True)
                  for r in range(args.world)]

        def step(x, dense):
            return simulate_token_step(blocks, x, dense)
    else:
        blk = ops.Block(bc, weights, production=True)

        def step(x, dense):
            return blk.step(x, dense)

    # latent: N(0,1) on the video grid, voxel-ordered (voxel.cpp) -- the sequence the block sees
    g = torch.Generator(device=dev).manual_seed(1235)
    lat = torch.randn((1, t_, hh, ww, cfg["dim"]), device=dev, generator=g)
    layout = ops.VoxelLayout(t_, hh, ww, *cfg["voxel"])
    x0, _ = ops.voxel_order(lat.to(torch.bfloat16), layout)
    del lat
    rows = torch.cat([torch.arange(c * cfg["chunk"], (c + 1) * cfg["chunk"]) for c in args.sample_chunks]).to(dev)
    sched = [1, 0, 0, 1, 0]
    res = {"config": {"workload": "HunyuanVideo-shaped DiT block (BASELINE configs[3])", "tokens": n,
                      "grid": list(cfg["grid"]), "voxel": list(cfg["voxel"]), "dim": cfg["dim"],
                      "heads": cfg["heads"], "head_dim": cfg["head_dim"], "hidden": cfg["hidden"],
                      "chunk": cfg["chunk"], "sparsity": cfg["sparsity"], "attn_k": ak, "mlp_k": mk,
                      "world": args.world,
                      "path": "token-sharded (simulated shards)" if args.world > 1 else "single block"},
           "steps": []}
    x = x0
    for t, dense in enumerate(sched):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y = step(x, bool(dense))
        e1.record()
        torch.cuda.synchronize()
        rec = {"step": t, "kind": "dense" if dense else "sparse", "ms": round(e0.elapsed_time(e1), 3)}
        if dense:
            ref = reference_rows(x, wref, rows, cfg["heads"], cfg["head_dim"])
            got = y[0, rows].float()
            xr = x[0, rows].float()
            rec["parity_rel_l2_branch"] = float((got - ref).norm() / (ref - xr).norm())
            rec["parity_rows"] = f"chunks {args.sample_chunks} x all heads (float32 restatement)"
        res["steps"].append(rec)
        print(json.dumps(rec), flush=True)
        x = (x.float() + y.float() * (1.0 / 50)).to(torch.bfloat16)  # harness.cpp:200
    # second pass over the same schedule kinds: warm timings
    warm = {}
    for dense in (1, 0):
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step(x, bool(dense))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        warm["dense_ms" if dense else "sparse_ms"] = round(min(ts), 3)
    res["warm"] = warm
    res["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    print(json.dumps(res["warm"]))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
