"""FLUX-shaped block at 85-95 % sparsity (north_star: "the speedup over the dense path at
85-95 % sparsity"): the sparse-delta MLP micro-benchmark (bench.mlp_kernel_bench, L2 flushed)
and the block's sparse step (one CUDA graph replay, CUDA events) per sparsity, next to the
dense step.
    python scripts/sparsity_sweep.py [--out gpurun_out/sparsity_sweep.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03275_b200 import ops  # noqa: E402


def step_ms(blk, x, dense, reps=20):
    y = torch.empty_like(x)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        blk.step(x, dense, out=y)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        blk.step(x, dense, out=y)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sparsity_sweep.json"))
    ap.add_argument("--sparsities", default="0.85,0.9,0.93,0.95")
    args = ap.parse_args()
    cfg = dict(bench.FLUX)
    n = cfg["grid"][0] * cfg["grid"][1] * cfg["grid"][2]
    w = bench.make_weights(cfg)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((1, n, cfg["dim"]), device="cuda", generator=g).to(torch.bfloat16)
    rows = []
    for sp in [float(v) for v in args.sparsities.split(",")]:
        ak, mk = bench.k_of(n, sp), bench.k_of(cfg["hidden"], sp)
        bc = ops.BlockConfig(batch=1, seq=n, dim=cfg["dim"], heads=cfg["heads"], head_dim=cfg["head_dim"],
                             hidden=cfg["hidden"], chunk=cfg["chunk"], attn_k=ak, mlp_k=mk)
        blk = ops.Block(bc, w, production=True)
        blk.step(x, True)
        dense = step_ms(blk, x, True)
        sparse = step_ms(blk, x, False)
        mlp = bench.mlp_kernel_bench(ops, torch, cfg, n, mk, 10)
        row = {"sparsity": sp, "attn_k": ak, "mlp_k": mk, "dense_step_ms": round(dense, 4),
               "sparse_step_ms": round(sparse, 4), "step_speedup": round(dense / sparse, 3),
               "mlp_sparse_ms": mlp["sparse"]["ms"], "mlp_dense_ms": mlp["dense"]["ms"],
               "mlp_speedup": mlp["speedup_vs_dense"], "mlp_eff_tflops": mlp["sparse"]["eff_tflops"],
               "mlp_dense_equiv_tflops": mlp["sparse"]["dense_equiv_tflops"]}
        print(json.dumps(row), flush=True)
        rows.append(row)
        blk.close()
        torch.cuda.empty_cache()
    with open(args.out, "w") as f:
        json.dump({"device": torch.cuda.get_device_name(), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
