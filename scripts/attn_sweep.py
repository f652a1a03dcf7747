"""Column-sparse vs same-kernel-family dense attention sweep (BASELINE.json configs[2]):
sparsity 50-97 %, sequence 4K-32K, head_dim 128, FLUX heads (24), chunk 192 (N % 192 == 0)
or 128.  Inputs resident in HBM, L2 flushed between repetitions (bench.attention_kernel_bench).

    python scripts/attn_sweep.py [--out profiles/attn_sweep.json]
Prints one JSON line per (N, sparsity) and writes the table.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "attn_sweep.json"))
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--seqs", default="4608,9216,18432,32768")
    ap.add_argument("--sparsities", default="0.5,0.75,0.85,0.9,0.93,0.95,0.97")
    args = ap.parse_args()
    rows = []
    dense_cache = {}
    for n in [int(v) for v in args.seqs.split(",")]:
        chunk = 192 if n % 192 == 0 else 128
        cfg = dict(bench.FLUX, chunk=chunk)
        for sp in [float(v) for v in args.sparsities.split(",")]:
            k = bench.k_of(n, sp)
            r = bench.attention_kernel_bench(ops, torch, cfg, n, k, args.reps,
                                             dense_ms=dense_cache.get(n))
            dense_cache[n] = r["dense"]["ms"]
            row = {"n": n, "chunk": chunk, "heads": cfg["heads"], "head_dim": cfg["head_dim"],
                   "sparsity": sp, "k": k, "sparse_ms": r["sparse"]["ms"],
                   "dense_ms": r["dense"]["ms"], "speedup_vs_dense": r["speedup_vs_dense"],
                   "eff_tflops": r["sparse"]["eff_tflops"],
                   "dense_equiv_tflops": r["sparse"]["dense_equiv_tflops"],
                   "hbm_gbs_alg": round(r["sparse"]["alg_bytes"] / (r["sparse"]["ms"] * 1e-3) / 1e9, 1)}
            print(json.dumps(row), flush=True)
            rows.append(row)
    with open(args.out, "w") as f:
        json.dump({"device": torch.cuda.get_device_name(), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
