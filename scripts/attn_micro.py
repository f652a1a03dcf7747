"""Column-sparse / dense attention micro-benchmark on the FLUX shape (bench.py's
attention_kernel_bench), with an optional profiler window around ONE sparse launch.

    python scripts/attn_micro.py                     # timings
    ncu --set full --import-source on --profile-from-start off -k regex:k_attn_tc \
        -o gpurun_out/attn python scripts/attn_micro.py --profile
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
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--sparsity", type=float, default=0.93)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between reps")
    ap.add_argument("--no-lpt", action="store_true", help="identity item order")
    args = ap.parse_args()
    cfg = dict(bench.FLUX)
    n = cfg["grid"][1] * cfg["grid"][2]
    ak = bench.k_of(n, args.sparsity)
    if args.profile:
        h, e, c = cfg["heads"], cfg["head_dim"], cfg["chunk"]
        g = torch.Generator(device="cuda").manual_seed(7)
        q, k, v, base = (torch.randn((1, n, h, e), device="cuda", generator=g).to(torch.bfloat16)
                         for _ in range(4))
        r = ops.column_sum_attention(q, k, v, None, c, layout=1)
        idx = ops.select_top_k(r.column_sums, ak, c)
        ops.context().set_validation(False)
        out = torch.empty_like(base)
        for _ in range(3):
            ops.sparse_delta_attention(q, k, v, idx, base, 1.0, layout=1, out=out)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        ops.sparse_delta_attention(q, k, v, idx, base, 1.0, layout=1, out=out)
        ops.dense_attention(q, k, v, layout=1)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    if args.no_lpt:
        ops.context().lib.csd_ctx_set_lpt(ops.context().h, 0)
    res = bench.attention_kernel_bench(ops, torch, cfg, n, ak, args.reps, flush_l2=not args.no_flush)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
