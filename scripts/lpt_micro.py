"""LPT item order on a ragged index set (FLUX shape, counts uniform in [0, 2k]):
sparse attention with and without the longest-first order, and parity of the two."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_03275_b200 import ops  # noqa: E402


def main():
    n, h, e, c, k = 4608, 24, 128, 192, 646
    g = torch.Generator(device="cuda").manual_seed(5)
    q, kk, v, base = (torch.randn((1, n, h, e), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    nc = n // c
    cnt = torch.randint(0, k + 1, (1, h, nc), device="cuda", generator=g, dtype=torch.int32)
    idx = torch.stack([torch.randperm(n, device="cuda", generator=g)[:k] for _ in range(h * nc)]).view(1, h, nc, k).to(torch.int32)
    s = ops.SparseIndexSet(1, h, nc, c, k, n, idx, cnt)
    ctx = ops.context()
    res = {}
    outs = {}
    for lpt in (1, 0):
        ctx.lib.csd_ctx_set_lpt(ctx.h, lpt)
        out = torch.empty_like(base)
        fn = lambda: ops.sparse_delta_attention(q, kk, v, s, base, 1.0, layout=1, out=out)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res["lpt" if lpt else "strided"] = round(statistics.median(ts) * 1e3, 1)
        outs[lpt] = out.clone()
    ctx.lib.csd_ctx_set_lpt(ctx.h, 1)
    res["identical"] = bool(torch.equal(outs[0], outs[1]))
    res["unit"] = "us (incl. validation + order kernels)"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
