"""Per-CTA [start, end] globaltimer spans of the sparse attention kernel at FLUX / 93 %
(csd_debug_set_attn_pp_span): launch time by CUDA events next to the CTA start skew and the
end-time distribution, L2-flushed and back-to-back.
    python scripts/attn_span.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03275_b200 import _capi, ops  # noqa: E402


def main():
    cfg = dict(bench.FLUX)
    n = cfg["grid"][1] * cfg["grid"][2]
    ak = bench.k_of(n, 0.93)
    h, e, c = cfg["heads"], cfg["head_dim"], cfg["chunk"]
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v, base = (torch.randn((1, n, h, e), device="cuda", generator=g).to(torch.bfloat16)
                     for _ in range(4))
    r = ops.column_sum_attention(q, k, v, None, c, layout=1)
    idx = ops.select_top_k(r.column_sums, ak, c)
    ops.context().set_validation(False)
    out = torch.empty_like(base)
    run = lambda: ops.sparse_delta_attention(q, k, v, idx, base, 1.0, layout=1, out=out)  # noqa: E731
    for _ in range(3):
        run()
    fn = _capi.lib().csd_debug_set_attn_pp_span
    fn.argtypes = [ctypes.c_void_p]
    span = torch.zeros(2 * 148, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    for mode in ("flushed", "back-to-back"):
        for rep in range(3):
            if mode == "flushed":
                flush.fill_(1.0)
            else:
                run()
            span.zero_()
            fn(span.data_ptr())
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            run()
            ev1.record()
            torch.cuda.synchronize()
            fn(None)
            s = span.view(148, 2).cpu().tolist()
            t0 = min(a for a, b in s)
            st = sorted((a - t0) / 1e3 for a, b in s)
            en = sorted((b - t0) / 1e3 for a, b in s)
            print(f"{mode:13s} launch {ev0.elapsed_time(ev1) * 1e3:6.1f} us | start skew {st[-1]:5.1f} us | "
                  f"end min {en[0]:5.1f} p10 {en[14]:5.1f} p50 {en[74]:5.1f} p90 {en[133]:5.1f} max {en[-1]:5.1f} us")
    # which CTAs end last
    ends = [((b - t0) / 1e3, i) for i, (a, b) in enumerate(s)]
    ends.sort()
    print("last 10 CTAs (end us, cta):", [(round(x, 1), i) for x, i in ends[-10:]])
    print("first 10 CTAs (end us, cta):", [(round(x, 1), i) for x, i in ends[:10]])


if __name__ == "__main__":
    main()
