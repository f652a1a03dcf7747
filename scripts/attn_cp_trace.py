"""Per-block timeline of the CTA-pair sparse attention kernel (k_attn_cp, debug).

csd_debug_set_attn_cp_trace: CTAs 0..3 stamp clock64() at slot event * 64 + index.
Prints for CTAs 0 and 1 (the first pair) every key block's events in kilocycles from entry.
    python scripts/attn_cp_trace.py [--blocks 30] [--flush]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03275_b200 import _capi, ops  # noqa: E402

EV = ["cpK", "cpV", "rlK", "rlV", "mS", "mP", "mPV", "sS", "sM", "sP"]
EV2 = [(15, "c0"), (16, "c1"), (17, "stw"), (18, "bS"), (19, "bM"), (20, "bc0"), (21, "bc1"), (22, "bstw"), (23, "bP")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=30)
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--sparsity", type=float, default=0.93)
    args = ap.parse_args()
    cfg = dict(bench.FLUX)
    n = cfg["grid"][1] * cfg["grid"][2]
    ak = bench.k_of(n, args.sparsity)
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
    fn = _capi.lib().csd_debug_set_attn_cp_trace
    fn.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(4 * 2048, dtype=torch.int64, device="cuda")
    if args.flush:
        torch.empty(64 * 1024 * 1024, device="cuda").fill_(1.0)
    torch.cuda.synchronize()
    fn(buf.data_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    run()
    ev1.record()
    torch.cuda.synchronize()
    fn(None)
    print("launch %.1f us (traced)" % (ev0.elapsed_time(ev1) * 1e3))
    t = buf.view(4, 2048).cpu().tolist()
    for cta in range(2):
        row = t[cta]
        t0 = row[31 * 64]

        def kc(ev, i):
            v = row[ev * 64 + (i & 63)]
            return "%6.1f" % ((v - t0) / 1e3) if v else "     -"
        print(f"--- CTA {cta} (kcycles from entry)")
        print("  Q issue per item:", " ".join(kc(12, li) for li in range(10)))
        print("  epilogue [start end] per item:", " ".join(f"[{kc(10, li)} {kc(11, li)}]" for li in range(10)))
        print("    g " + " ".join(f"{nm:>6s}" for nm in EV + [x for _, x in EV2]))
        for gi in range(args.blocks):
            if not any(row[ev * 64 + gi] for ev in range(10)):
                continue
            print(f"  {gi:3d} " + " ".join(kc(ev, gi) for ev in list(range(10)) + [e for e, _ in EV2]))


if __name__ == "__main__":
    main()
