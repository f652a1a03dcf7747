"""Per-block timeline of the ping-pong attention kernel (k_attn_pp, debug).

csd_debug_set_attn_pp_trace: CTAs 0..7 stamp clock64() at slot event * 64 + index.
Prints, for a few CTAs, every key block's events in kilocycles from kernel entry.
    python scripts/attn_pp_trace.py [--dense] [--ctas 2]
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

EV = ["cpK", "cpV", "mP0", "mV", "mQ", "mS0", "mP1", "s0S", "s0P", "s1S", "s1P"]
# softmax sub-phases: S loaded, max done, exps done (tile 0, tile 1)
EV2 = [(16, "s0L"), (18, "s0M"), (20, "s0E"), (17, "s1L"), (19, "s1M"), (21, "s1E")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sparsity", type=float, default=0.93)
    ap.add_argument("--ctas", type=int, default=2)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--blocks", type=int, default=40)
    ap.add_argument("--back-to-back", action="store_true",
                    help="trace a launch issued right after an identical one (warm caches)")
    ap.add_argument("--flush", action="store_true", help="write 256 MB before the traced launch")
    ap.add_argument("--in-step", action="store_true",
                    help="trace the attention launch inside a FLUX block sparse step")
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
    run = (lambda: ops.dense_attention(q, k, v, layout=1)) if args.dense else (
        lambda: ops.sparse_delta_attention(q, k, v, idx, base, 1.0, layout=1, out=out))
    for _ in range(3):
        run()
    lib = _capi.lib()
    fn = lib.csd_debug_set_attn_pp_trace
    fn.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(8 * 2048, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    fn(buf.data_ptr())
    if args.flush:
        torch.empty(64 * 1024 * 1024, device="cuda").fill_(1.0)
    if args.back_to_back:
        fn(None)
        run()  # untraced, immediately before
        fn(buf.data_ptr())
    if args.in_step:
        fn(None)
        bc = ops.BlockConfig(batch=1, seq=n, dim=cfg["dim"], heads=h, head_dim=e, hidden=cfg["hidden"],
                             chunk=c, attn_k=ak, mlp_k=bench.k_of(cfg["hidden"], args.sparsity))
        blk = ops.Block(bc, bench.make_weights(cfg), production=True)
        xb = torch.randn((1, n, cfg["dim"]), device="cuda", generator=g).to(torch.bfloat16)
        blk.step(xb, True)
        blk.step(xb, False)
        blk.step(xb, False)
        torch.cuda.synchronize()
        fn(buf.data_ptr())
        run = lambda: blk.step(xb, False)  # noqa: E731
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    run()
    ev1.record()
    torch.cuda.synchronize()
    fn(None)
    print("launch %.1f us (traced)" % (ev0.elapsed_time(ev1) * 1e3))
    t = buf.view(8, 2048).cpu().tolist()
    for cta in range(args.ctas):
        row = t[cta]
        t0 = row[15 * 64]

        def kc(ev, i):
            v = row[ev * 64 + (i & 63)]
            return "%6.1f" % ((v - t0) / 1e3) if v else "     -"
        print(f"--- CTA {cta} (kcycles from entry)")
        print("  Q issue t0/t1 per item:", " ".join(f"{kc(13, li)}/{kc(14, li)}" for li in range(6)))
        print("  epilogue t0 [start end] per item:",
              " ".join(f"[{kc(11, 2 * li)} {kc(11, 2 * li + 1)}]" for li in range(6)))
        print("  item set-up t0 / t1:", " ".join(f"{kc(22, li)}/{kc(23, li)}" for li in range(6)))
        print("  epilogue t1 [start end] per item:",
              " ".join(f"[{kc(12, 2 * li)} {kc(12, 2 * li + 1)}]" for li in range(6)))
        print("    g " + " ".join(f"{n:>6s}" for n in EV) + " " + " ".join(f"{n:>6s}" for _, n in EV2))
        for gi in range(args.blocks):
            if not any(row[ev * 64 + gi] for ev in range(11)):
                continue
            print(f"  {gi:3d} " + " ".join(kc(ev, gi) for ev in range(11)) + " " + " ".join(kc(ev, gi) for ev, _ in EV2))


if __name__ == "__main__":
    main()
