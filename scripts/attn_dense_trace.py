"""Per-block timeline of the dense attention pipeline, one item per CTA (debug).

Dense attention with 256-row items (NT = 2, both tiles live) on 8 heads x 4608 tokens
(144 items <= 148 SMs).  Prints, for CTA 0, per 128-key block: MMA S issue / S ready /
P done / PV issue for each tile, and K / V ready, in SM cycles relative to the first S.
    python scripts/attn_dense_trace.py [--heads 8] [--blocks 12]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_03275_b200 import _capi, ops  # noqa: E402

SLOTS = 1024


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--n", type=int, default=4608)
    ap.add_argument("--blocks", type=int, default=12)
    ap.add_argument("--cta", type=int, default=0)
    ap.add_argument("--colsum", type=int, default=0, help="column-sum chunk (0: plain dense)")
    args = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn((1, args.n, args.heads, 128), device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(3))
    stats = None
    if args.colsum:
        r0 = ops.column_sum_attention(q, k, v, None, args.colsum, layout=1)
        stats = r0.stats

    def launch():
        if args.colsum:
            return ops.column_sum_attention(q, k, v, stats, args.colsum, layout=1)
        return ops.dense_attention(q, k, v, layout=1)
    for _ in range(3):
        launch()
    lib = _capi.lib()
    fn = lib.csd_debug_set_attn_trace
    fn.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(8 * SLOTS, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    fn(buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launch()
    e1.record()
    torch.cuda.synchronize()
    fn(None)
    ms = e0.elapsed_time(e1)
    fl = 4.0 * args.heads * args.n * args.n * 128
    print(f"traced launch {ms * 1e3:.1f} us  ({fl / ms / 1e9:.0f} TF/s)")
    row = buf.view(8, SLOTS)[args.cta].cpu().tolist()
    t0 = row[512 + 0] or row[80]
    c = lambda s: (row[s] - t0) if row[s] else None  # noqa: E731
    print("blk | S0 iss  S0 rdy  P0 done PV0 iss | S1 iss  S1 rdy  P1 done PV1 iss |  K rdy   V rdy")
    prev = None
    for b in range(args.blocks):
        vals = [c(512 + b), c(256 + b), c(384 + b), c(640 + b),
                c(512 + 64 + b), c(256 + 64 + b), c(384 + 64 + b), c(640 + 64 + b),
                c(768 + b), c(832 + b)]
        f = lambda x: f"{x:7d}" if x is not None else "      -"  # noqa: E731
        print(f"{b:3d} | " + " ".join(f(x) for x in vals[:4]) + " | " + " ".join(f(x) for x in vals[4:8])
              + " | " + " ".join(f(x) for x in vals[8:]))
    # steady-state per-block period and phase lengths (tile 0 and 1)
    import statistics
    for t in range(2):
        per = [row[256 + 64 * t + b + 1] - row[256 + 64 * t + b] for b in range(2, args.blocks - 1)]
        sm = [row[384 + 64 * t + b] - row[256 + 64 * t + b] for b in range(2, args.blocks - 1)]
        wait = [row[256 + 64 * t + b + 1] - row[384 + 64 * t + b] for b in range(2, args.blocks - 1)]
        print(f"tile {t}: period {statistics.median(per)} cyc, softmax {statistics.median(sm)} cyc, "
              f"P-done -> next S ready {statistics.median(wait)} cyc")


if __name__ == "__main__":
    main()
