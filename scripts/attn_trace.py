"""Per-CTA timeline of one column-sparse attention launch on the FLUX shape (debug).

Uses csd_debug_set_attn_trace (attn_tc.cu): CTAs 0..7 stamp clock64() at fixed slots.
Prints, per CTA, the phase times in microseconds relative to kernel entry.
    python scripts/attn_trace.py [--dense]
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

SLOTS = 1024
GHZ = 1.965


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sparsity", type=float, default=0.93)
    ap.add_argument("--ctas", type=int, default=3)
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
    for _ in range(3):
        ops.sparse_delta_attention(q, k, v, idx, base, 1.0, layout=1, out=out)
    lib = _capi.lib()
    fn = lib.csd_debug_set_attn_trace
    fn.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(8 * SLOTS, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    fn(buf.data_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ops.sparse_delta_attention(q, k, v, idx, base, 1.0, layout=1, out=out)
    ev1.record()
    torch.cuda.synchronize()
    fn(None)
    print("launch %.1f us (traced)" % (ev0.elapsed_time(ev1) * 1e3))
    # untraced launch with per-CTA spans
    fs = lib.csd_debug_set_attn_span
    fs.argtypes = [ctypes.c_void_p]
    span = torch.zeros(2 * 148, dtype=torch.int64, device="cuda")
    fs(span.data_ptr())
    ops.sparse_delta_attention(q, k, v, idx, base, 1.0, layout=1, out=out)
    torch.cuda.synchronize()
    fs(None)
    sp = span.view(148, 2).cpu().tolist()
    t0 = min(a for a, _ in sp)
    ends = sorted(((e - t0) / 1e3, i) for i, (_, e) in enumerate(sp))
    print("CTA end times (us): min %.1f  median %.1f  max %.1f; slowest CTAs %s" % (
        ends[0][0], ends[len(ends) // 2][0], ends[-1][0], [i for _, i in ends[-6:]]))
    print("  start spread %.1f us" % ((max(a for a, _ in sp) - t0) / 1e3))
    t = buf.view(8, SLOTS).cpu().tolist()
    for cta in range(args.ctas):
        row = t[cta]
        t0 = row[0]

        def us(s):
            return "%7.2f" % ((row[s] - t0) / GHZ / 1e3) if row[s] else "      -"
        print(f"--- CTA {cta}: setup done {us(1)}")
        for li in range(5):
            if not row[8 + li]:
                continue
            print(f" item {li}: Q issue {us(2 + li)}  Q ready(MMA) {us(8 + li)}  "
                  f"epi start {us(240 + li)}  rmw done {us(232 + li)}  epi end {us(248 + li)}")
        for gbk in range(16):
            if not row[16 + gbk]:
                continue
            print(f"  blk {gbk:2d}: K issue {us(16 + gbk)} KV issued {us(48 + gbk)} | S issue "
                  f"{us(80 + gbk)} | t0 S-ready {us(144 + gbk)} "
                  f"P-done {us(168 + gbk)}")


if __name__ == "__main__":
    main()
