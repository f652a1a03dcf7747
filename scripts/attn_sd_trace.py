"""Per-block timeline of the dense-pass kernel k_attn_sd (debug): MMA S issue / P seen,
softmax S ready / max exchanged / P written for the two row halves of quadrant 0.
    python scripts/attn_sd_trace.py [--colsum]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03275_b200 import _capi, ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--colsum", action="store_true")
    args = ap.parse_args()
    n, h, e = 4608, 24, 128
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn((1, n, h, e), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    st = ops.column_sum_attention(q, k, v, None, 192, layout=1).stats
    run = (lambda: ops.column_sum_attention(q, k, v, st, 192, layout=1)) if args.colsum else (
        lambda: ops.dense_attention(q, k, v, layout=1))
    for _ in range(2):
        run()
    fn = _capi.lib().csd_debug_set_attn_sd_trace
    fn.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(8 * 2048, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    fn(buf.data_ptr())
    run()
    torch.cuda.synchronize()
    fn(None)
    row = buf.view(8, 2048)[0].cpu().tolist()
    t0 = min(x for x in row if x) if any(row) else 0
    names = ["mS_iss", "mP_seen", "sm0_S", "sm1_S", "sm0_P", "sm1_P", "sm0_xch"]
    print("   g " + " ".join(f"{x:>8s}" for x in names) + "   (kcycles from the first stamp)")
    for gi in range(40):
        vals = [row[ev * 64 + gi] for ev in range(7)]
        if not any(vals):
            continue
        print(f"{gi:4d} " + " ".join(f"{(v - t0) / 1e3:8.2f}" if v else "       -" for v in vals))


if __name__ == "__main__":
    main()
