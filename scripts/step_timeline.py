"""Kernel timeline of graph-replayed FLUX block steps (torch.profiler / CUPTI activity
records): per-kernel start, duration and the gap to the previous kernel's end, warm caches,
trajectory-perturbed inputs.

    python scripts/step_timeline.py [--kind sparse|dense] [--reps 3]
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
    ap.add_argument("--kind", default="sparse", choices=["sparse", "dense"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    ap.add_argument("--hunyuan", action="store_true",
                    help="the HunyuanVideo-shaped block (configs[3]: 118272 tokens, 95 %%)")
    args = ap.parse_args()
    cfg = dict(bench.FLUX)
    n = cfg["grid"][1] * cfg["grid"][2]
    sp = cfg["sparsity"]
    if args.hunyuan:
        n, sp = 32 * 42 * 88, 0.95
    ak, mk = bench.k_of(n, sp), bench.k_of(cfg["hidden"], sp)
    bc = ops.BlockConfig(batch=1, seq=n, dim=cfg["dim"], heads=cfg["heads"],
                         head_dim=cfg["head_dim"], hidden=cfg["hidden"], chunk=cfg["chunk"],
                         attn_k=ak, mlp_k=mk)
    blk = ops.Block(bc, bench.make_weights(cfg), production=True)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((1, n, cfg["dim"]), device="cuda", generator=g).to(torch.bfloat16)
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for dense in (True, False, False):
            blk.step(x, dense, out=y)
            x.copy_((x.float() + 0.1 * torch.randn(x.shape, device="cuda", generator=g)).to(torch.bfloat16))
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        blk.step(x, args.kind == "dense", out=y)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.reps):
            gr.replay()
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    # split into replays at gaps > 20 us (long steps: one replay per synchronize anyway)
    reps, cur = [], []
    for e in evs:
        if cur and e.time_range.start - cur[-1].time_range.end > 20:
            reps.append(cur)
            cur = []
        cur.append(e)
    if cur:
        reps.append(cur)
    rep = reps[-1]
    t0 = rep[0].time_range.start
    rows, prev_end = [], None
    for e in rep:
        st, en = e.time_range.start, e.time_range.end
        gap = 0.0 if prev_end is None else st - prev_end
        name = e.name.replace("(anonymous namespace)::", "").replace("csd::dev::", "").replace("void ", "")
        rows.append({"kernel": name.split("(")[0][:60], "start_us": round(st - t0, 1),
                     "dur_us": round(en - st, 1), "gap_us": round(gap, 1)})
        prev_end = en if prev_end is None else max(prev_end, en)
    total = rep[-1].time_range.end - t0
    for r in rows:
        print(f"{r['start_us']:8.1f} {r['dur_us']:7.1f} gap {r['gap_us']:6.1f}  {r['kernel']}")
    print(f"span {total:.1f} us, kernels {sum(r['dur_us'] for r in rows):.1f} us, "
          f"gaps {sum(r['gap_us'] for r in rows):.1f} us ({args.kind} step, one graph replay)")
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"kind": args.kind, "span_us": round(total, 1), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
