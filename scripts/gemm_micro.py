"""FLUX-shape GEMM timings through the public ops (CUDA-graph replays, L2 flushed between
reps): one projection [4608 x 3072] @ [3072 x 3072] and the dense MLP (D 3072, F 12288,
chunk 192).  Run with CSD_GEMM=cublas for the library baseline."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_03275_b200 import ops  # noqa: E402


def timed(fn, reps=20):
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        fn()
    s.wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for i in range(reps + 3):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])


def main():
    n, d, f, c = 4608, 3072, 12288, 192
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((1, n, d), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((d, d), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    w1 = (torch.randn((f, d), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn((f, d), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    b1 = torch.zeros(f, device="cuda")
    b2 = torch.zeros(d, device="cuda")
    wts = ops.MlpWeights(w1, b1, w2, b2)
    t_proj = timed(lambda: ops.project(x, w))
    t_mlp = timed(lambda: ops.dense_mlp(x, wts, c))
    fl_proj = 2.0 * n * d * d
    fl_mlp = 4.0 * n * d * f
    print(json.dumps({"gemm": os.environ.get("CSD_GEMM", "tc"),
                      "proj_ms": round(t_proj, 4), "proj_tflops": round(fl_proj / t_proj / 1e9, 1),
                      "mlp_ms": round(t_mlp, 4), "mlp_tflops": round(fl_mlp / t_mlp / 1e9, 1)}))


if __name__ == "__main__":
    main()
