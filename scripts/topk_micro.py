"""Top-k micro-benchmark on the FLUX selection shapes (debug / ncu target):
MLP change scores [24 x 12288] k = 860 and attention column sums [576 x 4608] k = 323."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03275_b200 import ops  # noqa: E402


def main():
    prof = len(sys.argv) > 1 and sys.argv[1] == "--profile"
    trace = len(sys.argv) > 1 and sys.argv[1] == "--trace"
    g = torch.Generator(device="cuda").manual_seed(3)
    cases = [("mlp", 24, 12288, 860, 1), ("attn", 576, 4608, 323, 192)]
    res = {}
    for name, rows, m, k, chunk in cases:
        s = torch.rand((1, 1, rows, m), device="cuda", generator=g).abs() * 3 + 1
        ops.select_top_k(s, k, chunk)
        torch.cuda.synchronize()
        if trace:
            import ctypes
            from paper_2506_03275_b200 import _capi
            fn = _capi.lib().csd_debug_set_topk_trace
            fn.argtypes = [ctypes.c_void_p]
            buf = torch.zeros(8, dtype=torch.int64, device="cuda")
            fn(buf.data_ptr())
            ops.context().set_sorted_topk(False)
            ops.select_top_k(s, k, chunk)
            ops.context().set_sorted_topk(True)
            torch.cuda.synchronize()
            fn(None)
            t = buf.cpu().tolist()
            print(name, " ".join("%.2f" % ((x - t[0]) / 1965.0) for x in t))
            continue
        if prof:
            torch.cuda.profiler.start()
            ops.select_top_k(s, k, chunk)
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            ops.select_top_k(s, k, chunk)
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 2)
    if not prof:
        print(json.dumps({"us": res}))


if __name__ == "__main__":
    main()
