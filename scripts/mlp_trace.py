"""Timelines of the FLUX sparse step's MLP kernels (debug).

k_smlp_up: CTAs (x<8, y=0) stamp clock64() per k-block (producer issue, MMA data-ready) and
around the epilogue.  k_smlp_down: CTAs x<8 stamp each persistent item's K loop and epilogue.
k_topk_cluster: CTA 0's phases.  x is perturbed between steps so every chunk has its own
index set (the generation trajectory, not a repeated input)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03275_b200 import _capi, ops  # noqa: E402

cfg = dict(bench.FLUX)
n = cfg["grid"][1] * cfg["grid"][2]
ak, mk = bench.k_of(n, cfg["sparsity"]), bench.k_of(cfg["hidden"], cfg["sparsity"])
bc = ops.BlockConfig(batch=1, seq=n, dim=cfg["dim"], heads=cfg["heads"], head_dim=cfg["head_dim"],
                     hidden=cfg["hidden"], chunk=cfg["chunk"], attn_k=ak, mlp_k=mk)
blk = ops.Block(bc, bench.make_weights(cfg), production=True)
x = torch.randn((1, n, cfg["dim"]), device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
g = torch.Generator(device="cuda").manual_seed(7)


def perturb(v):
    return (v.float() + 0.1 * torch.randn(v.shape, device="cuda", generator=g)).to(torch.bfloat16)


for dense in (True, False, False):
    blk.step(x, dense, out=y)
    x = perturb(x)
torch.cuda.synchronize()
tk = _capi.lib().csd_debug_set_topk_trace
tk.argtypes = [ctypes.c_void_p]
tbuf = torch.zeros(8, dtype=torch.int64, device="cuda")
tk(tbuf.data_ptr())
fn = _capi.lib().csd_debug_set_mlp_trace
fn.argtypes = [ctypes.c_void_p]
buf = torch.zeros(8 * 256, dtype=torch.int64, device="cuda")
fn(buf.data_ptr())
blk.step(x, False, out=y)
torch.cuda.synchronize()
fn(None)
tk(None)
tt = tbuf.cpu().tolist()
print("k_topk (last launch), CTA 0 phases [us]:", " ".join("%.2f" % ((v - tt[0]) / 1965.0) for v in tt))
t = buf.view(8, 256).cpu().tolist()
for cta in range(2):
    r = t[cta]
    t0 = r[0]
    us = lambda s: (r[s] - t0) / 1965.0 if r[s] else float("nan")  # noqa: E731
    print(f"CTA {cta}: setup {us(1):.2f}  epilogue {us(128):.2f} -> {us(129):.2f} us")
    print("  k-block issue :", " ".join(f"{us(2 + k):.1f}" for k in range(0, 48, 4)))
    print("  k-block ready :", " ".join(f"{us(64 + k):.1f}" for k in range(0, 48, 4)))
    print(f"  epilogue: act tile landed {us(130):.2f}  math done {us(131):.2f}")
print("k_smlp_down, CTAs 0-3 (persistent items) [us from CTA start]:")
for cta in range(4):
    r = t[cta]
    t0 = r[200]
    us = lambda s: (r[s] - t0) / 1965.0 if r[s] else float("nan")  # noqa: E731
    print(f" CTA {cta}: " + " | ".join(f"K {us(202 + 2 * li):.1f}-{us(203 + 2 * li):.1f} E {us(230 + 2 * li):.1f}-{us(231 + 2 * li):.1f}"
                                     for li in range(5) if r[202 + 2 * li]))
