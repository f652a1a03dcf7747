"""The hand-written tcgen05 GEMMs (gemm_tc.cu) against plain PyTorch fp32 references.

Projections (model.cpp:107-120) and the dense MLP (mlp.cpp:49-81) run in PROD mode on
bf16 inputs; the reference is the same op in float32 on the same bf16-rounded tensors.
Tolerance: relative L2 <= 1e-2 (bf16 output rounding is ~4e-3).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops(cuda):
    from paper_2506_03275_b200 import ops as _ops
    return _ops


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm())


def gelu(v):
    return 0.5 * v * (1.0 + torch.tanh(0.7978845608028654 * (v + 0.044715 * v ** 3)))


@pytest.mark.parametrize("rows,d,dout", [(256, 256, 512), (1024, 768, 768), (4608, 3072, 3072),
                                         (512, 384, 192), (384, 128, 64)])
def test_project_vs_torch(ops, rows, d, dout):
    g = torch.Generator(device="cuda").manual_seed(rows + d)
    x = torch.randn((1, rows, d), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((d, dout), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    y = ops.project(x, w)
    ref = x.float() @ w.float()
    assert y.dtype == torch.bfloat16
    assert rel(y.float(), ref) < 1e-2


@pytest.mark.parametrize("b,n,d,f,chunk", [(1, 1024, 768, 3072, 64), (1, 4608, 3072, 12288, 192),
                                           (2, 512, 256, 1024, 128), (1, 768, 256, 512, 256),
                                           (1, 512, 384, 1280, 64)])
def test_dense_mlp_vs_torch(ops, b, n, d, f, chunk):
    g = torch.Generator(device="cuda").manual_seed(n + f)
    x = torch.randn((b, n, d), device="cuda", generator=g).to(torch.bfloat16)
    w1 = (torch.randn((f, d), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    w2 = (0.5 * torch.randn((f, d), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    b1 = 0.1 * torch.randn(f, device="cuda", generator=g)
    b2 = 0.1 * torch.randn(d, device="cuda", generator=g)
    wts = ops.MlpWeights(w1, b1, w2, b2)
    out, act = ops.dense_mlp(x, wts, chunk)
    pre = x.float() @ w1.float().t() + b1
    a = gelu(pre)
    ref = a.to(torch.bfloat16).float() @ w2.float() + b2
    assert rel(out, ref) < 1e-2
    # chunk-major activation cache [B, C, F, chunk]
    cm_ref = a.view(b, n // chunk, chunk, f).permute(0, 1, 3, 2)
    assert rel(act.float(), cm_ref) < 1e-2
