"""Longest-first (LPT) work order of PROD sparse attention over ragged index sets
(attn_pp.cu k_lpt_order): the order moves items between CTAs only, so outputs must be
bit-identical with and without it, and both must match the CHECK path within tolerance."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops(cuda):
    from paper_2506_03275_b200 import ops as _ops
    return _ops


def test_lpt_order_bit_identical_on_ragged_counts(ops):
    n, h, e, c, k = 1536, 4, 128, 192, 300
    g = torch.Generator(device="cuda").manual_seed(11)
    q, kk, v, base = (torch.randn((1, n, h, e), device="cuda", generator=g).to(torch.bfloat16)
                      for _ in range(4))
    nc = n // c
    cnt = torch.randint(0, k + 1, (1, h, nc), device="cuda", generator=g, dtype=torch.int32)
    cnt[0, 0, 0] = 0  # an empty chunk passes base through
    idx = torch.stack([torch.randperm(n, device="cuda", generator=g)[:k] for _ in range(h * nc)])
    s = ops.SparseIndexSet(1, h, nc, c, k, n, idx.view(1, h, nc, k).to(torch.int32), cnt)
    ctx = ops.context()
    outs = []
    for lpt in (1, 0):
        ctx.lib.csd_ctx_set_lpt(ctx.h, lpt)
        outs.append(ops.sparse_delta_attention(q, kk, v, s, base, 1.0, layout=1))
    ctx.lib.csd_ctx_set_lpt(ctx.h, 1)
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[0][:, :c, 0], base[:, :c, 0])
    # against the CHECK path (float32, bit-exact with the reference) on the same inputs
    f = lambda t: t.float().permute(0, 2, 1, 3).contiguous()  # noqa: E731  BNHE -> BHNE
    sc = ops.SparseIndexSet(1, h, nc, c, k, n, s.indices, s.counts)
    ref = ops.sparse_delta_attention(f(q), f(kk), f(v), sc, f(base), 1.0)
    got = f(outs[0])
    rel = float((got - ref).norm() / (ref - f(base)).norm())
    assert rel < 2e-2, rel
