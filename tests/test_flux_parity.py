"""Parity at the benchmarked configuration (BASELINE.json configs[1], the FLUX.1-dev-shaped
block bench.py times): N 4608 (grid 1x48x96), D 3072, 24 x 128 heads, F 12288, chunk 192,
93 % sparsity (attn_k 323, mlp_k 860).

* The PROD block (bf16, tcgen05: k_attn_tc<128,2>, k_smlp_up<2> / k_smlp_down<2>, the
  fused selection chain) is run over D,S,S,D,S against the CHECK block -- the fp32 path
  that reproduces the reference's model_forward_step bit for bit
  (test_gpu_parity.py::test_check_block_trajectory_bit_exact, model.cpp:178-216) -- on
  the same bf16-rounded weights and latents.  Branch outputs (y - x) must agree within
  relative L2 2e-2 (north_star) on every step; the index sets each mode selects must
  overlap >= 0.95, and any row below that must be a near-tie in the CHECK scores.
* The chunk > 128 sparse-delta MLP kernels (k_smlp_up<2> / k_smlp_down<2>) are compared
  directly with the plain-C oracle (oracle/csd_oracle.c, mlp.cpp:120-182) on the same
  index set at chunk 192 and 256, with ragged counts including empty chunks.
"""
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL_L2_TOL = 2e-2
OVERLAP_MIN = 0.95

FLUX = dict(n=4608, d=3072, h=24, e=128, f=12288, c=192, ak=323, mk=860)


def T(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dtype).contiguous()


def N(t):
    return t.detach().float().cpu().numpy()


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf(a):
    return N(T(a, torch.bfloat16))


@pytest.fixture(scope="module")
def ops(cuda):
    from paper_2506_03275_b200 import ops as _ops
    return _ops


def _weights(d, f, seed):
    """model.cpp:79-99 distributions (wo / w2 / b2 at half scale), bf16-rounded so both
    modes see identical weights."""
    rng = np.random.default_rng(seed)
    std = 1.0 / np.sqrt(d)

    def g(shape, s):
        return rng.standard_normal(shape, dtype=np.float32) * np.float32(s)
    w = {"wq": g((d, d), std), "wk": g((d, d), std), "wv": g((d, d), std),
         "wo": g((d, d), std / 2), "w1": g((f, d), std), "b1": g((f,), std),
         "w2": g((f, d), std / 2), "b2": g((d,), std / 2)}
    return {k: (v if k in ("b1", "b2") else bf(v)) for k, v in w.items()}


def _overlap(a, b, ca, cb):
    """Mean / min per-row overlap |A & B| / max(|A|, 1) of two index sets."""
    a = a.reshape(-1, a.shape[-1])
    b = b.reshape(-1, b.shape[-1])
    ca, cb = ca.reshape(-1), cb.reshape(-1)
    ov = []
    for r in range(a.shape[0]):
        sa, sb = set(a[r, :ca[r]].tolist()), set(b[r, :cb[r]].tolist())
        ov.append(len(sa & sb) / max(len(sa), 1))
    ov = np.asarray(ov)
    return float(ov.mean()), float(ov.min()), ov


def test_flux_block_prod_vs_check(ops):
    """PROD vs the bit-exact CHECK block at the exact bench config, D S S D S."""
    p = FLUX
    n, d = p["n"], p["d"]
    w = _weights(d, p["f"], 1234)
    cfg = ops.BlockConfig(batch=1, seq=n, dim=d, heads=p["h"], head_dim=p["e"], hidden=p["f"],
                          chunk=p["c"], attn_k=p["ak"], mlp_k=p["mk"])
    prod = ops.Block(cfg, w, production=True)
    chk = ops.Block(cfg, w, production=False)
    rng = np.random.default_rng(1235)
    x0 = rng.standard_normal((1, n, d), dtype=np.float32)
    report = []
    for t, dense in enumerate([1, 0, 0, 1, 0]):
        x = bf(x0 + np.float32(0.05 * t) * rng.standard_normal(x0.shape, dtype=np.float32))
        yp = N(prod.step(T(x, torch.bfloat16), bool(dense)))
        yc = N(chk.step(T(x), bool(dense)))
        err = rel_l2(yp - x, yc - x)  # branch outputs (x cancels)
        pa, pc = (N(v).astype(np.int64) for v in prod.indices(False))
        ca, cc = (N(v).astype(np.int64) for v in chk.indices(False))
        a_mean, a_min, _ = _overlap(pa, ca, pc, cc)
        row = {"step": t, "dense": dense, "rel_l2": err, "attn_overlap": a_mean,
               "attn_min": a_min}
        if not dense:
            pm, pmc = (N(v).astype(np.int64) for v in prod.indices(True))
            cm, cmc = (N(v).astype(np.int64) for v in chk.indices(True))
            m_mean, m_min, _ = _overlap(pm, cm, pmc, cmc)
            row.update(mlp_overlap=m_mean, mlp_min=m_min)
        report.append(row)
        print(row)
        assert np.isfinite(yp).all(), t
        assert err < REL_L2_TOL, row
        assert a_mean >= OVERLAP_MIN, row
        if not dense:
            assert row["mlp_overlap"] >= OVERLAP_MIN, row
    prod.close()
    chk.close()
    out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, "flux_parity.json"), "w") as f:
            json.dump(report, f, indent=1)


def test_flux_attention_selection_misses_are_near_ties(ops):
    """The dense-step selection at FLUX on IDENTICAL q/k/v (bf16-rounded, fed to both modes):
    PROD's fused stale-stat column sums (tcgen05, attn_tc.cu) and the CHECK column sums
    (attention.cpp:76-145 bit for bit) pick top-323 sets that overlap >= 0.95, and every key
    PROD picks that CHECK does not sits within 2 % of CHECK's k-th score (a near-tie)."""
    p = FLUX
    n, h, e, c, k = p["n"], p["h"], p["e"], p["c"], p["ak"]
    g = torch.Generator(device="cuda").manual_seed(77)
    q, kk, v = (torch.randn((1, n, h, e), device="cuda", generator=g).to(torch.bfloat16)
                for _ in range(3))
    # BHNE fp32 copies of the same bf16 values for CHECK
    qf, kf, vf = (t.float().permute(0, 2, 1, 3).contiguous() for t in (q, kk, v))
    # stale stats: the previous dense step's, from slightly different q/k
    q0 = (q.float() + 0.1 * torch.randn(q.shape, device="cuda", generator=g)).to(torch.bfloat16)
    r0 = ops.column_sum_attention(q0.float().permute(0, 2, 1, 3).contiguous(), kf, vf, None, c)
    stats = ops.SoftmaxStats(r0.stats.row_max, r0.stats.exp_sum)
    rp = ops.column_sum_attention(q, kk, v, stats, c, layout=1)
    rc = ops.column_sum_attention(qf, kf, vf, stats, c)
    assert rel_l2(N(rp.output).transpose(0, 2, 1, 3), N(rc.output)) < REL_L2_TOL
    assert rel_l2(N(rp.column_sums), N(rc.column_sums)) < 2e-2
    ip = N(ops.select_top_k(rp.column_sums, k, c).indices).astype(np.int64).reshape(-1, k)
    ic = N(ops.select_top_k(rc.column_sums, k, c).indices).astype(np.int64).reshape(-1, k)
    cs = N(rc.column_sums).reshape(-1, n)
    ov = []
    for r in range(ip.shape[0]):
        extra = set(ip[r].tolist()) - set(ic[r].tolist())
        ov.append(1 - len(extra) / k)
        if extra:
            kth = cs[r, ic[r, -1]]
            worst = min(cs[r, j] for j in extra)
            assert worst >= kth * (1 - 2e-2), (r, worst, kth)
    assert np.mean(ov) >= OVERLAP_MIN, np.mean(ov)


@pytest.mark.parametrize("chunk,n", [(192, 768), (256, 1024)])
def test_prod_sparse_delta_mlp_wide_chunk_vs_oracle(ops, port, chunk, n):
    """k_smlp_up<2> / k_smlp_down<2> (chunk > 128: two M = 128 tiles) against the plain-C
    oracle (mlp.cpp:120-182) on the SAME ragged index set, empty chunks included."""
    d, f, kmax = 512, 2048, 300
    rng = np.random.default_rng(chunk)
    x0 = bf(rng.standard_normal((1, n, d), dtype=np.float32))
    w1 = bf(rng.standard_normal((f, d), dtype=np.float32) / np.sqrt(d))
    w2 = bf(rng.standard_normal((f, d), dtype=np.float32) / np.sqrt(d) / 2)
    b1 = (rng.standard_normal(f, dtype=np.float32) / np.sqrt(d)).astype(np.float32)
    b2 = (rng.standard_normal(d, dtype=np.float32) / np.sqrt(d) / 2).astype(np.float32)
    w = ops.MlpWeights(T(w1, torch.bfloat16), T(b1), T(w2, torch.bfloat16), T(b2))
    cache = ops.MlpCache()
    ops.mlp_step(T(x0, torch.bfloat16), w, cache, True, kmax, chunk)
    want_out, _, want_act = port.dense_mlp(x0, w1, b1, w2, b2)
    assert rel_l2(N(cache.outputs), want_out) < REL_L2_TOL
    nc = n // chunk
    acts, outs = want_act, want_out
    for step in range(2):
        x = bf(x0 + np.float32(0.2) * rng.standard_normal(x0.shape, dtype=np.float32))
        cnt = rng.integers(1, kmax + 1, size=(1, 1, nc)).astype(np.int32)
        cnt[0, 0, 0] = kmax
        if nc > 2:
            cnt[0, 0, 1] = 0  # empty chunk: caches untouched
        idx = np.zeros((1, 1, nc, kmax), np.int32)
        for z in range(nc):
            idx[0, 0, z, :cnt[0, 0, z]] = rng.permutation(f)[:cnt[0, 0, z]]
        st = ops.SparseIndexSet(1, 1, nc, chunk, kmax, f, T(idx, torch.int32), T(cnt, torch.int32))
        got = N(ops.sparse_delta_mlp(T(x, torch.bfloat16), w, st, cache))
        outs, acts = port.sparse_delta_mlp(x, w1, b1, w2, b2, idx, cnt, chunk, acts, outs)
        assert rel_l2(got, outs) < REL_L2_TOL, (step, rel_l2(got, outs))
        # the delta itself (what the kernels compute this step), bf16 activation cache
        # the step's delta alone: the PROD activation cache is bf16 (mlp_tc.cu), so delta =
        # gelu(new) - A_cache carries the cache's rounding (~2^-9 of |a|) relative to a
        # small |delta|; the block-output contract above is the 2e-2 one
        assert rel_l2(got - want_out, outs - want_out) < 1e-1
        got_act = N(cache.activations_ref())
        assert rel_l2(got_act, acts) < REL_L2_TOL
        if nc > 2:  # empty chunk: outputs and activations of its rows unchanged
            rows = slice(chunk, 2 * chunk)
            assert rel_l2(got[:, rows], want_out[:, rows]) < 1e-2


def test_flux_sparse_delta_mlp_prod_vs_check(ops):
    """The sparse-delta MLP at the FLUX shape (k_smlp_<2>, chunk 192, k 860) against the
    CHECK kernels (mlp.cpp:120-182 bit for bit) on the same index set and bf16 inputs."""
    p = FLUX
    n, d, f, c, k = p["n"], p["d"], p["f"], p["c"], p["mk"]
    w = _weights(d, f, 99)
    rng = np.random.default_rng(5)
    x0 = bf(rng.standard_normal((1, n, d), dtype=np.float32))
    wp = ops.MlpWeights(T(w["w1"], torch.bfloat16), T(w["b1"]), T(w["w2"], torch.bfloat16), T(w["b2"]))
    wc = ops.MlpWeights(T(w["w1"]), T(w["b1"]), T(w["w2"]), T(w["b2"]))
    cp, cc = ops.MlpCache(), ops.MlpCache()
    ops.mlp_step(T(x0, torch.bfloat16), wp, cp, True, k, c)
    ops.mlp_step(T(x0), wc, cc, True, k, c)
    base = N(cc.outputs)
    assert rel_l2(N(cp.outputs), base) < REL_L2_TOL
    nc = n // c
    x = bf(x0 + np.float32(0.1) * rng.standard_normal(x0.shape, dtype=np.float32))
    # the CHECK selection, applied verbatim in both modes
    sel = ops.mlp_change_indices(T(x), wc.w1, cc.tile_means, k, c)
    got = N(ops.sparse_delta_mlp(T(x, torch.bfloat16), wp, sel, cp))
    want = N(ops.sparse_delta_mlp(T(x), wc, sel, cc))
    assert rel_l2(got, want) < REL_L2_TOL
    assert rel_l2(got - base, want - base) < 1e-1  # delta alone: bf16 activation cache
    assert sel.counts.shape == (1, 1, nc)
