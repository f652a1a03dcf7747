"""GPU parity tests (B200): the CUDA path, called through the C ABI, against the oracle.

CHECK mode (float32) must be BIT-EXACT with the reference (golden fixtures produced by
the compiled reference, and the plain-C oracle on seeded inputs).  PROD mode (bf16,
tcgen05) must match the oracle within relative L2 <= 2e-2 (north_star tolerance) on the
same bf16-rounded inputs; its index sets must be exact wherever the selection inputs are
identical (top-k, voxel).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL_L2_TOL = 2e-2  # north_star: block outputs within relative L2 <= 2e-2 in bf16 mode


def T(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dtype).contiguous()


def N(t):
    return t.detach().float().cpu().numpy()


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf(a):
    """bf16-round a float32 array (what the PROD kernels actually see)."""
    return N(T(a, torch.bfloat16))


@pytest.fixture(scope="module")
def ops(cuda):
    from paper_2506_03275_b200 import ops as _ops
    return _ops


def index_set(ops, idx, cnt, chunk, domain):
    b, h, c, k = idx.shape
    return ops.SparseIndexSet(b, h, c, chunk, k, domain, T(idx, torch.int32), T(cnt, torch.int32))


# ------------------------------------------------------------------ voxel
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_voxel_bit_exact(ops, port, golden, dtype):
    g = golden("voxel")
    for i in range(6):
        grid, vox = tuple(g[f"grid{i}"]), tuple(g[f"voxel{i}"])
        lay = ops.VoxelLayout(*grid, *vox)
        assert np.array_equal(ops.voxel_permutation(lay).numpy(), g[f"perm{i}"])
        x = port.gaussian(100 + i, (2, *grid, 24))
        xt = T(x, dtype)
        y, perm = ops.voxel_order(xt, lay)
        want = port.voxel_order(N(xt), vox)
        assert np.array_equal(N(y), want)
        assert torch.equal(ops.reverse_voxel_order(y, lay), xt)
    # FLUX grid, bf16 D = 3072 rows (16-byte vector path)
    lay = ops.VoxelLayout(1, 48, 96, 1, 6, 32)
    x = torch.randn(1, 1, 48, 96, 3072, device="cuda").to(torch.bfloat16)
    y, perm = ops.voxel_order(x, lay)
    assert torch.equal(y[0], x.reshape(1, 4608, 3072)[0, perm.cuda()])
    assert torch.equal(ops.reverse_voxel_order(y, lay), x)


# ------------------------------------------------------------------ top-k
def test_topk_golden_bit_exact(ops, golden):
    g = golden("topk")
    for i in range(4):
        s = g[f"s{i}"]
        k = g[f"i{i}"].shape[-1]
        s4 = s.reshape((1, 1, -1, s.shape[-1]))
        got = ops.select_top_k(T(s4), k, 1)
        assert np.array_equal(N(got.indices).astype(np.int32).reshape(g[f"i{i}"].shape), g[f"i{i}"])
        assert (N(got.counts) == k).all()


@pytest.mark.parametrize("rows,m,k", [(576, 4608, 323), (24, 12288, 860), (3, 118272, 5914),
                                      (2, 40000, 16384), (1, 3000, 2999)])
def test_topk_random_bit_exact(ops, port, rows, m, k):
    rng = np.random.default_rng(rows + m + k)
    s = rng.standard_normal((rows, m)).astype(np.float32)
    s[:, ::7] = np.round(s[:, ::7])  # inject ties
    if rows > 1:
        s[1, :] = 0.0
        s[1, 1::3] = -0.0
    got = ops.select_top_k(T(s.reshape(1, 1, rows, m)), k, 1)
    want = port.select_top_k(s, k)
    assert np.array_equal(N(got.indices).astype(np.int32).reshape(rows, k), want)


def test_topk_large_k_global_path(ops, port):
    s = np.random.default_rng(5).standard_normal((2, 20000)).astype(np.float32)
    got = ops.select_top_k(T(s.reshape(1, 1, 2, 20000)), 17000, 1)
    assert np.array_equal(N(got.indices).astype(np.int32).reshape(2, 17000), port.select_top_k(s, 17000))


@pytest.mark.parametrize("rows,m,k,ties", [(24, 12288, 860, False), (24, 12288, 860, True),
                                           (8, 4096, 300, True), (3, 20000, 5000, False)])
def test_topk_unsorted_set_exact(ops, port, rows, m, k, ties):
    """PROD selection order (csd_ctx_set_sorted_topk(0)): the same exact index set as the
    reference, strictly-greater entries then the lowest-index ties, each in index order
    (cluster-of-CTAs path for few long rows)."""
    rng = np.random.default_rng(rows * m + k)
    s = rng.random((1, 1, rows, m), dtype=np.float32) * 3 + 1
    if ties:
        s = np.round(s * 8) / 8  # many equal scores: the tie rule decides membership
    want = port.select_top_k(s, k).reshape(rows, k)
    ctx = ops.context()
    ctx.set_sorted_topk(False)
    try:
        got = N(ops.select_top_k(T(s), k, 1).indices).astype(np.int64).reshape(rows, k)
    finally:
        ctx.set_sorted_topk(True)
    flat = s.reshape(rows, m)
    for r in range(rows):
        assert set(got[r].tolist()) == set(want[r].tolist()), r
        thr = flat[r, want[r][-1]]
        gt = [i for i in got[r] if flat[r, i] > thr]
        assert gt == sorted(gt) and list(got[r][:len(gt)]) == gt  # greater first, index order
        assert list(got[r][len(gt):]) == sorted(got[r][len(gt):].tolist())


def test_topk_value_error(ops):
    from paper_2506_03275_b200 import errors
    with pytest.raises(errors.ValueError):
        ops.select_top_k(T(np.zeros((1, 1, 1, 4), np.float32)), 5, 4)


# ------------------------------------------------------------------ CHECK-mode attention
def test_check_attention_golden_bit_exact(ops, golden):
    g = golden("attention")
    q, k, v = T(g["q"]), T(g["k"]), T(g["v"])
    r = ops.column_sum_attention(q, k, v, None, 4)
    assert np.array_equal(N(r.output), g["cs_out"])
    assert np.array_equal(N(r.column_sums), g["cs_cs"])
    assert np.array_equal(N(r.stats.row_max), g["cs_m"])
    assert np.array_equal(N(r.stats.exp_sum), g["cs_l"])
    st = ops.SoftmaxStats(T(g["prev_m"]), T(g["prev_l"]))
    r2 = ops.column_sum_attention(q, k, v, st, 4)
    assert np.array_equal(N(r2.column_sums), g["st_cs"])
    assert np.array_equal(N(ops.dense_attention(q, k, v)), g["dense_out"])
    idx = index_set(ops, g["sp_idx"], g["sp_cnt"], 4, 16)
    for sc, key in ((1.0, "sp_plus"), (-1.0, "sp_minus")):
        assert np.array_equal(N(ops.sparse_delta_attention(q, k, v, idx, T(g["sp_base"]), sc)), g[key])


def test_check_attention_flux_slice_bit_exact(ops, port, golden):
    g = golden("attention")
    q, k, v = (T(port.gaussian(int(s), (1, 1, 768, 128))) for s in g["f_seeds"])
    r = ops.column_sum_attention(q, k, v, None, 192)
    assert np.array_equal(N(r.output), g["f_out"])
    assert np.array_equal(N(r.column_sums), g["f_cs"])
    idx = ops.select_top_k(r.column_sums, 54, 192)
    assert np.array_equal(N(idx.indices).astype(np.int32), g["f_idx"])
    resid = ops.sparse_delta_attention(q, k, v, idx, r.output, -1.0)
    assert np.array_equal(N(resid), g["f_resid"])


def test_check_sparse_delta_random_oracle(ops, port):
    # test_attention.cpp:353-433 restated: random shapes / counts / signs, bit-exact
    rng = np.random.default_rng(555)
    for trial in range(12):
        chunk = int(rng.choice([2, 4]))
        n = chunk * int(rng.integers(2, 8))
        e = int(rng.integers(2, 8))
        b, h = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        k_max = int(rng.integers(1, n + 1))
        scale = 1.0 if rng.integers(2) else -1.0
        q, k, v, base = (port.gaussian(7000 + 4 * trial + i, (b, h, n, e)) for i in range(4))
        idx = np.zeros((b, h, n // chunk, k_max), np.int32)
        cnt = np.zeros((b, h, n // chunk), np.int32)
        for bb in range(b):
            for hh in range(h):
                for c in range(n // chunk):
                    m = int(rng.integers(0, k_max + 1))
                    idx[bb, hh, c, :m] = rng.permutation(n)[:m]
                    cnt[bb, hh, c] = m
        want = port.sparse_delta_attention(q, k, v, idx, cnt, chunk, base, scale)
        got = ops.sparse_delta_attention(T(q), T(k), T(v), index_set(ops, idx, cnt, chunk, n), T(base), scale)
        assert np.array_equal(N(got), want), trial


def test_check_attention_errors(ops, port):
    from paper_2506_03275_b200 import errors
    q = T(port.gaussian(1, (1, 1, 8, 4)))
    bad = np.zeros((1, 1, 2, 2), np.int32)
    cnt = np.array([[[2, 0]]], np.int32)
    bad[0, 0, 0] = [3, 3]
    with pytest.raises(errors.IndexError):
        ops.sparse_delta_attention(q, q, q, index_set(ops, bad, cnt, 4, 8), q, 1.0)
    bad[0, 0, 0] = [8, 1]
    with pytest.raises(errors.IndexError):
        ops.sparse_delta_attention(q, q, q, index_set(ops, bad, cnt, 4, 8), q, 1.0)
    with pytest.raises(errors.ShapeError):
        ops.column_sum_attention(q, q, q, None, 3)
    cache = ops.AttentionCache()
    with pytest.raises(errors.StateError):
        ops.attention_step(q, q, q, cache, False, 2, 4)
    # non-finite logits: softmax_rows raises NumericError (tensor.cpp:122-125)
    qn = q.clone()
    qn[0, 0, 3, 1] = float("inf")
    with pytest.raises(errors.NumericError):
        ops.dense_attention(qn, q, q)
    qn[0, 0, 3, 1] = float("nan")
    with pytest.raises(errors.NumericError):
        ops.column_sum_attention(qn, q, q, None, 4)
    # the context is usable again afterwards
    assert torch.isfinite(ops.dense_attention(q, q, q)).all()


def test_block_sparse_before_dense_is_state_error(ops, golden):
    """model_forward_step: a sparse step before any dense step throws StateError
    (attention.cpp:196-219) in both modes; the block stays usable."""
    from paper_2506_03275_b200 import errors
    g = golden("block")
    blk = _golden_block(ops, g, production=False)
    with pytest.raises(errors.StateError):
        blk.step(T(g["x0"]), False)
    y = blk.step(T(g["x0"]), True)
    assert np.array_equal(N(y), g["y0"])


# ------------------------------------------------------------------ CHECK-mode MLP
def test_check_mlp_golden_bit_exact(ops, golden):
    g = golden("mlp")
    w = ops.MlpWeights(T(g["w1"]), T(g["b1"]), T(g["w2"]), T(g["b2"]))
    cache = ops.MlpCache()
    out = ops.mlp_step(T(g["x1"]), w, cache, True, 7, 4)
    assert np.array_equal(N(out), g["d_out"])
    assert np.array_equal(N(cache.activations), g["d_act"])
    assert np.array_equal(N(cache.tile_means), g["tm"])
    o2 = ops.mlp_step(T(g["x2"]), w, cache, False, 7, 4)
    assert np.array_equal(N(cache.indices.indices).astype(np.int32), g["ci2"])
    assert np.array_equal(N(o2), g["o2"])
    assert np.array_equal(N(cache.activations), g["a2"])
    o3 = ops.mlp_step(T(g["x3"]), w, cache, False, 7, 4)
    assert np.array_equal(N(cache.indices.indices).astype(np.int32), g["ci3"])
    assert np.array_equal(N(o3), g["o3"])
    assert np.array_equal(N(cache.activations_ref()), g["a3"])


# ------------------------------------------------------------------ CHECK-mode block
def _golden_block(ops, g, production):
    misc = g["cfg_misc"]
    grid = g["cfg_grid"]
    n = int(np.prod(grid))
    cfg = ops.BlockConfig(batch=int(misc[0]), seq=n, dim=int(misc[1]), heads=int(misc[3]),
                          head_dim=int(misc[2]), hidden=int(misc[4]), chunk=int(misc[5]),
                          attn_k=int(g["ks"][0]), mlp_k=int(g["ks"][1]))
    w = {k[2:]: g[k] for k in g if k.startswith("w_")}
    return ops.Block(cfg, w, production=production)


def test_check_block_trajectory_bit_exact(ops, golden):
    g = golden("block")
    blk = _golden_block(ops, g, production=False)
    for t, dense in enumerate(g["sched"]):
        y = blk.step(T(g[f"x{t}"]), bool(dense))
        assert np.array_equal(N(y), g[f"y{t}"]), t
        ai, _ = blk.indices(False)
        assert np.array_equal(N(ai).astype(np.int32), g[f"aidx{t}"]), t
        if not dense:
            mi, _ = blk.indices(True)
            assert np.array_equal(N(mi).astype(np.int32), g[f"midx{t}"]), t


# ------------------------------------------------------------------ PROD-mode attention (tcgen05)
# h x (n / chunk) > 148 cases run several work items per persistent CTA
@pytest.mark.parametrize("e,chunk,n,layout,h", [(128, 192, 768, 0, 3), (64, 64, 512, 0, 3),
                                                (128, 128, 640, 1, 3), (64, 192, 384, 1, 3),
                                                (128, 256, 512, 0, 3), (128, 192, 4608, 1, 8),
                                                (64, 64, 2048, 0, 7)])
def test_prod_sparse_delta_attention(ops, port, e, chunk, n, layout, h):
    rng = np.random.default_rng(e * 7 + chunk + n)
    b = 1
    shape = (b, h, n, e) if layout == 0 else (b, n, h, e)
    q, k, v, base = (port.gaussian(300 + i, shape) for i in range(4))
    q16, k16, v16, b16 = (bf(a) for a in (q, k, v, base))
    nc = n // chunk
    k_max = max(1, n // 7)
    idx = np.zeros((b, h, nc, k_max), np.int32)
    cnt = np.zeros((b, h, nc), np.int32)
    for hh in range(h):
        for c in range(nc):
            m = k_max if c % 3 else int(rng.integers(0, k_max + 1))
            idx[0, hh, c, :m] = rng.permutation(n)[:m]
            cnt[0, hh, c] = m
    to_bhne = (lambda a: a) if layout == 0 else (lambda a: np.ascontiguousarray(a.transpose(0, 2, 1, 3)))
    # chunk 192 / 256 with E 128 also runs through the opt-in CTA-pair kernel (attn_cp.cu, mode
    # 1) and chunk 192 through the P-in-shared-memory kernel (attn_px.cu, mode 2)
    modes = (0,)
    if e == 128 and chunk in (192, 256):
        modes = (0, 1, 2) if chunk == 192 else (0, 1)
    from paper_2506_03275_b200 import _capi
    set_cp = _capi.lib().csd_debug_set_attn_cp
    set_px = _capi.lib().csd_debug_set_attn_px
    for scale, mode in [(sc, md) for sc in (1.0, -1.0) for md in modes]:
        want = port.sparse_delta_attention(to_bhne(q16), to_bhne(k16), to_bhne(v16), idx, cnt, chunk,
                                           to_bhne(b16), scale)
        set_cp(int(mode == 1))
        set_px(int(mode == 2))
        # the px kernel runs only in identity item order (no LPT)
        ctx = ops.context()
        ctx.lib.csd_ctx_set_lpt(ctx.h, int(mode != 2))
        try:
            got = ops.sparse_delta_attention(T(q16, torch.bfloat16), T(k16, torch.bfloat16),
                                             T(v16, torch.bfloat16), index_set(ops, idx, cnt, chunk, n),
                                             T(b16, torch.bfloat16), scale, layout=layout)
        finally:
            set_cp(0)
            set_px(0)
            ctx.lib.csd_ctx_set_lpt(ctx.h, 1)
        got = to_bhne(N(got))
        # delta part only (base cancels) must match to bf16 accuracy
        err = rel_l2(got - to_bhne(b16), want - to_bhne(b16))
        assert err < REL_L2_TOL, err
        # count-0 chunks pass base through exactly
        for hh in range(h):
            for c in range(nc):
                if cnt[0, hh, c] == 0:
                    assert np.array_equal(got[0, hh, c * chunk:(c + 1) * chunk], to_bhne(b16)[0, hh, c * chunk:(c + 1) * chunk])


# (192, 768) / (192, 1536) / (128, 1024): 256-row work items with per-chunk column sums merged
# across items (capi_ops.cpp); the others run one chunk per item
@pytest.mark.parametrize("e,chunk,n,h", [(128, 192, 768, 2), (64, 64, 512, 2), (128, 128, 384, 2),
                                         (64, 64, 1024, 10), (128, 192, 1536, 2),
                                         (128, 128, 1024, 3)])
def test_prod_dense_and_colsum_attention(ops, port, e, chunk, n, h):
    q, k, v = (bf(port.gaussian(400 + i, (1, h, n, e))) for i in range(3))
    want_o, want_cs, (wm, wl) = port.column_sum_attention(q, k, v, None, chunk)
    qt, kt, vt = (T(a, torch.bfloat16) for a in (q, k, v))
    o = ops.dense_attention(qt, kt, vt)
    assert rel_l2(N(o), want_o) < REL_L2_TOL
    r = ops.column_sum_attention(qt, kt, vt, None, chunk)
    assert rel_l2(N(r.output), want_o) < REL_L2_TOL
    assert rel_l2(N(r.stats.row_max), wm) < 1e-2
    assert rel_l2(N(r.stats.exp_sum), wl) < 2e-2
    assert rel_l2(N(r.column_sums), want_cs) < 3e-2
    # stale-stat column sums
    pm = (wm + 0.05 * port.gaussian(77, wm.shape)).astype(np.float32)
    pl = (wl * (1 + 0.05 * port.gaussian(78, wl.shape))).astype(np.float32)
    _, want_cs2, _ = port.column_sum_attention(q, k, v, (pm, pl), chunk)
    r2 = ops.column_sum_attention(qt, kt, vt, ops.SoftmaxStats(T(pm), T(pl)), chunk)
    assert rel_l2(N(r2.column_sums), want_cs2) < 3e-2
    # the selected sets agree with the fp32 selection up to near-ties
    kk = n // 10
    got_i = N(ops.select_top_k(r.column_sums, kk, chunk).indices)
    want_i = port.select_top_k(want_cs, kk)
    overlap = np.mean([len(set(a) & set(b)) / kk for a, b in zip(got_i.reshape(-1, kk), want_i.reshape(-1, kk))])
    assert overlap > 0.9, overlap


# ------------------------------------------------------------------ PROD-mode MLP
def test_prod_mlp_steps(ops, port):
    b, n, d, f, c, kk = 1, 384, 256, 1024, 64, 96
    x1 = bf(port.gaussian(500, (b, n, d)))
    w1 = bf(port.gaussian(501, (f, d), 1 / 16))
    w2 = bf(port.gaussian(502, (f, d), 1 / 32))
    b1, b2 = port.gaussian(503, (f,), 1 / 16), port.gaussian(504, (d,), 1 / 32)
    w = ops.MlpWeights(T(w1, torch.bfloat16), T(b1), T(w2, torch.bfloat16), T(b2))
    cache = ops.MlpCache()
    out = ops.mlp_step(T(x1, torch.bfloat16), w, cache, True, kk, c)
    want_out, _, want_act = port.dense_mlp(x1, w1, b1, w2, b2)
    assert rel_l2(N(out), want_out) < REL_L2_TOL
    want_tm = port.mlp_tile_means(x1, w1, c)
    assert rel_l2(N(cache.tile_means), want_tm) < 1e-3
    acts, outs, xs = want_act, want_out, x1
    for step in range(2):
        xs = bf(xs + 0.1 * port.gaussian(510 + step, xs.shape))
        got = ops.mlp_step(T(xs, torch.bfloat16), w, cache, False, kk, c)
        gi = N(cache.indices.indices).astype(np.int32)
        cnt = np.full(gi.shape[:-1], kk, np.int32)
        # oracle on the SAME index set (selection inputs differ by bf16 activations)
        outs, acts = port.sparse_delta_mlp(xs, w1, b1, w2, b2, gi, cnt, c, acts, outs)
        assert rel_l2(N(got) - want_out, outs - want_out) < 1e-1  # bf16 act-cache deltas
        assert rel_l2(N(got), outs) < REL_L2_TOL


# ------------------------------------------------------------------ PROD-mode block
def test_prod_block_trajectory_matches_oracle(ops, golden):
    g = golden("block")
    # desk config has head_dim 16 (outside the tcgen05 envelope) -> use a cfg1-shaped block
    from paper_2506_03275_b200 import errors
    blk16 = _golden_block(ops, g, production=True)
    with pytest.raises(errors.UnsupportedError):
        blk16.step(T(g["x0"], torch.bfloat16), True)


def test_prod_block_cfg1_vs_check_mode(ops, port):
    # cfg1-like: N 1024 (grid 1x32x32, voxel 1x8x8), D 768, H 12x64, F 3072, c 64, 90%
    n, d, h, e, f, c = 1024, 768, 12, 64, 3072, 64
    ak, mk = 102, 307
    std = 1 / np.sqrt(d)
    w = {"wq": port.gaussian(1, (d, d), std), "wk": port.gaussian(2, (d, d), std),
         "wv": port.gaussian(3, (d, d), std), "wo": port.gaussian(4, (d, d), std / 2),
         "w1": port.gaussian(5, (f, d), std), "b1": port.gaussian(6, (f,), std),
         "w2": port.gaussian(7, (f, d), std / 2), "b2": port.gaussian(8, (d,), std / 2)}
    w = {k: bf(v) if k not in ("b1", "b2") else v for k, v in w.items()}
    cfg = ops.BlockConfig(batch=1, seq=n, dim=d, heads=h, head_dim=e, hidden=f, chunk=c,
                          attn_k=ak, mlp_k=mk)
    prod = ops.Block(cfg, w, production=True)
    chk = ops.Block(cfg, w, production=False)
    x0 = port.gaussian(1235, (1, n, d))
    for t, dense in enumerate([1, 0, 0, 0]):
        x = bf(x0 + 0.02 * t * port.gaussian(3000 + t, x0.shape))
        yp = prod.step(T(x, torch.bfloat16), bool(dense))
        yc = chk.step(T(x), bool(dense))
        err = rel_l2(N(yp) - x, N(yc) - x)  # branch outputs (x cancels)
        assert err < REL_L2_TOL, (t, err)


def test_prod_mlp_change_indices_fused_unsorted_same_set(ops, port):
    """The PROD block's fused selection (split-K tile-means reduction inside the cluster
    top-k, unsorted) yields the same index sets as the sorted public path."""
    b, n, d, f, c, kk = 1, 1536, 512, 4096, 64, 300
    x = bf(port.gaussian(700, (b, n, d)))
    w1 = bf(port.gaussian(701, (f, d), 1 / 16))
    tm = T(port.gaussian(702, (b, n // c, f), 0.1))
    xt, wt = T(x, torch.bfloat16), T(w1, torch.bfloat16)
    want = N(ops.mlp_change_indices(xt, wt, tm, kk, c).indices).astype(np.int64)
    ctx = ops.context()
    ctx.set_sorted_topk(False)
    try:
        got = N(ops.mlp_change_indices(xt, wt, tm, kk, c).indices).astype(np.int64)
    finally:
        ctx.set_sorted_topk(True)
    got, want = got.reshape(-1, kk), want.reshape(-1, kk)
    for r in range(got.shape[0]):
        assert set(got[r].tolist()) == set(want[r].tolist()), r


def test_prod_block_batch2_vs_check_mode(ops, port):
    """Batch 2 through the PROD block step (every kernel's batch indexing) against CHECK mode
    on the same bf16-rounded inputs: dense then sparse steps, branch outputs within 2e-2."""
    b, n, d, h, e, f, c = 2, 512, 256, 2, 128, 1024, 64
    ak, mk = 52, 103
    std = 1 / np.sqrt(d)
    w = {"wq": port.gaussian(11, (d, d), std), "wk": port.gaussian(12, (d, d), std),
         "wv": port.gaussian(13, (d, d), std), "wo": port.gaussian(14, (d, d), std / 2),
         "w1": port.gaussian(15, (f, d), std), "b1": port.gaussian(16, (f,), std),
         "w2": port.gaussian(17, (f, d), std / 2), "b2": port.gaussian(18, (d,), std / 2)}
    w = {k: bf(v) if k not in ("b1", "b2") else v for k, v in w.items()}
    cfg = ops.BlockConfig(batch=b, seq=n, dim=d, heads=h, head_dim=e, hidden=f, chunk=c,
                          attn_k=ak, mlp_k=mk)
    prod = ops.Block(cfg, w, production=True)
    chk = ops.Block(cfg, w, production=False)
    x0 = port.gaussian(2235, (b, n, d))
    for t, dense in enumerate([1, 0, 0]):
        x = bf(x0 + 0.02 * t * port.gaussian(4000 + t, x0.shape))
        yp = prod.step(T(x, torch.bfloat16), bool(dense))
        yc = chk.step(T(x), bool(dense))
        for bb in range(b):
            err = rel_l2(N(yp)[bb] - x[bb], N(yc)[bb] - x[bb])
            assert err < REL_L2_TOL, (t, bb, err)


def test_check_block_static_pattern_bit_exact(ops, golden):
    """Static attention pattern (model.hpp:97-99, attention.hpp:50-52): applied verbatim on
    dense steps, ragged counts including 0 (test_attention.cpp:441-459); the reference's
    model_forward_step outputs reproduced bit-for-bit over D S S D S."""
    g = golden("block_static")
    gb = golden("block")
    misc, grid = gb["cfg_misc"], gb["cfg_grid"]
    n = int(np.prod(grid))
    cfg = ops.BlockConfig(batch=int(misc[0]), seq=n, dim=int(misc[1]), heads=int(misc[3]),
                          head_dim=int(misc[2]), hidden=int(misc[4]), chunk=int(misc[5]),
                          attn_k=int(g["idx"].shape[-1]), mlp_k=int(gb["ks"][1]))
    blk = ops.Block(cfg, {k[2:]: g[k] for k in g if k.startswith("w_")}, production=False)
    idx, cnt = g["idx"], g["counts"]
    st = index_set(ops, idx, cnt, cfg.chunk, n)
    for t, dense in enumerate(g["sched"]):
        y = blk.step(T(g[f"x{t}"]), bool(dense), static=st if dense else None)
        assert np.array_equal(N(y), g[f"y{t}"]), t
        ai, ac = blk.indices(False)
        assert np.array_equal(N(ac), cnt), t
        for ii in np.ndindex(*cnt.shape):
            assert np.array_equal(N(ai)[ii][:cnt[ii]], idx[ii][:cnt[ii]]), (t, ii)


def test_prod_block_static_pattern_vs_check(ops, port):
    """The same static-pattern semantics in PROD (cfg1-like shapes, ragged counts with empty
    chunks), against CHECK mode on identical bf16-rounded inputs."""
    n, d, h, e, f, c = 1024, 768, 12, 64, 3072, 64
    ak, mk = 102, 307
    std = 1 / np.sqrt(d)
    w = {"wq": port.gaussian(21, (d, d), std), "wk": port.gaussian(22, (d, d), std),
         "wv": port.gaussian(23, (d, d), std), "wo": port.gaussian(24, (d, d), std / 2),
         "w1": port.gaussian(25, (f, d), std), "b1": port.gaussian(26, (f,), std),
         "w2": port.gaussian(27, (f, d), std / 2), "b2": port.gaussian(28, (d,), std / 2)}
    w = {k: bf(v) if k not in ("b1", "b2") else v for k, v in w.items()}
    cfg = ops.BlockConfig(batch=1, seq=n, dim=d, heads=h, head_dim=e, hidden=f, chunk=c,
                          attn_k=ak, mlp_k=mk)
    rng = np.random.default_rng(459)
    nc = n // c
    idx = np.zeros((1, h, nc, ak), np.int32)
    cnt = rng.integers(0, ak + 1, size=(1, h, nc)).astype(np.int32)
    cnt[0, 0, :3] = 0  # empty chunks pass the cached residual through
    for ii in np.ndindex(1, h, nc):
        idx[ii][:cnt[ii]] = rng.permutation(n)[:cnt[ii]]
    st = index_set(ops, idx, cnt, c, n)
    prod = ops.Block(cfg, w, production=True)
    chk = ops.Block(cfg, w, production=False)
    x0 = port.gaussian(2300, (1, n, d))
    for t, dense in enumerate([1, 0, 0, 1, 0]):
        x = bf(x0 + 0.02 * t * port.gaussian(4100 + t, x0.shape))
        yp = prod.step(T(x, torch.bfloat16), bool(dense), static=st if dense else None)
        yc = chk.step(T(x), bool(dense), static=st if dense else None)
        err = rel_l2(N(yp) - x, N(yc) - x)
        assert err < REL_L2_TOL, (t, err)
        _, pc = prod.indices(False)
        assert np.array_equal(N(pc), cnt), t
