"""CPU tests of the oracle itself (no GPU): it must be pinned before it is trusted.

1. glibc-compatible expf / tanhf vs the host libm (sampled; the exhaustive sweeps
   are oracle/check_{expf,tanhf}_exhaustive.c).
2. The reference's own known-answer tests (test_voxel.cpp, test_attention.cpp,
   test_mlp.cpp) restated against the oracle.
3. Golden fixtures produced by the compiled reference (tests/golden, oracle/gen_golden.py):
   bit-exact.
4. Differential vs the compiled reference on random shapes when oracle/_ref exists.
"""
import numpy as np
import pytest


def test_expf_tanhf_match_libm(port):
    # strided sweep over every exponent: ~2.7M patterns each, finite and special values
    for which in (0, 1):
        assert port.libm_mismatches(0, 0xFFFFFFFF, 1601, which) == 0
    # dense sweep of the softmax working range [-40, 0]
    import struct
    lo = struct.unpack("<I", struct.pack("<f", -40.0))[0]
    hi = struct.unpack("<I", struct.pack("<f", -0.0))[0]
    assert port.libm_mismatches(hi, lo, 97, 0) == 0


def test_gaussian_stream_matches_reference(port, ref):
    assert np.array_equal(port.gaussian(7, (1001,), 0.5), ref.gaussian(7, (1001,), 0.5))


# ---------------------------------------------------------------- voxel (test_voxel.cpp)
def test_voxel_spot_value(port):
    # test_voxel.cpp:38-44: grid (2,2,4), voxel (1,2,2) -> perm[4] == 2
    assert port.voxel_permutation((2, 2, 4), (1, 2, 2))[4] == 2


def test_voxel_random_layouts_bijection_roundtrip(port):
    rng = np.random.default_rng(0)
    for _ in range(40):
        vt, vh, vw = rng.integers(1, 4, 3)
        t, h, w = vt * rng.integers(1, 4), vh * rng.integers(1, 4), vw * rng.integers(1, 4)
        perm = port.voxel_permutation((t, h, w), (vt, vh, vw))
        assert sorted(perm.tolist()) == list(range(t * h * w))
        x = port.gaussian(int(rng.integers(1 << 30)), (2, t, h, w, 3))
        y = port.voxel_order(x, (vt, vh, vw))
        assert np.array_equal(port.reverse_voxel_order(y, (t, h, w), (vt, vh, vw)), x)


def test_voxel_rejects_non_tiling(port, O):
    with pytest.raises(O.OracleError) as e:
        port.voxel_permutation((2, 3, 4), (1, 2, 2))
    assert e.value.kind == "ConfigError"


def test_voxel_golden(port, golden):
    g = golden("voxel")
    for i in range(6):
        assert np.array_equal(port.voxel_permutation(tuple(g[f"grid{i}"]), tuple(g[f"voxel{i}"])),
                              g[f"perm{i}"])
    assert np.array_equal(port.voxel_order(g["x"], (2, 3, 4)), g["x_ordered"])


# ---------------------------------------------------------------- top-k
def test_topk_tie_rule(port):
    # test_attention.cpp:105-111: [0.1, 0.9, 0.5, 0.5], k=2 -> [1, 2]
    assert port.select_top_k(np.array([[0.1, 0.9, 0.5, 0.5]], np.float32), 2).tolist() == [[1, 2]]


def test_topk_vs_full_sort(port):
    s = port.gaussian(123, (24, 16))
    got = port.select_top_k(s, 3)
    for r in range(24):
        order = sorted(range(16), key=lambda j: (-s[r, j], j))
        assert got[r].tolist() == order[:3]


def test_topk_golden(port, golden):
    g = golden("topk")
    for i in range(4):
        k = g[f"i{i}"].shape[-1]
        assert np.array_equal(port.select_top_k(g[f"s{i}"], k), g[f"i{i}"])


def test_topk_rejects_bad_k(port, O):
    for k in (0, 5):
        with pytest.raises(O.OracleError):
            port.select_top_k(np.zeros((1, 4), np.float32), k)


# ---------------------------------------------------------------- attention
def test_colsum_uniform_is_ones(port):
    # test_attention.cpp:45-52
    q = np.ones((1, 1, 4, 2), np.float32)
    _, cs, _ = port.column_sum_attention(q, q, port.gaussian(3, (1, 1, 4, 2)), None, 4)
    assert np.allclose(cs, 1.0, atol=1e-6)


def test_colsum_fresh_rows_sum_to_chunk_and_stats_roundtrip(port):
    q, k, v = (port.gaussian(s, (1, 1, 8, 4)) for s in (10, 11, 12))
    o, cs, st = port.column_sum_attention(q, k, v, None, 2)
    assert np.allclose(cs.sum(-1), 2.0, atol=1e-3)
    _, cs2, _ = port.column_sum_attention(q, k, v, st, 2)
    assert np.array_equal(cs, cs2)  # test_attention.cpp:71-73, bit-identical
    assert np.array_equal(o, port.dense_attention(q, k, v))


def test_attention_golden(port, golden):
    g = golden("attention")
    o, cs, (m, l) = port.column_sum_attention(g["q"], g["k"], g["v"], None, 4)
    for a, b in ((o, g["cs_out"]), (cs, g["cs_cs"]), (m, g["cs_m"]), (l, g["cs_l"])):
        assert np.array_equal(a, b)
    o, cs, (m, l) = port.column_sum_attention(g["q"], g["k"], g["v"], (g["prev_m"], g["prev_l"]), 4)
    for a, b in ((o, g["st_out"]), (cs, g["st_cs"]), (m, g["st_m"]), (l, g["st_l"])):
        assert np.array_equal(a, b)
    assert np.array_equal(port.dense_attention(g["q"], g["k"], g["v"]), g["dense_out"])
    for sc, key in ((1.0, "sp_plus"), (-1.0, "sp_minus")):
        got = port.sparse_delta_attention(g["q"], g["k"], g["v"], g["sp_idx"], g["sp_cnt"], 4,
                                          g["sp_base"], sc)
        assert np.array_equal(got, g[key])


def test_attention_golden_flux_slice(port, golden):
    g = golden("attention")
    q, k, v = (port.gaussian(int(s), (1, 1, 768, 128)) for s in g["f_seeds"])
    o, cs, (m, l) = port.column_sum_attention(q, k, v, None, 192)
    assert np.array_equal(o, g["f_out"]) and np.array_equal(cs, g["f_cs"])
    idx = port.select_top_k(cs, 54)
    assert np.array_equal(idx, g["f_idx"])
    cnt = np.full(idx.shape[:-1], 54, np.int32)
    assert np.array_equal(port.sparse_delta_attention(q, k, v, idx, cnt, 192, o, -1.0), g["f_resid"])


def test_sparse_delta_count0_and_duplicate(port, O):
    q, k, v = (port.gaussian(s, (1, 1, 8, 4)) for s in (20, 21, 22))
    base = port.gaussian(23, q.shape)
    idx = np.zeros((1, 1, 2, 3), np.int32)
    cnt = np.zeros((1, 1, 2), np.int32)
    assert np.array_equal(port.sparse_delta_attention(q, k, v, idx, cnt, 4, base, 1.0), base)
    idx[0, 0, 0, :2] = [5, 5]
    cnt[0, 0, 0] = 2
    with pytest.raises(O.OracleError) as e:
        port.sparse_delta_attention(q, k, v, idx, cnt, 4, base, 1.0)
    assert e.value.kind == "IndexError"


# ---------------------------------------------------------------- MLP
def test_change_indices_known_answers(port):
    # test_mlp.cpp:124-144
    w1 = port.gaussian(20, (6, 3))
    x = port.gaussian(21, (1, 4, 3))
    fresh = port.mlp_tile_means(x, w1, 2)
    assert port.mlp_change_indices(x, w1, fresh, 3, 2)[0, 0].tolist() == [[0, 1, 2], [0, 1, 2]]
    x1 = port.gaussian(22, (1, 2, 3))
    cache = port.mlp_tile_means(x1, w1, 2).copy()
    cache[0, 0] -= np.array([3, 1, 2, 0, 0, 0], np.float32)
    assert port.mlp_change_indices(x1, w1, cache, 2, 2)[0, 0, 0].tolist() == [0, 2]


def test_mlp_golden(port, golden):
    g = golden("mlp")
    out, pre, act = port.dense_mlp(g["x1"], g["w1"], g["b1"], g["w2"], g["b2"])
    assert np.array_equal(out, g["d_out"]) and np.array_equal(act, g["d_act"])
    assert np.array_equal(port.mlp_tile_means(g["x1"], g["w1"], 4), g["tm"])
    ci = port.mlp_change_indices(g["x2"], g["w1"], g["tm"], 7, 4)
    assert np.array_equal(ci, g["ci2"])
    cnt = np.full(ci.shape[:-1], 7, np.int32)
    o2, a2 = port.sparse_delta_mlp(g["x2"], g["w1"], g["b1"], g["w2"], g["b2"], ci, cnt, 4, act, out)
    assert np.array_equal(o2, g["o2"]) and np.array_equal(a2, g["a2"])
    ci3 = port.mlp_change_indices(g["x3"], g["w1"], g["tm"], 7, 4)
    assert np.array_equal(ci3, g["ci3"])
    o3, a3 = port.sparse_delta_mlp(g["x3"], g["w1"], g["b1"], g["w2"], g["b2"], ci3, cnt, 4, a2, o2)
    assert np.array_equal(o3, g["o3"]) and np.array_equal(a3, g["a3"])


def test_mlp_stationary_is_exact(port):
    # test_mlp.cpp:177-184: unchanged input -> sparse step reproduces dense bit-exactly
    x = port.gaussian(40, (1, 8, 5))
    w1, b1, w2, b2 = port.gaussian(41, (9, 5)), port.gaussian(42, (9,)), port.gaussian(43, (9, 5)), port.gaussian(44, (5,))
    out, _, act = port.dense_mlp(x, w1, b1, w2, b2)
    tm = port.mlp_tile_means(x, w1, 4)
    ci = port.mlp_change_indices(x, w1, tm, 3, 4)
    o2, _ = port.sparse_delta_mlp(x, w1, b1, w2, b2, ci, np.full(ci.shape[:-1], 3, np.int32), 4, act, out)
    assert np.array_equal(o2, out)


# ---------------------------------------------------------------- differential vs reference
def test_random_shapes_match_reference(port, ref):
    rng = np.random.default_rng(7)
    for trial in range(12):
        chunk = int(rng.choice([2, 4, 8]))
        n = chunk * int(rng.integers(2, 6))
        e = int(rng.integers(2, 9))
        b, h = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        q, k, v = (port.gaussian(9000 + 3 * trial + i, (b, h, n, e)) for i in range(3))
        o1, c1, s1 = port.column_sum_attention(q, k, v, None, chunk)
        o2, c2, s2 = ref.column_sum_attention(q, k, v, None, chunk)
        assert np.array_equal(o1, o2) and np.array_equal(c1, c2)
        kk = int(rng.integers(1, n + 1))
        i1, i2 = port.select_top_k(c1, kk), ref.select_top_k(c2, kk)
        assert np.array_equal(i1, i2)
        cnt = np.full(i1.shape[:-1], kk, np.int32)
        assert np.array_equal(port.sparse_delta_attention(q, k, v, i1, cnt, chunk, o1, -1.0),
                              ref.sparse_delta_attention(q, k, v, i2, cnt, chunk, o2, -1.0))
