"""TEST INFRASTRUCTURE ONLY — regenerate tests/golden/*.npz from the REFERENCE.

Runs the unmodified reference library (oracle/_ref/libcsd_ref.so, built from
/root/reference/proj/src by `make -C oracle ref`) on small seeded inputs and
stores inputs + outputs.  The fixtures are committed; the GPU box never needs
/root/reference.  Inputs come from the reference's own GaussianRng
(rng.hpp:12-44) so every case is reproducible from its seed.

    python oracle/gen_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def g(seed, shape, std=1.0):
    return O.gaussian(seed, shape, std)


def random_index_set(rng, b, h, nc, k_max, domain, allow_zero=True):
    idx = np.zeros((b, h, nc, k_max), np.int32)
    cnt = np.zeros((b, h, nc), np.int32)
    for bb in range(b):
        for hh in range(h):
            for c in range(nc):
                n = int(rng.integers(0 if allow_zero else 1, k_max + 1))
                sel = rng.permutation(domain)[:n]
                idx[bb, hh, c, :n] = sel
                cnt[bb, hh, c] = n
    return idx, cnt


def main():
    os.makedirs(OUT, exist_ok=True)
    R = O.Oracle("reference")
    rng = np.random.default_rng(2506_03275)

    # ---- voxel permutations (voxel.cpp:18-42): the test_voxel.cpp spot case + random layouts
    vox = {}
    layouts = [((2, 2, 4), (1, 2, 2)), ((1, 48, 96), (1, 6, 32)), ((4, 6, 8), (2, 3, 4)),
               ((2, 8, 8), (1, 2, 2)), ((3, 5, 7), (3, 5, 7)), ((6, 4, 10), (2, 2, 5))]
    for i, (grid, vox_) in enumerate(layouts):
        vox[f"grid{i}"] = np.array(grid, np.int64)
        vox[f"voxel{i}"] = np.array(vox_, np.int64)
        vox[f"perm{i}"] = R.voxel_permutation(grid, vox_)
    x = g(11, (2, 4, 6, 8, 5))
    vox["x"] = x
    vox["x_ordered"] = R.voxel_order(x, (2, 3, 4))
    np.savez_compressed(os.path.join(OUT, "voxel.npz"), **vox)

    # ---- top-k (sparse_index.cpp:64-96): random rows, heavy ties, the tie-rule example
    tk = {}
    s = g(123, (2, 3, 4, 16))
    tk["s0"] = s
    tk["i0"] = R.select_top_k(s, 3)
    s1 = np.round(g(124, (5, 64)) * 2) / 2  # many exact ties
    s1[0, :] = 0.0
    s1[1, ::2] = -0.0
    tk["s1"] = s1.astype(np.float32)
    tk["i1"] = R.select_top_k(tk["s1"], 17)
    tk["s2"] = np.array([[0.1, 0.9, 0.5, 0.5]], np.float32)
    tk["i2"] = R.select_top_k(tk["s2"], 2)
    s3 = g(125, (7, 4608))
    tk["s3"] = s3
    tk["i3"] = R.select_top_k(s3, 323)
    np.savez_compressed(os.path.join(OUT, "topk.npz"), **tk)

    # ---- attention (attention.cpp:59-194)
    at = {}
    q, k, v = g(10, (1, 2, 16, 8)), g(11, (1, 2, 16, 8)), g(12, (1, 2, 16, 8))
    at.update(q=q, k=k, v=v)
    o, cs, (m, l) = R.column_sum_attention(q, k, v, None, 4)
    at.update(cs_out=o, cs_cs=cs, cs_m=m, cs_l=l)
    pm = (m + 0.05 * g(77, m.shape)).astype(np.float32)
    pl = (l * (1 + 0.05 * g(78, l.shape))).astype(np.float32)
    o2, cs2, (m2, l2) = R.column_sum_attention(q, k, v, (pm, pl), 4)
    at.update(prev_m=pm, prev_l=pl, st_out=o2, st_cs=cs2, st_m=m2, st_l=l2)
    at["dense_out"] = R.dense_attention(q, k, v)
    idx, cnt = random_index_set(rng, 1, 2, 4, 6, 16)
    base = g(13, q.shape)
    at.update(sp_idx=idx, sp_cnt=cnt, sp_base=base)
    at["sp_plus"] = R.sparse_delta_attention(q, k, v, idx, cnt, 4, base, 1.0)
    at["sp_minus"] = R.sparse_delta_attention(q, k, v, idx, cnt, 4, base, -1.0)
    # a head_dim-128, chunk-192 slice of the FLUX shape (1 head, N = 768); inputs are
    # regenerated from their seeds (20, 21, 22) by the bit-identical csdo_gaussian
    qf, kf, vf = g(20, (1, 1, 768, 128)), g(21, (1, 1, 768, 128)), g(22, (1, 1, 768, 128))
    of, csf, (mf, lf) = R.column_sum_attention(qf, kf, vf, None, 192)
    idf = R.select_top_k(csf, 54)
    cntf = np.full(idf.shape[:-1], 54, np.int32)
    spf = R.sparse_delta_attention(qf, kf, vf, idf, cntf, 192, of, -1.0)
    at.update(f_seeds=np.array([20, 21, 22]), f_out=of, f_cs=csf, f_m=mf, f_l=lf, f_idx=idf, f_resid=spf)
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **at)

    # ---- MLP (mlp.cpp:49-211)
    ml = {}
    b, n, d, f, c = 2, 16, 12, 40, 4
    x1 = g(30, (b, n, d))
    w1, b1, w2, b2 = g(31, (f, d)), g(32, (f,), 0.5), g(33, (f, d)), g(34, (d,), 0.5)
    out, pre, act = R.dense_mlp(x1, w1, b1, w2, b2)
    tm = R.mlp_tile_means(x1, w1, c)
    ml.update(x1=x1, w1=w1, b1=b1, w2=w2, b2=b2, d_out=out, d_pre=pre, d_act=act, tm=tm)
    x2 = (x1 + 0.1 * g(35, x1.shape)).astype(np.float32)
    ci = R.mlp_change_indices(x2, w1, tm, 7, c)
    cnt = np.full(ci.shape[:-1], 7, np.int32)
    o2, a2 = R.sparse_delta_mlp(x2, w1, b1, w2, b2, ci, cnt, c, act, out)
    x3 = (x2 + 0.1 * g(36, x1.shape)).astype(np.float32)
    ci3 = R.mlp_change_indices(x3, w1, tm, 7, c)
    o3, a3 = R.sparse_delta_mlp(x3, w1, b1, w2, b2, ci3, cnt, c, a2, o2)
    ml.update(x2=x2, ci2=ci, o2=o2, a2=a2, x3=x3, ci3=ci3, o3=o3, a3=a3)
    np.savez_compressed(os.path.join(OUT, "mlp.npz"), **ml)

    # ---- block trajectory (model.cpp:178-216): desk-like config, D S S D S
    cfg = dict(batch=1, grid=(2, 8, 8), dim=64, head_dim=16, heads=4, hidden=128, layers=1,
               voxel=(1, 2, 2), chunk=4, seed=1234)
    M = O.RefModel(cfg)
    bl = {"cfg_grid": np.array(cfg["grid"]), "cfg_misc": np.array(
        [cfg["batch"], cfg["dim"], cfg["head_dim"], cfg["heads"], cfg["hidden"], cfg["chunk"],
         cfg["seed"]])}
    for kname, val in M.weights(0).items():
        bl["w_" + kname] = val
    attn_k, mlp_k = 8, 32
    bl["ks"] = np.array([attn_k, mlp_k])
    sched = [1, 0, 0, 1, 0]
    bl["sched"] = np.array(sched)
    xs = g(1235, (1, M.n, cfg["dim"]))
    for t, dense in enumerate(sched):
        xin = (xs + 0.05 * t * g(2000 + t, xs.shape)).astype(np.float32)
        y = M.step(xin, dense, attn_k, mlp_k)
        bl[f"x{t}"] = xin
        bl[f"y{t}"] = y
        ai, ac = M.indices(0, False, attn_k)
        bl[f"aidx{t}"] = ai
        if not dense:
            mi, mc = M.indices(0, True, mlp_k)
            bl[f"midx{t}"] = mi
    np.savez_compressed(os.path.join(OUT, "block.npz"), **bl)

    # ---- static attention pattern (model.hpp:97-99, attention.hpp:50-52): applied verbatim
    # on dense steps, ragged counts including 0 (test_attention.cpp:441-459); D S S D S
    cfg = dict(batch=1, grid=(2, 8, 8), dim=64, head_dim=16, heads=4, hidden=128, layers=1,
               voxel=(1, 2, 2), chunk=4, seed=1234)
    M = O.RefModel(cfg)
    rng = np.random.default_rng(441)
    nc = M.n // cfg["chunk"]
    sidx, scnt = random_index_set(rng, 1, cfg["heads"], nc, 8, M.n)
    st = {"idx": sidx, "counts": scnt, "sched": np.array(sched)}
    for kname, val in M.weights(0).items():
        st["w_" + kname] = val
    for t, dense in enumerate(sched):
        xin = (xs + 0.05 * t * g(2000 + t, xs.shape)).astype(np.float32)
        st[f"x{t}"] = xin
        st[f"y{t}"] = M.step_static(xin, dense, attn_k, mlp_k, sidx, scnt)
    np.savez_compressed(os.path.join(OUT, "block_static.npz"), **st)

    # ---- block stack through model_forward_step (model.hpp defaults, 2 layers), fed back
    # step to step like harness.cpp:186-212; tests/cpp/model_mirror.cpp replays it
    cfg = dict(batch=1, grid=(2, 8, 8), dim=64, head_dim=16, heads=4, hidden=128, layers=2,
               voxel=(1, 2, 2), chunk=4, seed=1234)
    M = O.RefModel(cfg)
    x = g(1235, (1, M.n, cfg["dim"]))
    ms = {"x": x}
    cur = x
    for t, dense in enumerate([1, 0, 0, 1, 0]):
        cur = M.step(cur, dense, 8, 32)
        ms[f"y{t}"] = cur
    ms["dense"] = M.dense(x)
    np.savez_compressed(os.path.join(OUT, "model_stack.npz"), **ms)

    # ---- generation driver (harness.cpp:123-224, schedule.cpp:44-87):
    # 2-layer desk model, 12 steps, dense every 4th, step cache window 6 stride 2
    cfg = dict(batch=1, grid=(2, 8, 8), dim=64, head_dim=16, heads=4, hidden=128, layers=2,
               voxel=(1, 2, 2), chunk=4, seed=1234)
    sched = dict(total_steps=12, dense_interval=3, step_cache=True, window=6, stride=2,
                 attn_k=8, mlp_k=32)
    modes, r2, e2e, fin = O.run_generation(cfg, sched)
    M = O.RefModel(cfg)
    gen = {"cfg_grid": np.array(cfg["grid"]), "cfg_voxel": np.array(cfg["voxel"]),
           "cfg_misc": np.array([cfg["batch"], cfg["dim"], cfg["head_dim"], cfg["heads"],
                                 cfg["hidden"], cfg["layers"], cfg["chunk"], cfg["seed"]]),
           "sched": np.array([sched[k] for k in ("total_steps", "dense_interval", "step_cache",
                                                 "window", "stride", "attn_k", "mlp_k")]),
           "grid0": g(cfg["seed"] + 1, (cfg["batch"], *cfg["grid"], cfg["dim"])),  # harness.cpp:16-22
           "modes": modes, "latent_r2": r2, "e2e_r2": np.array([e2e]), "final": fin}
    for layer in range(cfg["layers"]):
        for kname, val in M.weights(layer).items():
            gen[f"l{layer}_{kname}"] = val
    np.savez_compressed(os.path.join(OUT, "generation.npz"), **gen)
    # schedule cases (schedule.cpp): (total, interval, cache, window, stride) -> modes
    cases = [(1, 0, 0, 0, 1), (20, 10, 0, 0, 1), (50, 10, 1, 30, 4), (12, 3, 1, 6, 2),
             (7, 0, 1, 7, 3), (9, 2, 1, 1, 1), (30, 4, 1, 10, 1)]
    sc = {"cases": np.array(cases, np.int64)}
    for i, cs in enumerate(cases):
        sc[f"modes{i}"] = O.resolve_schedule(*cs)
    np.savez_compressed(os.path.join(OUT, "schedule.npz"), **sc)
    for fn in sorted(os.listdir(OUT)):
        print(fn, os.path.getsize(os.path.join(OUT, fn)))


if __name__ == "__main__":
    main()
