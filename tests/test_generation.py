"""Multi-step generation driver (harness.cpp:123-224,
schedule.cpp:44-87, metrics.cpp:5-30).

CPU: the schedule resolver against the reference's own resolutions (tests/golden/
schedule.npz, produced by oracle/gen_golden.py from the compiled reference) and its
ConfigError cases.  GPU: a CHECK-mode generation (2 layers, 12 steps with a step-cache
window) reproduces the reference's decoded final latent bit-for-bit and its per-step
latent R^2; a PROD generation (cfg1-shaped, CUDA graphs) stays within the bf16 tolerance
of the CHECK run.
"""
import numpy as np
import pytest

from paper_2506_03275_b200 import errors, generation as G

REL_L2_TOL = 2e-2


def test_schedule_matches_reference(golden):
    g = golden("schedule")
    for i, case in enumerate(g["cases"]):
        total, interval, cache, window, stride = (int(v) for v in case)
        modes = G.resolve_schedule(total, interval, bool(cache), window, stride)
        assert modes == g[f"modes{i}"].tolist(), case


def test_schedule_reference_counts():
    # test_schedule.cpp:42-43: 50 steps, dense every 11th, window 30 stride 4 -> 22 skipped
    modes = G.resolve_schedule(50, 10, True, 30, 4)
    assert modes.count(G.SKIPPED) == 22
    # window [10, 40): the dense boundaries 11 and 33 fall off the stride grid and are skipped
    assert [s for s, m in enumerate(modes) if m == G.DENSE] == [0, 22, 44]
    # no step cache: dense at every (interval + 1) boundary
    assert G.resolve_schedule(5, 0) == [G.DENSE] * 5
    assert G.resolve_schedule(7, 2) == [0, 1, 1, 0, 1, 1, 0]


@pytest.mark.parametrize("args", [(0, 1, False, 0, 1), (5, -1, False, 0, 1),
                                  (5, 1, True, 0, 1), (5, 1, True, 6, 1), (5, 1, True, 3, 0)])
def test_schedule_config_errors(args):
    with pytest.raises(errors.ConfigError):
        G.resolve_schedule(*args)


def _golden_layers(ops, g, production):
    misc = [int(v) for v in g["cfg_misc"]]  # batch, dim, head_dim, heads, hidden, layers, chunk, seed
    n = int(np.prod(g["cfg_grid"]))
    sch = [int(v) for v in g["sched"]]
    cfg = ops.BlockConfig(batch=misc[0], seq=n, dim=misc[1], heads=misc[3], head_dim=misc[2],
                          hidden=misc[4], chunk=misc[6], attn_k=sch[5], mlp_k=sch[6])
    names = ("wq", "wk", "wv", "wo", "w1", "b1", "w2", "b2")
    return [ops.Block(cfg, {k: g[f"l{layer}_{k}"] for k in names}, production=production)
            for layer in range(misc[5])]


@pytest.mark.gpu
def test_check_generation_matches_reference(cuda, golden):
    import torch
    from paper_2506_03275_b200 import ops
    g = golden("generation")
    layers = _golden_layers(ops, g, production=False)
    base = _golden_layers(ops, g, production=False)
    t, h, w = (int(v) for v in g["cfg_grid"])
    vt, vh, vw = (int(v) for v in g["cfg_voxel"])
    gen = G.Generation(layers, ops.VoxelLayout(t, h, w, vt, vh, vw), baseline=base)
    sch = [int(v) for v in g["sched"]]
    rep = gen.run(torch.as_tensor(g["grid0"]).cuda(),
                  G.ScheduleParams(total_steps=sch[0], dense_interval=sch[1],
                                   step_cache=bool(sch[2]), window=sch[3], stride=sch[4]))
    assert rep.modes == g["modes"].tolist()
    assert np.array_equal(rep.final_latent.cpu().numpy(), g["final"])
    r2 = np.array([np.nan if s.latent_r2 is None else s.latent_r2 for s in rep.steps])
    np.testing.assert_allclose(r2, g["latent_r2"], rtol=0, atol=1e-9, equal_nan=True)
    assert abs(rep.end_to_end_r2 - float(g["e2e_r2"][0])) < 1e-9


@pytest.mark.gpu
def test_prod_generation_vs_check(cuda, port):
    import torch
    from paper_2506_03275_b200 import ops
    # cfg1-like block (SURVEY 8 conventions), 1 layer, 8 steps: D S S S D + a skip window
    n, d, hh, e, f, c = 1024, 768, 12, 64, 3072, 64
    std = 1 / np.sqrt(d)
    w = {"wq": port.gaussian(11, (d, d), std), "wk": port.gaussian(12, (d, d), std),
         "wv": port.gaussian(13, (d, d), std), "wo": port.gaussian(14, (d, d), std / 2),
         "w1": port.gaussian(15, (f, d), std), "b1": port.gaussian(16, (f,), std),
         "w2": port.gaussian(17, (f, d), std / 2), "b2": port.gaussian(18, (d,), std / 2)}
    w = {k: (v.astype(np.float32) if k in ("b1", "b2") else
             torch.as_tensor(v).to(torch.bfloat16).float().numpy()) for k, v in w.items()}
    cfg = ops.BlockConfig(batch=1, seq=n, dim=d, heads=hh, head_dim=e, hidden=f, chunk=c,
                          attn_k=102, mlp_k=307)
    layout = ops.VoxelLayout(1, 32, 32, 1, 8, 8)
    grid0 = torch.as_tensor(port.gaussian(1235, (1, 1, 32, 32, d))).cuda()
    grid0 = grid0.to(torch.bfloat16).float()  # identical inputs in both modes
    sched = G.ScheduleParams(total_steps=8, dense_interval=3, step_cache=True, window=4, stride=2)
    outs = {}
    for prod in (False, True):
        gen = G.Generation([ops.Block(cfg, w, production=prod)], layout)
        rep = gen.run(grid0, sched)
        assert rep.modes == G.resolve_schedule(8, 3, True, 4, 2)
        assert G.SKIPPED in rep.modes
        outs[prod] = rep.final_latent.double()
        if prod:
            assert gen.use_graphs and len(gen._graphs) == 3
    # the bf16 output contract on the generated latent, and the reference's own quality
    # figure (R^2 of the latent change, metrics.cpp:5-30) between the two modes
    err = float((outs[True] - outs[False]).norm() / outs[False].norm())
    assert err < REL_L2_TOL, err
    x0 = grid0.double()
    dc, dp = outs[False] - x0, outs[True] - x0
    r2 = 1.0 - float(((dc - dp) ** 2).sum() / ((dc - dc.mean()) ** 2).sum())
    assert r2 > 0.99, r2


@pytest.mark.gpu
def test_r_squared_matches_definition(cuda):
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    t = torch.randn(1000003, device="cuda", generator=g)
    a = t + 0.1 * torch.randn(t.shape, device="cuda", generator=g)
    o = torch.randn(t.shape, device="cuda", generator=g)
    got = G.r_squared(t, a, o)
    dt, da = t.double() - o.double(), a.double() - o.double()  # deltas in double, like the kernel
    want = 1.0 - float(((dt - da) ** 2).sum() / ((dt - dt.mean()) ** 2).sum())
    assert abs(got - want) < 1e-10
    with pytest.raises(errors.NumericError):
        G.r_squared(o, a, o)  # zero-variance true delta


@pytest.mark.gpu
@pytest.mark.parametrize("layers,prod", [(4, True), (3, True), (3, False)])
def test_offloaded_caches_match_resident(cuda, port, layers, prod):
    """Cache offload (memory.cpp:33-58: two layers' caches on the device, the rest in host
    memory, streamed per layer) runs the same kernels on the same data, so the generated
    latent must be BIT-identical to the all-resident run -- PROD with CUDA graphs (the
    captured step includes the copy-stream traffic) and CHECK eagerly, even and odd stacks."""
    import torch
    from paper_2506_03275_b200 import ops
    n, d, hh, e, f, c = 512, 256, 4, 64, 1024, 64
    std = 1 / np.sqrt(d)
    cfg = ops.BlockConfig(batch=1, seq=n, dim=d, heads=hh, head_dim=e, hidden=f, chunk=c,
                          attn_k=64, mlp_k=128)

    def weights(l):
        base = 100 * (l + 1)
        return {"wq": port.gaussian(base + 1, (d, d), std), "wk": port.gaussian(base + 2, (d, d), std),
                "wv": port.gaussian(base + 3, (d, d), std), "wo": port.gaussian(base + 4, (d, d), std / 2),
                "w1": port.gaussian(base + 5, (f, d), std), "b1": port.gaussian(base + 6, (f,), std),
                "w2": port.gaussian(base + 7, (f, d), std / 2), "b2": port.gaussian(base + 8, (d,), std / 2)}
    ws = [weights(l) for l in range(layers)]
    layout = ops.VoxelLayout(1, 16, 32, 1, 8, 8)
    grid0 = torch.as_tensor(port.gaussian(77, (1, 1, 16, 32, d))).cuda().to(torch.bfloat16).float()
    sched = G.ScheduleParams(total_steps=7, dense_interval=2, step_cache=True, window=3, stride=2)
    finals, mems = {}, {}
    for off in (False, True):
        gen = G.Generation([ops.Block(cfg, w, production=prod) for w in ws], layout, offload=off)
        assert gen.offload == off
        rep = gen.run(grid0, sched)
        finals[off] = rep.final_latent.cpu()
        mems[off] = gen.memory_report()
    assert torch.equal(finals[True], finals[False])
    assert mems[True]["cache_device_bytes"] * layers == 2 * mems[False]["cache_device_bytes"]


@pytest.mark.gpu
@pytest.mark.parametrize("prod", [True, False])
def test_forward_dense_equals_dense_step_output(cuda, port, prod):
    """model_forward_dense (csd_block_step kind 2): the output of a Chipmunk dense step (the
    exact attention and MLP the caches are refreshed from), with every cache left untouched."""
    import torch
    from paper_2506_03275_b200 import ops
    n, d, hh, e, f, c = 512, 256, 4, 64, 1024, 64
    std = 1 / np.sqrt(d)
    w = {"wq": port.gaussian(1, (d, d), std), "wk": port.gaussian(2, (d, d), std),
         "wv": port.gaussian(3, (d, d), std), "wo": port.gaussian(4, (d, d), std / 2),
         "w1": port.gaussian(5, (f, d), std), "b1": port.gaussian(6, (f,), std),
         "w2": port.gaussian(7, (f, d), std / 2), "b2": port.gaussian(8, (d,), std / 2)}
    cfg = ops.BlockConfig(batch=1, seq=n, dim=d, heads=hh, head_dim=e, hidden=f, chunk=c,
                          attn_k=64, mlp_k=128)
    blk = ops.Block(cfg, w, production=prod)
    dt = torch.bfloat16 if prod else torch.float32
    x = torch.as_tensor(port.gaussian(9, (1, n, d))).cuda().to(dt)
    x2 = torch.as_tensor(port.gaussian(10, (1, n, d))).cuda().to(dt)
    y_dense = blk.step(x, True)
    caches = [blk.cache(i) for i in range(6)] + list(blk.indices(False)) + list(blk.indices(True))
    y_plain = blk.forward_dense(x2)  # a different input: the caches must not move
    after = [blk.cache(i) for i in range(6)] + list(blk.indices(False)) + list(blk.indices(True))
    for a, b in zip(caches, after):
        assert torch.equal(a, b)
    y_plain_x = blk.forward_dense(x)
    if prod:  # same kernels except the attention pass (dense vs column-sum): bf16 contract
        err = float((y_plain_x.float() - y_dense.float()).norm() / y_dense.float().norm())
        assert err < 1e-2, err
    else:
        assert torch.equal(y_plain_x, y_dense)
    assert not torch.equal(y_plain, y_plain_x)
