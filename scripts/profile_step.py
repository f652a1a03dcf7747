"""Run a few eager FLUX-block steps for ncu launch lists / full captures.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python scripts/profile_step.py
Runs: dense (init), sparse x2 (warm), then the profiled pair: one dense + one sparse step.
--only sparse|dense: profile a single step of that kind (use ncu --profile-from-start off).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03275_b200 import ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="step", choices=["step", "sparse", "dense"])
    args = ap.parse_args()
    cfg = dict(bench.FLUX)
    n = cfg["grid"][1] * cfg["grid"][2]
    ak, mk = bench.k_of(n, cfg["sparsity"]), bench.k_of(cfg["hidden"], cfg["sparsity"])
    bc = ops.BlockConfig(batch=1, seq=n, dim=cfg["dim"], heads=cfg["heads"],
                         head_dim=cfg["head_dim"], hidden=cfg["hidden"], chunk=cfg["chunk"],
                         attn_k=ak, mlp_k=mk)
    blk = ops.Block(bc, bench.make_weights(cfg), production=True)
    x = torch.randn((1, n, cfg["dim"]), device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    for dense in (True, False, False):
        blk.step(x, dense, out=y)
    torch.cuda.synchronize()
    kinds = {"step": (True, False), "sparse": (False,), "dense": (True,)}[args.only]
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures only this window
    for dense in kinds:
        blk.step(x, dense, out=y)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled steps:", kinds, flush=True)


if __name__ == "__main__":
    main()
