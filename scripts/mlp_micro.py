"""Sparse-delta MLP (up + down) at the FLUX shape, L2 flushed between repetitions (the
bench's mlp_kernel_bench), for A/B runs of kernel variants selected by environment, e.g.

    python scripts/mlp_micro.py; CSD_SMLP_DOWN=cta python scripts/mlp_micro.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03275_b200 import ops  # noqa: E402

cfg = dict(bench.FLUX)
n = cfg["grid"][1] * cfg["grid"][2]
mk = bench.k_of(cfg["hidden"], cfg["sparsity"])
r = bench.mlp_kernel_bench(ops, torch, cfg, n, mk, 20)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("CSD_")},
                  "sparse_us": round(r["sparse"]["ms"] * 1e3, 1), "dense_us": round(r["dense"]["ms"] * 1e3, 1)}))
