"""The opt-in launch modes give the default path's results (B200).

* ``CSD_PDL=2`` (programmatic dependent launch of every block-step kernel: each kernel's
  prologue overlaps its predecessor, ``pdl_wait`` before its first global access) runs the
  same kernels, so the PROD block trajectory must be BIT-identical to the plain launches.
* ``CSD_ATTN_CP=1`` routes the block's sparse-delta attention through the CTA-pair kernel
  (attn_cp.cu): a different summation order, so the trajectory must agree within the bf16
  contract (relative L2 <= 2e-2 on the branch outputs).

The knobs are read once per process, so each mode runs in a subprocess.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import bench
from paper_2506_03275_b200 import ops
cfg = dict(bench.FLUX, dim=1024, heads=8, hidden=4096, grid=[1, 12, 64])
n = 12 * 64
bc = ops.BlockConfig(batch=1, seq=n, dim=1024, heads=8, head_dim=128, hidden=4096, chunk=192,
                     attn_k=bench.k_of(n, 0.9), mlp_k=bench.k_of(4096, 0.9))
blk = ops.Block(bc, bench.make_weights(cfg), production=True)
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn((1, n, 1024), device="cuda", generator=g).to(torch.bfloat16)
outs = []
for dense in (True, False, False, True, False):
    y = blk.step(x, dense)
    outs.append((y.float() - x.float()).cpu().numpy())
    x = (x.float() + 0.02 * y.float()).to(torch.bfloat16)
torch.cuda.synchronize()
np.save({out!r}, np.stack(outs))
"""


def _run(tmp_path, name, env):
    out = str(tmp_path / f"{name}.npy")
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, out=out)], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_pdl_and_pair_attention_match_default(tmp_path):
    base = _run(tmp_path, "default", {"CSD_PDL": "0", "CSD_ATTN_CP": "0"})
    pdl = _run(tmp_path, "pdl", {"CSD_PDL": "2", "CSD_ATTN_CP": "0"})
    assert np.array_equal(pdl, base)
    cp = _run(tmp_path, "cp", {"CSD_PDL": "0", "CSD_ATTN_CP": "1"})
    for s in range(base.shape[0]):
        assert _rel(cp[s], base[s]) < 2e-2, s
