"""The block-stack API (include/csd/model.hpp) as a reference caller uses it.

tests/cpp/model_mirror.cpp is compiled against our headers and libcsd_host.so exactly as a
reference user would recompile (build_toy_model -> make_state -> model_forward_step over a
D S S D S schedule, 2 layers, outputs fed back), then run on the GPU; every output must equal
the reference library's bit for bit (tests/golden/model_stack.npz, oracle/gen_golden.py).
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2506_03275_b200")


def _compile(tmp_path):
    exe = str(tmp_path / "model_mirror")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "model_mirror.cpp"), "-o", exe,
           "-L", PKG, "-l:libcsd_host.so", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_model_mirror_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(PKG, "libcsd_host.so")):
        pytest.skip("libcsd_host.so not built")
    exe = _compile(tmp_path)
    out = subprocess.run(["nm", "-D", "--undefined-only", exe], capture_output=True, text=True).stdout
    for sym in ("model_forward_step", "model_forward_dense", "build_toy_model", "make_state"):
        assert sym in out, sym


@pytest.mark.gpu
def test_model_forward_step_bit_exact(cuda, golden, tmp_path):
    g = golden("model_stack")
    exe = _compile(tmp_path)
    path = str(tmp_path / "out.bin")
    r = subprocess.run([exe, path], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stderr)
    got = np.fromfile(path, dtype=np.float32).reshape(6, *g["x"].shape)
    for t in range(5):
        assert np.array_equal(got[t], g[f"y{t}"]), t
    assert np.array_equal(got[5], g["dense"])
