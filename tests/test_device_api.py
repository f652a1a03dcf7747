"""The production (bf16 / tcgen05) route behind the reference C++ API, include/csd/device.hpp.

tests/cpp/device_api.cpp is compiled against our headers and libcsd_host.so as a reference
caller would; on the GPU it checks csd::dev:: attention / MLP ops and DeviceModel (a 2-layer
toy model over D S S D S) against the CHECK-mode csd:: functions within relative L2 2e-2.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2506_03275_b200")


def _compile(tmp_path):
    exe = str(tmp_path / "device_api")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "device_api.cpp"), "-o", exe,
           "-L", PKG, "-l:libcsd_host.so", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_device_api_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(PKG, "libcsd_host.so")):
        pytest.skip("libcsd_host.so not built")
    exe = _compile(tmp_path)
    out = subprocess.run(["nm", "-D", "-C", "--undefined-only", exe], capture_output=True,
                         text=True).stdout
    for sym in ("csd::dev::DeviceModel::forward_step", "csd::dev::sparse_delta_attention",
                "csd::dev::dense_mlp"):
        assert sym in out, sym


@pytest.mark.gpu
def test_device_api_on_b200(cuda, tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "device api tests passed" in r.stdout
