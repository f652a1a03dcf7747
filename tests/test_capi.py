"""CPU tests of the C-ABI library: it loads, exports exactly what include/csd_b200.h
declares, reports errors without a GPU, and its SASS carries the Blackwell-native
instructions (tcgen05 MMA, TMEM loads, TMA gather4) the design claims."""
import ctypes as C
import os
import shutil
import subprocess

import pytest

from paper_2506_03275_b200 import _capi


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_capi.LIB_PATH):
        from paper_2506_03275_b200 import build
        build.build()
    return _capi.lib()


def test_exports_every_header_symbol(lib):
    syms = _capi.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the binding covers the whole header too
    assert set(syms) <= set(_capi.SIGNATURES)


def test_abi_version_and_status_names(lib):
    assert lib.csd_abi_version() == 1
    names = [lib.csd_status_name(i).decode() for i in range(9)]
    assert names[:7] == ["OK", "ShapeError", "IndexError", "NumericError", "StateError",
                         "ValueError", "ConfigError"]


def test_host_permutation_and_config_error(lib):
    perm = (C.c_int64 * 16)()
    assert lib.csd_voxel_permutation(2, 2, 4, 1, 2, 2, perm) == 0
    assert perm[4] == 2  # test_voxel.cpp:38-44
    assert lib.csd_voxel_permutation(2, 3, 4, 1, 2, 2, perm) == _capi.ERR_CONFIG
    assert b"does not tile" in lib.csd_last_error()


def test_ctx_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert lib.csd_ctx_create(0, C.byref(h)) == _capi.ERR_CUDA


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")
def test_sass_is_blackwell_native(lib):
    sass = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTCHMMA", "LDTM", "UTMALDG.2D.GATHER4", "UTMALDG.2D"):
        assert mnemonic in sass, mnemonic
    assert "arch = sm_100a" in sass
