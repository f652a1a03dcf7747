"""Bitpacked index-set masks on the device (bitmask.cpp:55-85,
bitmask.hpp:13-17, the reference's test_cache_store.cpp:62-110 cases) against a numpy
restatement, plus the reference's validation errors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _set(ops, torch, idx, cnt, domain):
    b, h, c, k = idx.shape
    return ops.SparseIndexSet(b, h, c, 4, k, domain, torch.as_tensor(idx, dtype=torch.int32).cuda(),
                              torch.as_tensor(cnt, dtype=torch.int32).cuda())


def _np_masks(idx, cnt, n):
    b, h, c, _ = idx.shape
    out = np.zeros((b, h, c, (n + 7) // 8), np.uint8)
    for ii in np.ndindex(b, h, c):
        bits = np.zeros(((n + 7) // 8) * 8, np.uint8)
        bits[idx[ii][:cnt[ii]]] = 1
        out[ii] = np.packbits(bits, bitorder="little")
    return out


def test_reference_examples(cuda):
    import torch
    from paper_2506_03275_b200 import ops
    m = ops.index_set_to_masks(_set(ops, torch, np.array([[[[1, 3]]]]), np.array([[[2]]]), 4), 4)
    assert m.cpu().numpy().ravel().tolist() == [0x0A]
    full = np.arange(8, dtype=np.int32).reshape(1, 1, 1, 8)
    m = ops.index_set_to_masks(_set(ops, torch, full, np.array([[[8]]]), 8), 8)
    assert m.cpu().numpy().ravel().tolist() == [0xFF]


@pytest.mark.parametrize("n,k", [(16, 5), (4608, 323), (12288, 860), (1000, 999), (37, 0)])
def test_random_sets_match_numpy(cuda, n, k):
    import torch
    from paper_2506_03275_b200 import ops
    rng = np.random.default_rng(n + k)
    b, h, c = 2, 3, 5
    idx = np.zeros((b, h, c, max(k, 1)), np.int32)
    cnt = rng.integers(0, k + 1, size=(b, h, c)).astype(np.int32)
    for ii in np.ndindex(b, h, c):
        idx[ii][:cnt[ii]] = rng.permutation(n)[:cnt[ii]]
    s = _set(ops, torch, idx, cnt, n)
    s.k_max = k
    got = ops.index_set_to_masks(s, n + 5).cpu().numpy()  # longer masks than the domain are fine
    assert np.array_equal(got, _np_masks(idx, cnt, n + 5))
    pop = np.unpackbits(got, axis=-1, bitorder="little").sum(-1)
    assert np.array_equal(pop, cnt)


def test_validation_errors(cuda):
    import torch
    from paper_2506_03275_b200 import errors, ops
    dup = _set(ops, torch, np.array([[[[2, 2]]]]), np.array([[[2]]]), 8)
    with pytest.raises(errors.IndexError):
        ops.index_set_to_masks(dup, 8)
    oor = _set(ops, torch, np.array([[[[1, 9]]]]), np.array([[[2]]]), 8)
    with pytest.raises(errors.IndexError):
        ops.index_set_to_masks(oor, 8)
    with pytest.raises(errors.ValueError):
        ops.index_set_to_masks(_set(ops, torch, np.array([[[[1, 3]]]]), np.array([[[2]]]), 8), 4)
    # the context is clean again after an error
    ok = ops.index_set_to_masks(_set(ops, torch, np.array([[[[1, 3]]]]), np.array([[[2]]]), 4), 4)
    assert ok.cpu().numpy().ravel().tolist() == [0x0A]
