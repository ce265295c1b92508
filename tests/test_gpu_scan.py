"""The device exclusive scan behind the compactions and counting sorts
(mpmrb_scan_exclusive_i32; the offsets of the reference's np.flatnonzero in
collision.py:105 / solver.py:202 and its stable argsort in transfer.py:89):
bit-exact against np.cumsum at tile edges (4096 elements per tile), for the
empty input, repeated calls (the single-pass kernel's epoch-tagged tile status
is never reset), and past the single-pass limit (2^25, three-kernel path)."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import paper_2503_05046_b200 as m  # noqa: F401
    from paper_2503_05046_b200 import _lib
    return _lib


def _scan(_lib, a):
    d = torch.from_numpy(a).cuda()
    out = torch.full_like(d, -7)
    tot = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().mpmrb_scan_exclusive_i32(_lib.ctx(), _lib.ptr(d), a.size, _lib.ptr(out),
                                                   _lib.ptr(tot)))
    torch.cuda.synchronize()
    return out.cpu().numpy(), int(tot.item())


@pytest.mark.parametrize("n", [0, 1, 31, 4095, 4096, 4097, 8191, 8193, 100_003, 1 << 20,
                               (1 << 25) - 1, (1 << 25) + 4097])
def test_scan_matches_cumsum(lib, n):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 5, size=n).astype(np.int32)
    if n > 10:
        a[n // 3: n // 2] = 0  # long zero runs (the sparse flags of a compaction)
    want = np.zeros(n, np.int64)
    if n:
        np.cumsum(a[:-1], out=want[1:])
    for _ in range(3):  # the same buffers again: stale tile status must never be read as current
        out, tot = _scan(lib, a)
        assert np.array_equal(out, want.astype(np.int32))
        assert tot == int(a.sum())


def test_scan_rejects_bad_arguments(lib):
    with pytest.raises(Exception):
        lib.check(lib.lib().mpmrb_scan_exclusive_i32(lib.ctx(), None, 5, None, None))
