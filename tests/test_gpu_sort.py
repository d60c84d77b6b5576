"""Kernel 2's hand-written primitives (csrc/scan.cu): the single-pass
decoupled look-back exclusive scan and the stable LSD radix sort of
(u64 key, u32 index) pairs, against numpy (cumsum; stable argsort).  The BSP
build (bsp.cu) orders points by (coord key, index) with this sort, so
stability is what makes it the reference comparator's order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 7, 2047, 2048, 2049, 100_003, 1_000_000, 5_000_000])
def test_exclusive_scan(gctx, n):
    a = np.random.default_rng(n).integers(0, 50, n, dtype=np.uint32)
    want = np.concatenate([[0], np.cumsum(a, dtype=np.uint64)[:-1]]).astype(np.uint32)
    assert np.array_equal(gctx.debug_scan(a), want)
    assert np.array_equal(gctx.debug_scan(a), want)  # the look-back state re-arms between calls


@pytest.mark.parametrize("n,bits,dup", [(1, 64, 0), (1000, 64, 0), (1025, 32, 1), (250_000, 64, 1),
                                        (250_000, 12, 1), (1_000_000, 64, 0)])
def test_radix_sort_pairs_stable(gctx, n, bits, dup):
    rng = np.random.default_rng(n + bits)
    if dup:  # many equal keys: stability decides the order
        keys = rng.integers(0, 64, n, dtype=np.uint64) << np.uint64(20)
    else:
        keys = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    vals = np.arange(n, dtype=np.uint32)
    mask = np.uint64((1 << bits) - 1) if bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    order = np.argsort(keys & mask, kind="stable")
    ko, vo = gctx.debug_sort_pairs(keys, vals, bits)
    assert np.array_equal(vo, vals[order])
    assert np.array_equal(ko, keys[order])
