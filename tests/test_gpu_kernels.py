"""Kernel-backend parity on the GPU: libmdrq_b200 vs the reference's golden
vectors and the pinned CPU oracle (pkg/tests/test_kernels.py counterpart)."""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    return golden("kernels.npz")


@pytest.mark.parametrize("m", [1, 7, 8, 9, 20, 100])
def test_match_rows_vs_golden(gpu, K, m):
    rows, lo, hi = K[f"match_m{m}_row"], K[f"match_m{m}_lo"], K[f"match_m{m}_hi"]
    exp = K[f"match_m{m}_scalar"]
    assert np.array_equal(exp, K[f"match_m{m}_blocked"])
    for i in range(0, rows.shape[0], 15):
        assert gpu.kernels.match_row(rows[i], lo[i], hi[i], gpu.kernels.MODE_SCALAR) == exp[i]
    # all 300 rows through the batched entry point, each against its own box
    got = np.array([gpu.kernels.match_rows(rows[i:i + 1], lo[i], hi[i])[0] for i in range(rows.shape[0])])
    assert np.array_equal(got, exp)


def test_match_with_sentinels(gpu):
    row = np.array([0.5, 0.5], dtype=np.float32)
    lower = np.array([-np.inf, 0.4], dtype=np.float32)
    upper = np.array([np.inf, 0.6], dtype=np.float32)
    for mode in (0, 1):
        assert gpu.kernels.match_row(row, lower, upper, mode) is True


def test_scan_rows_vs_golden(gpu, K):
    for ci, (n, m) in enumerate(K["scan_cases"]):
        v, lo, hi = K[f"scan{ci}_values"], K[f"scan{ci}_lo"], K[f"scan{ci}_hi"]
        for mode in (0, 1):
            ids, compared, early = gpu.kernels.scan_rows(v, lo, hi, mode)
            assert np.array_equal(ids, K[f"scan{ci}_ids"]), (n, m, mode)
            assert ids.dtype == np.int64
            assert compared == n
            assert early == K[f"scan{ci}_early"][mode], (n, m, mode)


def test_scan_rows_early_break_counter(gpu):
    values = np.array([[0.5, 0.5], [2.0, 0.5], [0.5, 2.0]], dtype=np.float32)
    ids, compared, early = gpu.kernels.scan_rows(values, np.zeros(2, np.float32), np.ones(2, np.float32), 0)
    assert ids.tolist() == [0] and compared == 3 and early == 1


def test_scan_column_vs_golden(gpu, K):
    for ci, n in enumerate(K["col_cases"]):
        col = K[f"col{ci}_col"]
        lo, hi = K[f"col{ci}_lohi"]
        assert np.array_equal(gpu.kernels.scan_column(col, lo, hi), K[f"col{ci}_mask"]), n


@given(n=st.integers(0, 3000), m=st.integers(1, 24), seed=st.integers(0, 2**20))
@settings(max_examples=40, deadline=None)
def test_scan_rows_random_vs_oracle(gpu, n, m, seed):
    rng = np.random.default_rng(seed)
    v = rng.random((n, m), dtype=np.float32)
    lo = (rng.random(m) * 0.6).astype(np.float32)
    hi = lo + (rng.random(m) * 0.8).astype(np.float32)
    for mode in (0, 1):
        exp = oracle.scan_rows(v, lo, hi, mode)
        got = gpu.kernels.scan_rows(v, lo, hi, mode)
        assert np.array_equal(got[0], exp[0]) and got[1] == exp[1] and got[2] == exp[2]


@given(nbytes=st.integers(0, 700), k=st.integers(1, 20), seed=st.integers(0, 999))
@settings(max_examples=30, deadline=None)
def test_mask_algebra_vs_oracle(gpu, nbytes, k, seed):
    rng = np.random.default_rng(seed)
    masks = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(k)]
    merged = gpu.kernels.and_masks(masks)
    exp = oracle.and_masks(masks) if nbytes else np.zeros(0, np.uint8)
    assert np.array_equal(merged, exp)
    assert gpu.kernels.mask_popcount(merged) == (oracle.mask_popcount(merged) if nbytes else 0)
    n = max(0, nbytes * 8 - int(rng.integers(0, 8)))
    assert np.array_equal(gpu.kernels.mask_to_ids(merged, n), oracle.np_mask_to_ids(merged, n))


def test_mask_to_ids_large(gpu):
    rng = np.random.default_rng(1)
    mask = (rng.random(1_000_003 // 8 + 1) < 0.3).astype(np.uint8) * rng.integers(0, 256, 1_000_003 // 8 + 1,
                                                                                   dtype=np.uint8)
    n = 1_000_003
    assert np.array_equal(gpu.kernels.mask_to_ids(mask, n), oracle.np_mask_to_ids(mask, n))


def test_nan_rejected_at_kernel_level(gpu):
    v = np.array([[0.1, np.nan]], np.float32)
    with pytest.raises(ValueError, match="NaN"):
        gpu.kernels.scan_rows(v, np.zeros(2, np.float32), np.ones(2, np.float32), 0)


def test_copy_segments_merge_vs_numpy(gpu):
    """mdrq_copy_segments, the device placement of the multi-GPU id merge
    (parallel.combine_ids): random aligned / unaligned segments of three
    simulated ranks land where the rank-ordered concatenation puts them."""
    import ctypes
    import torch
    from paper_1801_03644_b200 import _lib
    from paper_1801_03644_b200.parallel import combine_ids
    rng = np.random.default_rng(9)
    world, nq = 3, 57
    counts = rng.integers(0, 300, (world, nq))
    counts[1, 5] = 0
    counts[:, 7] = 0
    stride = int(counts.sum(1).max()) + 3
    gathered = np.zeros((world, stride), np.uint32)
    expect = []
    per_q = [[] for _ in range(nq)]
    for r in range(world):
        o = 0
        for q in range(nq):
            seg = np.sort(rng.integers(r * 10**6, (r + 1) * 10**6, counts[r, q])).astype(np.uint32)
            gathered[r, o:o + seg.size] = seg
            per_q[q].append(seg)
            o += seg.size
    expect = np.concatenate([np.concatenate(x) for x in per_q])
    out_off = np.zeros(nq + 1, np.int64)
    out_off[1:] = np.cumsum(counts.sum(0))
    rank_prefix = np.cumsum(counts, 0) - counts
    loff = np.cumsum(counts, 1) - counts
    src_off = (loff + np.arange(world)[:, None] * stride).astype(np.int64).ravel()
    dst_off = (out_off[:-1][None, :] + rank_prefix).astype(np.int64).ravel()
    seg_len = counts.astype(np.int64).ravel()
    dev = torch.device("cuda", 0)
    t = {k: torch.as_tensor(v).to(dev) for k, v in dict(g=gathered.view(np.int32), s=src_off, d=dst_off,
                                                           n=seg_len).items()}
    out = torch.zeros(int(out_off[-1]) + 1, dtype=torch.int32, device=dev)
    rc = _lib.load().mdrq_copy_segments(ctypes.c_void_p(t["g"].data_ptr()), ctypes.c_void_p(out.data_ptr() + 4),
                                        ctypes.c_void_p(t["s"].data_ptr()), ctypes.c_void_p(t["d"].data_ptr()),
                                        ctypes.c_void_p(t["n"].data_ptr()), world * nq, None)
    _lib.check(rc)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)
    assert got[0] == 0 and np.array_equal(got[1:], expect)
