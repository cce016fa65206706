"""GPU parity: K1 (h/s), K2 (plan), K3/K4 (S.A), column sketch, K5 against the
oracle and the reference's golden outputs.  Bit-exact for h, s, plan and fp64
S.A; tolerances are stated where the arithmetic differs."""

import ctypes
import hashlib
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import oracle as O
from paper_1207_6365_b200 import SparseEmbedding, apply_right, make_sparse_embedding
from paper_1207_6365_b200 import _lib
from paper_1207_6365_b200.sketch import pcg64_state

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def gpu_hash(n, t, seed, r0=0, r1=None):
    r1 = n if r1 is None else r1
    L = _lib.lib()
    hs, ss = pcg64_state(seed, (0, 0)), pcg64_state(seed, (0, 1))
    h = torch.empty(r1 - r0, dtype=torch.int32, device="cuda")
    s = torch.empty(r1 - r0, dtype=torch.int8, device="cuda")
    nb = ctypes.c_size_t()
    _lib.check(L.skt_hash_signs_workspace(r1, t, ctypes.byref(nb)))
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device="cuda")
    _lib.check(L.skt_hash_signs(ctypes.byref(hs), ctypes.byref(ss), r0, r1, t, h.data_ptr(), s.data_ptr(),
                                ws.data_ptr(), nb.value, torch.cuda.current_stream().cuda_stream))
    return h.cpu().numpy().view(np.uint32), s.cpu().numpy()


# ---------------------------------------------------------------- K1
def test_hash_signs_golden():
    z = load("hash_cases.npz")
    meta = json.load(open(os.path.join(GOLDEN, "hash_cases.json")))
    for k, (n, t, seed) in enumerate(meta):
        h, s = gpu_hash(n, t, seed)
        assert np.array_equal(h, z[f"h{k}"]), (n, t, seed)
        assert np.array_equal(s, z[f"s{k}"]), (n, t, seed)


@pytest.mark.parametrize("t", [4000, 65536, 3 * 2**30, 2**31 + 1, 7])
def test_hash_signs_row_ranges(t):
    n = 50_001
    h_full, s_full = O.hash_signs(n, t, 3)
    for r0, r1 in [(0, 1), (1, 2), (17, 4111), (4096, 50_001), (25_000, 25_001), (0, n)]:
        h, s = gpu_hash(n, t, 3, r0, r1)
        assert np.array_equal(h, h_full[r0:r1]), (r0, r1)
        assert np.array_equal(s, s_full[r0:r1]), (r0, r1)


def test_hash_signs_config_sizes():
    """Full-size h/s for configs 1-5 (n up to 16.8M) against the C oracle."""
    for n, t in [(100_000, 4000), (1_000_000, 25_000), (16_777_216, 65_536), (4_194_304, 16_384), (262_144, 400)]:
        h, s = gpu_hash(n, t, 1)
        ho, so = O.hash_signs(n, t, 1)
        assert np.array_equal(h, ho) and np.array_equal(s, so), (n, t)
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))
    for c in ("config1", "config2"):
        h, s = gpu_hash(cfg[c]["n"], cfg[c]["t"], cfg[c]["seed"])
        assert sha(h) == cfg[c]["sha_h"] and sha(s) == cfg[c]["sha_s"]


# ---------------------------------------------------------------- K2
@pytest.mark.parametrize("n,t", [(1, 1), (64, 1), (5, 7), (1000, 2), (4097, 255), (4096, 256), (20_000, 257),
                                 (100_000, 4000), (1_000_000, 25_000), (300_000, 2**20 + 7), (5000, 3 * 2**30)])
def test_plan_matches_stable_counting_sort(n, t):
    op = SparseEmbedding(n, t, seed=n + t)
    h, s = O.hash_signs(n, t, n + t)
    indptr, rows = O.plan(h, t)
    got_rows = op.plan_rows.cpu().numpy().view(np.uint32)
    assert np.array_equal(op.plan_indptr.cpu().numpy(), indptr)
    assert np.array_equal((got_rows & 0x7FFFFFFF).astype(np.int32), rows)
    assert np.array_equal((got_rows >> 31).astype(bool), s[rows] < 0)


@pytest.mark.parametrize("n,t,shift", [(1000, 7, 1), (100_000, 4000, 3), (300_000, 16_384, 2), (50_000, 300, 8),
                                       (20_000, 257, 4), (5000, 1, 2), (4_194_304, 16_384, 2)])
def test_grouped_plan_is_stable_sort_by_group(n, t, shift):
    op = SparseEmbedding(n, t, seed=3)
    h, s = O.hash_signs(n, t, 3)
    gptr, grows, gblo = op.grouped_plan(shift)
    order = np.argsort(h >> shift, kind="stable")
    got = grows.cpu().numpy().view(np.uint32)
    assert np.array_equal((got & 0x7FFFFFFF).astype(np.int64), order)
    assert np.array_equal((got >> 31).astype(bool), s[order] < 0)
    assert np.array_equal(gblo.cpu().numpy(), (h[order] & ((1 << shift) - 1)).astype(np.uint8))
    ngroups = ((t - 1) >> shift) + 1
    want = np.searchsorted(h[order] >> shift, np.arange(ngroups + 1), side="left")
    assert np.array_equal(gptr.cpu().numpy(), want)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("t,d", [(1000, 48), (37, 5), (33, 700), (4096, 1)])
def test_apply_csr_bucket_lane_kernel(dtype, t, d, rng):
    """Long rows (> 16 nonzeros), empty rows, partial last warp of buckets."""
    n = 20_000
    shift = 0
    a = sp.csr_array(sp.random_array((n, d), density=0.15, rng=rng, format="csr"), dtype=dtype)
    # a few long rows (> 16 nonzeros) and empty rows
    a = a.tolil()
    a[17, :] = rng.standard_normal(d)
    a[18, :] = 0
    a[19000, ::2] = rng.standard_normal(len(range(0, d, 2)))
    a = sp.csr_array(a, dtype=dtype)
    op = SparseEmbedding(n, t, seed=d)
    h, s = O.hash_signs(n, t, d)
    ref = O.np_apply_csr(h, s, t, a)
    dev = [torch.from_numpy(x).cuda() for x in (a.indptr, a.indices, a.data)]
    got = op._apply_csr_device(*dev, d, torch.float64, canonical=True, shift=shift)
    assert np.array_equal(got.cpu().numpy(), ref)
    for gshift in (1, 3):  # grouped sweep kernel over bucket-group plans
        if (1 << gshift) * d * 8 <= 24 * 1024:
            got = op._apply_csr_device(*dev, d, torch.float64, canonical=True, shift=gshift)
            assert np.array_equal(got.cpu().numpy(), ref), gshift
    with pytest.raises(ValueError):  # non-canonical input needs the per-bucket plan
        op._apply_csr_device(*dev, d, torch.float64, canonical=False, shift=2)


@pytest.mark.parametrize("itype", [np.int32, np.int64])
@pytest.mark.parametrize("d", [64, 40])
def test_apply_csr_quad_alignment(itype, d, rng):
    """csr_quad (fp32 values, int32 columns, d <= 64; 128-bit loads of the 16
    aligned slots around a row's start): rows of 0..22 entries at every
    alignment -- entries past the 16 slots take the extra slot group, past 20
    the whole-warp tail -- plus dense rows; bit-identical for int32 and int64
    row pointers."""
    n, t = 40_000, 777
    lens = rng.integers(0, min(d, 22) + 1, size=n)
    lens[::97] = d  # dense rows
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(lens)
    indices = np.concatenate([np.sort(rng.choice(d, size=k, replace=False)) for k in lens]).astype(np.int32)
    data = rng.standard_normal(indptr[-1]).astype(np.float32)
    a = sp.csr_array((data, indices, indptr), shape=(n, d))
    op = SparseEmbedding(n, t, seed=d)
    h, s = O.hash_signs(n, t, d)
    ref = O.np_apply_csr(h, s, t, a)
    dev = [torch.from_numpy(x).cuda() for x in (indptr.astype(itype), indices, data)]
    for out_dtype in (torch.float64, torch.float32):
        got = op._apply_csr_device(*dev, d, out_dtype, canonical=True).cpu().numpy()
        assert np.array_equal(got, ref.astype(got.dtype)), out_dtype


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("d", [64, 100, 200])
@pytest.mark.parametrize("tile_rows", ["16", "32"])
def test_apply_csr_sweep_kernel(dtype, d, tile_rows, rng, monkeypatch):
    """csr_sweep (bucket groups of 2 / 4 walked in ascending row order, rows
    of ~16 nonzeros): bit-identical to the reference, incl. dense, empty and
    rows longer than the prefetch width."""
    monkeypatch.setenv("SKT_SWEEP_R", tile_rows)
    n, t = 30_000, 1001
    a = sp.csr_array(sp.random_array((n, d), density=16 / d, rng=rng, format="csr"), dtype=dtype)
    a = a.tolil()
    a[5, :] = rng.standard_normal(d)
    a[6, :] = 0
    a[29_999, ::3] = rng.standard_normal(len(range(0, d, 3)))
    a = sp.csr_array(a, dtype=dtype)
    op = SparseEmbedding(n, t, seed=d + 1)
    h, s = O.hash_signs(n, t, d + 1)
    ref = O.np_apply_csr(h, s, t, a)
    dev = [torch.from_numpy(x).cuda() for x in (a.indptr, a.indices, a.data)]
    for shift in (1, 2):
        for out_dtype in (torch.float64, torch.float32):
            got = op._apply_csr_device(*dev, d, out_dtype, canonical=True, shift=shift).cpu().numpy()
            assert np.array_equal(got, ref.astype(got.dtype)), (shift, out_dtype)


def test_host_views_match_reference_layout():
    op = make_sparse_embedding(9, 5, seed=1)
    h, s = O.hash_signs(9, 5, 1)
    assert np.array_equal(op.bucket, h.astype(np.int64)) and op.bucket.dtype == np.int64
    assert np.array_equal(op.sign, s.astype(np.float64))
    ref = sp.csr_array((s.astype(np.float64), (h.astype(np.int64), np.arange(9))), shape=(5, 9))
    assert np.array_equal(op._mat.toarray(), ref.toarray()) and op._mat.nnz == 9


# ---------------------------------------------------------------- K3 / K4
def _golden_cases():
    return [m for m in json.load(open(os.path.join(GOLDEN, "apply_cases.json"))) if m["kind"] != "right"]


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda m: m["name"])
def test_apply_golden_bit_exact(case):
    z = load("apply_cases.npz")
    name = case["name"]
    op = SparseEmbedding(case["n"], case["t"], case["seed"])
    if case["kind"] == "csr":
        a = sp.csr_array((z[f"{name}_data"], z[f"{name}_indices"], z[f"{name}_indptr"]),
                         shape=tuple(z[f"{name}_shape"]))
    else:
        a = z[f"{name}_a"]
    got = op.apply(a)
    assert got.dtype == np.float64
    assert np.array_equal(got, z[f"{name}_sa"]), name
    # torch CUDA input path, same bits
    if case["kind"] == "dense":
        gt = op.apply(torch.from_numpy(np.ascontiguousarray(a)).cuda())
        assert np.array_equal(gt.cpu().numpy().reshape(got.shape), got)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("d", [1, 2, 3, 5, 20, 33, 64, 128, 130, 257])
def test_apply_dense_shapes(dtype, d, rng):
    n, t = 3000, 211
    a = rng.standard_normal((n, d)).astype(dtype)
    op = SparseEmbedding(n, t, seed=d)
    h, s = O.hash_signs(n, t, d)
    ref = O.apply_dense(h, s, t, a)
    assert np.array_equal(op.apply(a), ref)
    f32 = op.apply(torch.from_numpy(a).cuda(), out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(f32, ref.astype(np.float32))  # one rounding of the exact fp64 sum


def test_apply_dense_bucket_ranges(rng):
    """The multi-GPU pipeline computes SA in bucket ranges: same bits as one launch."""
    n, t, d = 50_000, 1_003, 32
    a = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
    op = SparseEmbedding(n, t, seed=12)
    full = op.apply(a)
    out = torch.empty_like(full)
    for b0, b1 in [(0, 1), (1, 500), (500, 1002), (1002, 1003)]:
        op._apply_dense_device(a, torch.float64, out=out, buckets=(b0, b1))
    assert torch.equal(out, full)
    with pytest.raises(ValueError):
        op._apply_dense_device(a, torch.float64, buckets=(5, 5))


def test_apply_dense_strided_rows(rng):
    n, t = 1000, 37
    big = torch.from_numpy(rng.standard_normal((n, 40))).cuda()
    view = big[:, 3:19]  # lda = 40, misaligned start
    op = SparseEmbedding(n, t, seed=4)
    h, s = O.hash_signs(n, t, 4)
    assert np.array_equal(op.apply(view).cpu().numpy(), O.apply_dense(h, s, t, view.cpu().numpy()))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("d,density", [(1, 0.5), (50, 0.1), (64, 0.25), (300, 0.02), (2000, 0.005)])
def test_apply_csr_shapes(dtype, d, density, rng):
    n, t = 5000, 97
    a = sp.csr_array(sp.random_array((n, d), density=density, rng=rng, format="csr"), dtype=dtype)
    op = SparseEmbedding(n, t, seed=d)
    h, s = O.hash_signs(n, t, d)
    ref = O.np_apply_csr(h, s, t, a)
    assert np.array_equal(op.apply(a), ref)
    a64 = sp.csr_array((a.data, a.indices.astype(np.int64), a.indptr.astype(np.int64)), shape=a.shape)
    assert np.array_equal(op.apply(a64), ref)


def test_apply_csr_long_rows_and_duplicates(rng):
    # rows longer than the staging window and non-canonical duplicates
    n, d, t = 300, 5000, 11
    dense = rng.standard_normal((n, d)) * (rng.random((n, d)) < 0.6)
    a = sp.csr_array(dense)
    op = SparseEmbedding(n, t, seed=9)
    h, s = O.hash_signs(n, t, 9)
    assert np.array_equal(op.apply(a), O.np_apply_csr(h, s, t, a))
    rows = np.repeat(np.arange(50), 40)
    cols = rng.integers(0, 7, size=rows.size)
    vals = rng.standard_normal(rows.size)
    dup = sp.csr_array((vals, cols, np.arange(0, rows.size + 1, 40)), shape=(50, 7))
    assert not dup.has_canonical_format
    op2 = SparseEmbedding(50, 3, seed=2)
    h2, s2 = O.hash_signs(50, 3, 2)
    assert np.array_equal(op2.apply(dup), O.np_apply_csr(h2, s2, 3, dup))


def test_apply_torch_sparse_csr(rng):
    n, d, t = 4000, 64, 300
    a = sp.csr_array(sp.random_array((n, d), density=0.2, rng=rng, format="csr"), dtype=np.float32)
    ta = torch.sparse_csr_tensor(torch.from_numpy(a.indptr.astype(np.int64)), torch.from_numpy(a.indices.astype(np.int64)),
                                 torch.from_numpy(a.data), size=a.shape).cuda()
    op = SparseEmbedding(n, t, seed=1)
    h, s = O.hash_signs(n, t, 1)
    assert np.array_equal(op.apply(ta).cpu().numpy(), O.np_apply_csr(h, s, t, a))


@pytest.mark.parametrize("dtype,d", [(np.float32, 32), (np.float32, 64), (np.float32, 128), (np.float32, 144),
                                     (np.float32, 200), (np.float32, 256), (np.float32, 272), (np.float32, 384),
                                     (np.float32, 512), (np.float64, 20), (np.float64, 64), (np.float64, 100),
                                     (np.float64, 128), (np.float64, 192), (np.float64, 256)])
def test_apply_dense_tma_gather4(dtype, d, rng, monkeypatch):
    """Rows of 512 B .. 2 KB go through the TMA gather4 kernel (dense_g4.cuh;
    one or two column boxes per row), smaller ones through the register gather: bit-identical to the reference order and to the register
    kernel (SKT_DENSE_G4=0 only switches kernels inside the library, so the
    A/B runs in one process through a fresh call), bucket ranges, partial last
    quads, empty buckets, a strided view, and the fused finiteness check."""
    n, t = 5003, 97
    a = (rng.standard_normal((n, d)) * np.exp(rng.standard_normal((n, 1)))).astype(dtype)
    op = SparseEmbedding(n, t, seed=d)
    h, s = O.hash_signs(n, t, d)
    ref = O.apply_dense(h, s, t, a)
    assert np.array_equal(op.apply(a), ref)
    dev = torch.from_numpy(a).cuda()
    for b0, b1 in [(0, 13), (13, 60), (60, 97)]:
        part = op._apply_dense_device(dev, torch.float64, buckets=(b0, b1))
        assert np.array_equal(part[b0:b1].cpu().numpy(), ref[b0:b1])
    wide = torch.zeros((n, d + 8), dtype=dev.dtype, device="cuda")
    wide[:, :d] = dev
    assert np.array_equal(op.apply(wide[:, :d]).cpu().numpy(), ref)  # lda = d + 8 (16-byte multiple)
    sparse_op = SparseEmbedding(50, 40, seed=1)  # most buckets hold 0-3 rows
    a2 = a[:50]
    h2, s2 = O.hash_signs(50, 40, 1)
    assert np.array_equal(sparse_op.apply(a2), O.apply_dense(h2, s2, 40, a2))
    for bad in (np.nan, np.inf, -np.inf):
        b = a.copy()
        b[4321, d // 2] = bad
        with pytest.raises(ValueError):
            op.apply(b)
    b = a.copy()  # +inf and -inf in the same bucket and column: NaN, still caught
    rows = np.flatnonzero(h == h[0])[:2]
    b[rows[0], 3], b[rows[1], 3] = np.inf, -np.inf
    with pytest.raises(ValueError):
        op.apply(b)
    if dtype == np.float64:  # finite values whose fp64 sum overflows: no error, inf in SA (as the reference)
        b = a.copy()
        same = np.flatnonzero((h == h[0]) & (s == s[np.flatnonzero(h == h[0])[0]]))[:2]  # same bucket, same sign
        b[same, 5] = 1.5e308
        got = op.apply(b)
        assert np.isinf(got[h[0], 5]) and np.array_equal(got, O.apply_dense(h, s, t, b))


@pytest.mark.parametrize("d", [452, 500])
def test_apply_dense_rows_beyond_gather4(d, rng, monkeypatch):
    """fp32 rows of 1.8-2 KB that gather4 does not take (d not a multiple of 8)
    fall back to a kernel that fits shared memory; with gather4 disabled the
    2 KB rows too."""
    n, t = 2000, 37
    a = rng.standard_normal((n, d)).astype(np.float32)
    op = SparseEmbedding(n, t, seed=d)
    h, s = O.hash_signs(n, t, d)
    assert np.array_equal(op.apply(a), O.apply_dense(h, s, t, a))


def test_nonfinite_and_shape_errors(rng):
    op = SparseEmbedding(10, 4, seed=0)
    a = rng.standard_normal((10, 3))
    for bad in (np.nan, np.inf, -np.inf):
        b = a.copy()
        b[7, 2] = bad
        with pytest.raises(ValueError):
            op.apply(b)
        with pytest.raises(ValueError):
            op.apply(torch.from_numpy(b.astype(np.float32)).cuda())
    with pytest.raises(ValueError):
        op.apply(rng.standard_normal((11, 2)))
    with pytest.raises(ValueError):
        SparseEmbedding(4, 0, seed=0)
    with pytest.raises(ValueError):
        SparseEmbedding(0, 4, seed=0)


# ---- the reference's own hot-path properties (test_sketch.py:37-84, 231-273)
def test_unit_vector_maps_to_signed_basis():
    op = make_sparse_embedding(5, 7, seed=3)
    for j in range(5):
        e = np.zeros((5, 1))
        e[j] = 1.0
        out = op.apply(e).ravel()
        assert np.count_nonzero(out) == 1 and out[op.bucket[j]] == op.sign[j]


def test_structure_zero_linearity_determinism(rng):
    op = make_sparse_embedding(9, 5, seed=1)
    dense = op.dense()
    assert all(np.count_nonzero(dense[:, j]) == 1 and abs(dense[:, j]).max() == 1.0 for j in range(9))
    assert np.all(make_sparse_embedding(4, 8, seed=0).apply(np.zeros((4, 1))) == 0)
    op = make_sparse_embedding(20, 9, seed=3)
    a, b = rng.standard_normal((20, 4)), rng.standard_normal((20, 4))
    assert np.abs(op.apply(a + b) - op.apply(a) - op.apply(b)).max() <= 1e-12
    x, y = (make_sparse_embedding(30, 10, seed=5) for _ in range(2))
    assert np.array_equal(x.bucket, y.bucket) and np.array_equal(x.sign, y.sign)
    dense = rng.standard_normal((30, 5)) * (rng.random((30, 5)) < 0.4)
    op = make_sparse_embedding(30, 11, seed=1)
    assert np.array_equal(op.apply(dense), op.apply(sp.csr_array(dense)))


def test_concurrent_apply_from_host_threads(rng):
    """The reference CLI fans apply() over a ThreadPoolExecutor (cli.py:227-231):
    concurrent calls on one operator give the same bits as serial ones."""
    from concurrent.futures import ThreadPoolExecutor

    n, t = 20_000, 500
    op = SparseEmbedding(n, t, seed=4)
    mats = [rng.standard_normal((n, 8)) for _ in range(6)]
    mats += [sp.csr_array(sp.random_array((n, 40), density=0.05, rng=rng, format="csr")) for _ in range(6)]
    serial = [op.apply(m) for m in mats]
    with ThreadPoolExecutor(4) as ex:
        par = list(ex.map(op.apply, mats))
    assert all(np.array_equal(x, y) for x, y in zip(serial, par))


def test_monte_carlo_unbiased():
    x = np.ones((4, 1))
    total = sum(float(np.sum(make_sparse_embedding(4, 8, seed=seed).apply(x) ** 2)) for seed in range(2000))
    assert 3.8 <= total / 2000 <= 4.2


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_apply_csr_wide_d(dtype, rng):
    """Config-5 shape (d too wide for on-chip accumulators): the deterministic
    wide kernel is bit-exact; fast mode (unordered atomics) is within rounding."""
    n, d, t = 6000, 60_000, 23
    a = sp.random_array((n, d), density=0.002, rng=rng, format="csr").tolil()
    for r in (3, 4, 2500):  # rows longer than one block pass (> 1024 stored entries)
        cols = np.sort(rng.choice(d, size=3000, replace=False))
        a[r, cols] = rng.standard_normal(3000)
    a = sp.csr_array(a, dtype=dtype)
    op = SparseEmbedding(n, t, seed=5)
    h, s = O.hash_signs(n, t, 5)
    ref = O.np_apply_csr(h, s, t, a)
    assert np.array_equal(op.apply(a), ref)
    got32 = op.apply(a, out_dtype=torch.float32)
    assert np.array_equal(got32, ref.astype(np.float32))
    fast = op.apply(a, deterministic=False)
    assert np.linalg.norm(fast - ref) <= 1e-12 * np.linalg.norm(ref)
    fast32 = op.apply(a, out_dtype=torch.float32, deterministic=False)
    assert np.linalg.norm(fast32 - ref) <= 1e-5 * np.linalg.norm(ref)
    # fast mode on a narrow matrix too
    b = sp.csr_array(sp.random_array((n, 40), density=0.2, rng=rng, format="csr"), dtype=dtype)
    ref_b = O.np_apply_csr(h, s, t, b)
    assert np.linalg.norm(op.apply(b, deterministic=False) - ref_b) <= 1e-12 * np.linalg.norm(ref_b)


# ---------------------------------------------------------------- column sketch
def test_apply_right_golden():
    z = load("apply_cases.npz")
    op = SparseEmbedding(60, 9, 13)
    assert np.array_equal(apply_right(z["right_dense_a"], op), z["right_dense_y"])
    ac = sp.csr_array((z["right_csr_data"], z["right_csr_indices"], z["right_csr_indptr"]), shape=(25, 60))
    assert np.array_equal(apply_right(ac, op), z["right_csr_y"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_apply_right_matches_transpose_formula(dtype, rng):
    n_cols, t = 3000, 150
    op = SparseEmbedding(n_cols, t, seed=8)
    h, s = O.hash_signs(n_cols, t, 8)
    a = rng.standard_normal((40, n_cols)).astype(dtype)
    ref = O.apply_dense(h, s, t, np.ascontiguousarray(a.T)).T
    assert np.array_equal(apply_right(a, op), ref)
    ac = sp.csr_array(sp.random_array((40, n_cols), density=0.05, rng=rng, format="csr"), dtype=dtype)
    ref2 = O.np_apply_csr(h, s, t, sp.csr_array(ac.T)).T
    assert np.array_equal(apply_right(ac, op), ref2)


# ---------------------------------------------------------------- K5
def test_lev_rownorms_golden():
    from paper_1207_6365_b200.solvers import lev_rownorms
    from tests import synth

    z = load("lev_case.npz")
    a, m, k, seed = synth.lev_case()
    got = lev_rownorms(a, z["probe"])
    assert np.max(np.abs(got - z["scores"]) / np.abs(z["scores"])) <= 1e-12
    a32 = sp.csr_array(a, dtype=np.float32)
    ref32 = O.lev_rownorms_csr(a32, z["probe"])
    got32 = lev_rownorms(a32, z["probe"], out_dtype=torch.float32)
    assert np.max(np.abs(got32 - ref32) / ref32) <= 1e-5
    gd = lev_rownorms(a.toarray(), z["probe"])
    assert np.max(np.abs(gd - z["scores"]) / np.abs(z["scores"])) <= 1e-12


@pytest.mark.parametrize("n,d,k,density", [(20_000, 64, 32, 0.26), (5_000, 16, 8, 0.5), (3_001, 100, 40, 0.1),
                                           (4_000, 256, 256, 0.05), (1_000, 8, 16, 1.0),
                                           (2_000, 200, 32, 0.5)])  # every row long
def test_lev_tensor_core_3xtf32(n, d, k, density, rng):
    """fp32 CSR runs on tcgen05 (3xTF32): scores within 1e-5 of the fp64 oracle."""
    from paper_1207_6365_b200.solvers import lev_rownorms

    a = sp.csr_array(sp.random_array((n, d), density=density, rng=rng, format="csr"), dtype=np.float32)
    a = a.tolil()
    a[5, :] = rng.standard_normal(d).astype(np.float32) * 10  # a dense row (long-row path)
    a = sp.csr_array(a, dtype=np.float32)
    probe = rng.standard_normal((d, k)) / np.sqrt(k)
    ref = O.lev_rownorms_csr(a, probe)
    got = lev_rownorms(a, probe)
    nz = ref > 0
    assert np.all(got[~nz] == 0)
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz]) <= 1e-5


@pytest.mark.parametrize("k", [32, 64, 128])
def test_lev_tensor_core_row_scaling_extremes(k, rng):
    """The scaled 2xFP16 kernel (lev_tc3.cuh, k % 32 == 0): rows spanning 1e-30 ..
    1e30, entries inside a row spanning 1e-6, empty rows, a 300-entry row, a
    partial last tile -- 1e-5 relative to the fp64 oracle."""
    from paper_1207_6365_b200.solvers import lev_rownorms

    n, d = 9_001, 300
    a = sp.random_array((n, d), density=0.05, rng=rng, format="csr").tolil()
    a[7, :] = rng.standard_normal(d)  # one full row (long-row path, > 80 entries)
    a[11, :] = 0  # empty row
    a = sp.csr_array(a)
    row_scale = 10.0 ** rng.uniform(-30, 30, n)
    a = sp.csr_array(sp.diags_array(row_scale) @ a, dtype=np.float32)
    a.data *= np.where(rng.random(a.nnz) < 0.1, 1e-6, 1.0).astype(np.float32)
    probe = rng.standard_normal((d, k)) * 1e3
    ref = O.lev_rownorms_csr(a, probe)
    got = lev_rownorms(a, probe)
    nz = ref > 0
    assert np.all(got[~nz] == 0)
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz]) <= 1e-5


@pytest.mark.parametrize("d,k", [(64, 32), (128, 32), (64, 40)])  # k=32: lev_tc3.cuh, k=40: lev_tc.cuh
def test_lev_tensor_core_noncanonical_rows(d, k, rng):
    """Duplicate and unsorted column indices are summed like scipy's a @ probe
    (the dirty-tile rebuild), on both tensor-core kernels."""
    from paper_1207_6365_b200.solvers import lev_rownorms

    n = 3_000
    counts = rng.integers(0, 40, size=n)
    indptr = np.concatenate([[0], np.cumsum(counts)])
    indices = np.concatenate([np.sort(rng.choice(d, size=c, replace=False)) for c in np.minimum(counts, d)])
    indices = indices.astype(np.int32)
    # every 7th row: duplicates (same column repeated); every 11th: reversed order
    for r in range(0, n, 7):
        b, e = indptr[r], indptr[r + 1]
        if e - b >= 3:
            indices[b + 1] = indices[b]
            indices[e - 1] = indices[b]
    for r in range(3, n, 11):
        b, e = indptr[r], indptr[r + 1]
        indices[b:e] = indices[b:e][::-1].copy()
    vals = rng.standard_normal(indptr[-1]).astype(np.float32)
    a = sp.csr_array((vals, indices, indptr), shape=(n, d))
    assert not a.has_canonical_format
    probe = rng.standard_normal((d, k)) / np.sqrt(k)
    ref = O.lev_rownorms_csr(a, probe)
    got = lev_rownorms(a, probe)
    nz = ref > 1e-12
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz]) <= 1e-5
    assert np.all(np.abs(got[~nz]) <= 1e-6)


_TC2_SCRIPT = r"""
import sys, numpy as np, scipy.sparse as sp
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_1207_6365_b200.solvers import lev_rownorms
rng = np.random.default_rng(7)
worst = 0.0
for n, d, k, dens in [(20000, 64, 32, 0.26), (3001, 100, 40, 0.1), (5000, 16, 8, 0.5), (2000, 128, 128, 0.3)]:
    a = sp.csr_array(sp.random_array((n, d), density=dens, rng=rng, format="csr"), dtype=np.float32).tolil()
    a[5, :] = rng.standard_normal(d).astype(np.float32) * 1e3   # long row, large scale
    a[9, :3] = np.float32(1e-30)                                # tiny row
    a = sp.csr_array(a, dtype=np.float32)
    p = rng.standard_normal((d, k)) / np.sqrt(k)
    ref = O.lev_rownorms_csr(a, p)
    got = lev_rownorms(a, p)
    nz = ref > 0
    assert np.all(got[~nz] == 0)
    worst = max(worst, float(np.max(np.abs(got[nz] - ref[nz]) / ref[nz])))
print(worst)
"""


def test_lev_staged_fp16_kernel():
    """The opt-in staged 2xFP16 kernel (SKT_LEV_TC2=1, lev_tc2.cuh), run in a
    child process (the selector is read once per process): 1e-5 vs the oracle,
    incl. per-row scaling extremes."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SKT_LEV_TC2="1")
    out = subprocess.run([sys.executable, "-c", _TC2_SCRIPT, root], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-5


def test_leverage_pipeline_matches_reference_pieces():
    from paper_1207_6365_b200.solvers import leverage_scores_sketched
    from tests import synth

    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["lev"]
    z = load("lev_case.npz")
    a, m, k, seed = synth.lev_case()
    run = leverage_scores_sketched(a, m, k, seed)
    assert sha(run.sa) == cfg["sha_sa"]  # GPU S.A bit-identical to the reference
    assert run.rank == cfg["rank"]
    # the probe comes from the host QR / inverse (LAPACK: last bits host-dependent)
    assert np.linalg.norm(run.probe - z["probe"]) <= 1e-12 * np.linalg.norm(z["probe"])
    assert np.max(np.abs(run.scores - z["scores"]) / np.abs(z["scores"])) <= 1e-12


def test_approx_leverage_scores_end_to_end():
    """leverage.py:50-97 mirror (GPU sketch + GPU contraction, host QR/SRHT/median)
    against the reference run on the same input (fp64: 1e-12)."""
    from paper_1207_6365_b200.solvers import approx_leverage_scores

    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["approx_lev"]
    z = load("approx_lev.npz")
    res = approx_leverage_scores(sp.csr_array(z["a"]), cfg["eps"], cfg["repetitions"], cfg["seed"])
    assert res.rank == cfg["rank"]
    ref = z["scores"]
    assert np.max(np.abs(res.scores - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-10
    res_d = approx_leverage_scores(z["a"], cfg["eps"], cfg["repetitions"], cfg["seed"])
    assert np.max(np.abs(res_d.scores - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-10
    with pytest.raises(ValueError):
        approx_leverage_scores(z["a"], 0.5, repetitions=2)


# ---------------------------------------------------------------- low-rank caller (config-5 shape)
def test_low_rank_approx_matches_reference():
    from paper_1207_6365_b200.lowrank import best_rank_k_error_gpu, low_rank_approx
    from tests import synth

    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["lowrank"]
    z = load("lowrank_case.npz")
    a, k, seed, t_r, t_s = synth.lowrank_case()
    r_op = SparseEmbedding(a.shape[1], t_r, cfg["r_op_seed"])
    s_op = SparseEmbedding(a.shape[0], t_s, cfg["s_op_seed"])
    res = low_rank_approx(a, k, cfg["eps"], seed=seed, r_op=r_op, s_op=s_op)
    # sketches are bit-exact; the small SVDs are LAPACK on the host -> 1e-9
    assert abs(res.err - cfg["err"]) <= 1e-9 * cfg["err"]
    assert abs(res.cond_su - cfg["cond_su"]) <= 1e-9 * cfg["cond_su"]
    assert np.max(np.abs(res.factors.d - z["d"])) <= 1e-9 * z["d"][0]
    for name in ("l", "w"):
        got, want = getattr(res.factors, name), z[name]
        sgn = np.sign(np.sum(got * want, axis=0))  # SVD column signs
        assert np.max(np.abs(got * sgn - want)) <= 1e-7
    # substitute oracle for Delta_k (randomized subspace iteration) vs the dense SVD
    dense = a.toarray()
    sig = np.linalg.svd(dense, compute_uv=False)
    delta = float(np.sqrt(np.sum(sig[k:] ** 2)))
    assert abs(best_rank_k_error_gpu(a, k) - delta) <= 1e-6 * delta
    assert res.err >= delta * (1 - 1e-9)


@pytest.mark.parametrize("n,d,k,density,itype", [
    (20_000, 64, 32, 0.26, np.int32),   # config 4's shape
    (3_001, 33, 16, 0.3, np.int64),     # d not a multiple of 4, int64 index arrays, partial last tile
    (1_000, 20, 32, 1.0, np.int32),     # every row full (d <= 32 tile)
    (2_500, 64, 32, 0.02, np.int32),    # many empty rows
])
def test_lev_fp64_tensor_core(n, d, k, density, itype, rng):
    """fp64 CSR values (the reference API's dtype, as_csr's upcast) run on the
    fp64 tensor cores (lev_dmma.cuh, DMMA.8x8x4): scores within 1e-12 relative
    of the fp64 oracle (leverage.py:90-91), incl. rows scaled 1e-150 .. 1e150
    and non-canonical rows (duplicates summed like scipy's a @ probe)."""
    from paper_1207_6365_b200.solvers import lev_rownorms

    a = sp.csr_array(sp.random_array((n, d), density=density, rng=rng, format="csr")).tolil()
    a[5, :] = rng.standard_normal(d) * 1e150
    a[9, :3] = 1e-150
    a = sp.csr_array(a)
    if n > 100:  # a duplicate column and an unsorted row
        a = sp.csr_array((a.data.copy(), a.indices.copy(), a.indptr.copy()), shape=a.shape)
        b, e = a.indptr[5], a.indptr[6]
        a.indices[b + 1] = a.indices[b]
        b, e = a.indptr[7], a.indptr[8]
        a.indices[b:e] = a.indices[b:e][::-1].copy()
    a = sp.csr_array((a.data, a.indices.astype(itype), a.indptr.astype(itype)), shape=a.shape)
    probe = rng.standard_normal((d, k)) / np.sqrt(k)
    ref = O.lev_rownorms_csr(a, probe)
    got = lev_rownorms(a, probe)
    nz = ref > 0
    assert np.all(got[~nz] == 0)
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz]) <= 1e-12
    got32 = lev_rownorms(a, probe, out_dtype=torch.float32)
    fin = nz & (ref < 1e38) & (ref > 1e-37)  # scores representable in fp32
    assert np.max(np.abs(got32[fin] - ref[fin]) / ref[fin]) <= 1e-6


def test_csr_check_sorted_device(rng):
    """skt_csr_check_sorted: the device form of scipy's has_canonical_format
    (strictly increasing columns per row), incl. empty rows, a duplicate at a
    row start, and int64 index arrays."""
    from paper_1207_6365_b200.sketch import csr_is_canonical_device

    for it in (np.int32, np.int64):
        a = sp.csr_array(sp.random_array((5_000, 300), density=0.05, rng=rng, format="csr"))
        ip, ix = (torch.from_numpy(x.astype(it)).cuda() for x in (a.indptr, a.indices))
        assert a.has_canonical_format and csr_is_canonical_device(ip, ix, a.shape[0])
        for r in (0, 1234, 4999):  # duplicate / unsorted pair inside one row
            b, e = a.indptr[r], a.indptr[r + 1]
            if e - b < 2:
                continue
            bad = a.indices.copy()
            bad[e - 1] = bad[e - 2]
            ixb = torch.from_numpy(bad.astype(it)).cuda()
            assert not csr_is_canonical_device(ip, ixb, a.shape[0])
        # a smaller column at a row start is canonical (different rows)
        z = sp.csr_array((np.ones(4), np.array([5, 7, 1, 2]), np.array([0, 2, 2, 4])), shape=(3, 9))
        ipz, ixz = (torch.from_numpy(x.astype(it)).cuda() for x in (z.indptr, z.indices))
        assert csr_is_canonical_device(ipz, ixz, 3)


@pytest.mark.parametrize("nbytes", [1, 1_600_004, 4_000_003, 4 << 20, (4 << 20) * 8 + 12345, (4 << 20) * 19 + 8,
                                    123_456_789, (1 << 20) + 4])
def test_memcpy_staged_round_trip(nbytes):
    """skt_memcpy_staged (page-locked ring for pageable host memory): both
    directions byte-exact for sizes below, at and across the 4 MB chunks and
    the 8-buffer ring."""
    host = np.frombuffer(np.random.default_rng(nbytes).bytes(nbytes), dtype=np.uint8).copy()
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().skt_memcpy_staged(dev.data_ptr(), host.ctypes.data, nbytes, 0, st))
    assert torch.equal(dev.cpu(), torch.from_numpy(host))
    back = np.zeros(nbytes, dtype=np.uint8)
    _lib.check(_lib.lib().skt_memcpy_staged(back.ctypes.data, dev.data_ptr(), nbytes, 1, st))
    assert np.array_equal(back, host)
