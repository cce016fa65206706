"""Bucket-range S.A on the GPU (the building block of bucket-ownership
sharding, distributed.BucketShardedSparseEmbedding): SA rows [b0, b1) computed
alone equal the same rows of the full apply, bit for bit, for every CSR
kernel family (tile, lane, grouped sweep, wide row-sequential) and to
rounding for the atomic fast mode."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from paper_1207_6365_b200 import SparseEmbedding

pytestmark = pytest.mark.gpu


def _csr(rng, n, d, per_row, dtype):
    rows = []
    for _ in range(n):
        k = min(d, per_row if rng.random() > 0.02 else 4 * per_row)
        rows.append(np.sort(rng.choice(d, size=k, replace=False)))
    indptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    indices = np.concatenate(rows).astype(np.int32)
    vals = rng.standard_normal(len(indices)).astype(dtype)
    return sp.csr_array((vals, indices, indptr), shape=(n, d))


def _dev(a):
    return tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a.indptr, a.indices, a.data))


def _ranges(t):
    cuts = sorted({0, t, t // 7, t // 3 + 1, (2 * t) // 3})
    return [(a, b) for a, b in zip(cuts, cuts[1:]) if b > a]


@pytest.mark.parametrize("n,d,t,per,dtype,out", [
    (20_000, 64, 512, 16, np.float32, torch.float32),    # tile kernel
    (3_000, 300, 97, 12, np.float64, torch.float64),     # lane kernel (d > 256)
    (200_000, 8, 20_000, 3, np.float64, torch.float64),  # grouped sweep (short rows)
    (400, 60_000, 50, 40, np.float32, torch.float64),    # wide row-sequential
])
def test_csr_bucket_ranges_bit_exact(n, d, t, per, dtype, out):
    rng = np.random.default_rng(n + d)
    a = _csr(rng, n, d, per, dtype)
    op = SparseEmbedding(n, t, 7)
    ip, ix, vv = _dev(a)
    full = op._apply_csr_device(ip, ix, vv, d, out, canonical=True)
    pieced = torch.empty_like(full)
    for b0, b1 in _ranges(t):
        op._apply_csr_device(ip, ix, vv, d, out, canonical=True, out=pieced, buckets=(b0, b1))
    assert torch.equal(pieced, full)


def test_csr_bucket_ranges_fast_mode():
    rng = np.random.default_rng(5)
    n, d, t = 30_000, 2_000, 40
    a = _csr(rng, n, d, 30, np.float32)
    op = SparseEmbedding(n, t, 11)
    ip, ix, vv = _dev(a)
    full = op._apply_csr_device(ip, ix, vv, d, torch.float32, canonical=True, deterministic=False)
    pieced = torch.empty_like(full)
    for b0, b1 in _ranges(t):
        op._apply_csr_device(ip, ix, vv, d, torch.float32, canonical=True, deterministic=False, out=pieced,
                             buckets=(b0, b1))
    assert torch.allclose(pieced, full, rtol=1e-5, atol=1e-5)


def test_bucket_sharded_operator_single_rank_gpu():
    """BucketShardedSparseEmbedding's GPU block path on one rank (gloo group of
    one): the block is the whole SA and equals the plain operator's apply."""
    import torch.distributed as dist

    from paper_1207_6365_b200.distributed import BucketShardedSparseEmbedding

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(9)
        n, d, t = 5_000, 40, 128
        a = _csr(rng, n, d, 10, np.float64)
        op = BucketShardedSparseEmbedding(n, t, 3, device=torch.device("cuda", 0))
        at = torch.sparse_csr_tensor(*(torch.from_numpy(x) for x in (a.indptr, a.indices, a.data)), size=(n, d))
        blk = op.apply(at)
        ref = SparseEmbedding(n, t, 3).apply(a)
        assert np.array_equal(op.gather(blk).cpu().numpy(), ref)
        dense = torch.from_numpy(a.toarray()).cuda()
        assert np.array_equal(op.apply(dense).cpu().numpy(), SparseEmbedding(n, t, 3).apply(a.toarray()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_fused_exchange_emulated(world, dtype):
    """The fused exchange (K3 pushing partial rows into owner receive slots,
    owners summing their slots in rank order) with every rank's data on one
    GPU: equal to the rank-order sum of the shards' partials (bit for bit) and
    to the single-GPU SA within 1e-12."""
    import torch

    from paper_1207_6365_b200 import SparseEmbedding
    from paper_1207_6365_b200.distributed import fused_apply_emulated, shard_rows

    n, d, t, seed = 30_011, 128 if dtype == np.float32 else 64, 1001, 5
    a = torch.from_numpy(np.random.default_rng(world).standard_normal((n, d)).astype(dtype)).cuda()
    ops, shards = [], []
    for g in range(world):
        r0, r1 = shard_rows(n, world, g)
        ops.append(SparseEmbedding(n, t, seed, row_range=(r0, r1)))
        shards.append(a[r0:r1].contiguous())
    for out_dtype in (torch.float64, torch.float32):
        got = fused_apply_emulated(ops, shards, out_dtype)
        parts = [op.apply(x, out_dtype=out_dtype).double() for op, x in zip(ops, shards)]
        ref = parts[0].clone()
        for p in parts[1:]:
            ref += p
        assert torch.equal(got, ref.to(out_dtype))
    full = SparseEmbedding(n, t, seed).apply(a)
    got = fused_apply_emulated(ops, shards, torch.float64)
    assert float((got - full).norm() / full.norm()) <= 1e-12
