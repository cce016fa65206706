"""N > 1 path on CPU: world_size-2 gloo ranks run the row sharding and the
all-reduce of partial SA; the per-shard partial is computed by the oracle (the
GPU kernel's role), the result must equal the single-process reference SA to
1e-12 (reassociation across shards)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1207_6365_b200.distributed import ShardedSparseEmbedding, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_rows_cover_disjoint():
    for n in (1, 7, 100, 16_777_216):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def _worker(rank, world, port, n, t, d, seed, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        import scipy.sparse as sp

        rng = np.random.default_rng(123)
        h, s = O.hash_signs(n, t, seed)
        if kind == "dense":
            a = rng.standard_normal((n, d))
        else:
            a = sp.csr_array(sp.random_array((n, d), density=0.2, rng=rng, format="csr"))

        def partial(a_local, out_dtype, buckets=None, out=None, flag=None):
            r0, r1 = op.row_begin, op.row_end
            if isinstance(a_local, torch.Tensor):
                a_local = a_local.numpy()
            if flag is not None and kind == "dense" and not np.isfinite(a_local).all():
                flag.fill_(1)  # the kernel's fused non-finite scan
            if kind == "dense":
                p = O.apply_dense(h[r0:r1], s[r0:r1], t, a_local)
            else:
                p = O.apply_csr(h[r0:r1], s[r0:r1], t, a_local)
            p = torch.from_numpy(p).to(out_dtype)
            return p if buckets is None else p[buckets[0] : buckets[1]]

        op = ShardedSparseEmbedding(n, t, seed, partial_fn=partial)
        local = a[op.row_begin : op.row_end]
        out = op.apply(local).numpy()
        full = O.apply(h, s, t, a)
        if kind == "dense":  # pipelined exchange: bucket ranges reduced as they finish
            out_c = op.apply(torch.from_numpy(local), chunks=5).numpy()
            assert np.array_equal(out_c, out)
            assert op.bucket_chunks(5)[0][0] == 0 and op.bucket_chunks(5)[-1][1] == t
            # a NaN on rank 1 only: both ranks raise (as_dense, _validation.py:25-26)
            bad = torch.from_numpy(local.copy())
            if rank == 1:
                bad[7, 2] = float("nan")
            with pytest.raises(ValueError, match="non-finite"):
                op.apply(bad, chunks=3)
        if rank == 0:
            rel = np.linalg.norm(out - full) / max(np.linalg.norm(full), 1e-300)
            q.put((rel, op.row_begin, op.row_end))
        with pytest.raises(ValueError):
            op.apply(a[:1] if op.row_end - op.row_begin != 1 else a[:2])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_two_rank_gloo_allreduce_matches_reference(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, t, d, seed = 5_001, 97, 6, 3
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, t, d, seed, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    rel, r0, r1 = q.get(timeout=10)
    assert (r0, r1) == (0, 2500)
    assert rel <= 1e-12


def _bucket_worker(rank, world, port, n, t, d, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        import scipy.sparse as sp

        from paper_1207_6365_b200.distributed import BucketShardedSparseEmbedding

        rng = np.random.default_rng(321)
        h, s = O.hash_signs(n, t, seed)
        a = sp.csr_array(sp.random_array((n, d), density=0.05, rng=rng, format="csr"))

        def block(a_full, out_dtype, buckets):
            # the GPU kernel's role: SA rows [b0, b1) only, from the rows hashed there
            b0, b1 = buckets
            mine = np.flatnonzero((h >= b0) & (h < b1))
            part = O.apply_csr(h[mine] - b0, s[mine], b1 - b0, sp.csr_array(a_full)[mine])
            return torch.from_numpy(part).to(out_dtype)

        op = BucketShardedSparseEmbedding(n, t, seed, block_fn=block)
        blk = op.apply(a)
        full = op.gather(blk).numpy()
        ref = O.apply(h, s, t, a)
        if rank == 0:
            q.put((bool(np.array_equal(full, ref)), op.bucket_begin, op.bucket_end, blk.shape[0]))
        with pytest.raises(ValueError):
            op.apply(a[:10])
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_bucket_ownership_matches_reference():
    """Bucket-ownership sharding (config 5's multi-GPU layout): each rank's SA
    block covers its bucket range, computed from the rows hashed there; the
    all-gathered SA equals the single-process reference bit for bit (no
    reassociation: every bucket is summed on one rank, in ascending row order)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, t, d, seed = 4_001, 101, 300, 5
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, n, t, d, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    same, b0, b1, rows = q.get(timeout=10)
    assert (b0, b1, rows) == (0, 50, 50)
    assert same


# ---------------------------------------------------------------------------
# The same two-rank layouts with the REAL kernels: both gloo ranks run their
# shard operator (K1 with a row range, K2, K3/K4) on cuda:0; the collectives
# move the partials through gloo (CPU), so no rank ever waits on another's
# kernel.  This runs the sharded rejection offsets and bucket ranges
# multi-process on the B200.
# ---------------------------------------------------------------------------
def _gpu_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import scipy.sparse as sp

        from oracle import oracle as O
        from paper_1207_6365_b200.distributed import BucketShardedSparseEmbedding

        torch.cuda.set_device(0)
        res = {}
        # row shards, t with Lemire rejections (threshold 2^32 mod t != 0)
        n, t, d, seed = 60_001, 25_000, 20, 11
        rng = np.random.default_rng(9)
        a = rng.standard_normal((n, d))
        h, s = O.hash_signs(n, t, seed)
        op = ShardedSparseEmbedding(n, t, seed, device="cuda:0")
        r0, r1 = op.row_begin, op.row_end
        res["h_shard"] = bool(np.array_equal(op.local.bucket, h[r0:r1].astype(np.int64)))
        local = torch.from_numpy(a[r0:r1]).cuda()
        part = op.partial_fn(local, torch.float64)
        full = part.cpu()
        dist.all_reduce(full)
        ref = O.apply_dense(h, s, t, a)
        res["rel_dense"] = float(np.linalg.norm(full.numpy() - ref) / np.linalg.norm(ref))
        mine = O.apply_dense(h[r0:r1], s[r0:r1], t, a[r0:r1])
        res["partial_exact"] = bool(np.array_equal(part.cpu().numpy(), mine))
        # bucket ownership over CSR (config 5's layout), duplicate columns included
        c = sp.csr_array(sp.random_array((n, 300), density=0.02, rng=rng, format="csr"))
        cd = sp.csr_array((np.r_[c.data, 1.5], np.r_[c.indices, c.indices[c.indptr[4]]],
                           np.r_[c.indptr[:5], c.indptr[5:] + 1]), shape=c.shape)  # row 4 repeats a column
        bop = BucketShardedSparseEmbedding(n, t, seed, device="cuda:0")
        tc = torch.sparse_csr_tensor(torch.from_numpy(cd.indptr).long(), torch.from_numpy(cd.indices).long(),
                                     torch.from_numpy(cd.data), size=cd.shape)
        blk = bop.apply(tc)
        gathered = bop.gather(blk.cpu()).numpy()
        res["bucket_exact"] = bool(np.array_equal(gathered, O.apply_csr(h, s, t, cd)))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gloo_real_kernels_on_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = q.get(timeout=10)
    assert res["h_shard"] and res["partial_exact"] and res["bucket_exact"], res
    assert res["rel_dense"] <= 1e-12, res
