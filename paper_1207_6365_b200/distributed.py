"""Row-sharded S.A across GPUs: one process per GPU.

S.A = sum_g S_g A_g over contiguous row shards [r_g, r_{g+1}).  Each rank
builds only its shard of the operator (K1 with a row range -- bit-exact h/s
for those rows, including the Lemire-rejection offset -- and K2 over the
shard), computes its partial m x d SA with K3/K4, and the partials are summed
with one NCCL all-reduce over NVLink.  Across shards the fp64 sum is
reassociated, so multi-GPU SA matches the reference to ~1e-16 relative
(tolerance 1e-12), not bit-for-bit; with one rank it is bit-identical.

The compute step is injectable (``partial_fn``) so the sharding and the
collective can be exercised on CPU with the gloo backend in tests.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced, disjoint row ranges covering [0, n)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    return rank * n // world, (rank + 1) * n // world


class ShardedSparseEmbedding:
    """SparseEmbedding(n, t, seed) whose rows are distributed over a process group."""

    family = "sparse"

    def __init__(self, n: int, t: int, seed: int, group=None, device=None, partial_fn=None):
        self.input_dim, self.output_dim, self.seed = int(n), int(t), int(seed)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.row_begin, self.row_end = shard_rows(self.input_dim, self.world, self.rank)
        self.local = None
        if partial_fn is None:
            from .sketch import SparseEmbedding

            self.local = SparseEmbedding(n, t, seed, device=device, row_range=(self.row_begin, self.row_end))
            partial_fn = self._gpu_partial
        self.partial_fn = partial_fn

    def _gpu_partial(self, a_local, out_dtype, buckets=None, out=None):
        if buckets is None:
            return self.local.apply(a_local, out_dtype=out_dtype)
        if out is None:
            out = torch.empty((self.output_dim, a_local.shape[1]), dtype=out_dtype, device=a_local.device)
        self.local._apply_dense_device(a_local, out_dtype, check_finite=False, out=out, buckets=buckets)
        return out[buckets[0] : buckets[1]]

    def bucket_chunks(self, chunks: int):
        """Contiguous bucket ranges of the pipelined apply."""
        t = self.output_dim
        chunks = max(1, min(int(chunks), t))
        return [(k * t // chunks, (k + 1) * t // chunks) for k in range(chunks)]

    def apply(self, a_local, out_dtype=torch.float64, async_op: bool = False, chunks: int = 1):
        """Full S.A on every rank from this rank's rows ``a_local``.

        ``chunks > 1`` (dense input) pipelines the exchange: SA is computed in
        contiguous bucket ranges and each range's all-reduce is issued
        asynchronously as soon as it is written, so NCCL traffic for range k
        overlaps the computation of range k+1."""
        if a_local.shape[0] != self.row_end - self.row_begin:
            raise ValueError(
                f"rank {self.rank} expects rows [{self.row_begin}, {self.row_end}), got {a_local.shape[0]} rows"
            )
        if chunks <= 1:
            part = self.partial_fn(a_local, out_dtype)
            work = dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group, async_op=async_op)
            return (part, work) if async_op else part
        device = a_local.device if isinstance(a_local, torch.Tensor) else torch.device("cpu")
        out = torch.empty((self.output_dim, a_local.shape[1]), dtype=out_dtype, device=device)
        works = []
        for b0, b1 in self.bucket_chunks(chunks):
            piece = self.partial_fn(a_local, out_dtype, buckets=(b0, b1), out=out)
            if piece.data_ptr() != out[b0:b1].data_ptr():
                out[b0:b1].copy_(piece)
            works.append(dist.all_reduce(out[b0:b1], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        if async_op:
            return out, works
        for w in works:
            w.wait()
        return out

    def descriptor(self) -> dict:
        return {"family": self.family, "n": self.input_dim, "t": self.output_dim, "seed": self.seed}


class BucketShardedSparseEmbedding:
    """Bucket-ownership sharding ("when row sharding is wrong"):
    every rank holds the whole operator and the whole input, rank g owns the
    contiguous bucket range [b_g, b_{g+1}) and computes only those SA rows,
    reading only the rows of A hashed there (the plan's bucket-range slice).
    There is no collective on the data path: SA stays row-block distributed
    (``gather()`` assembles it when a caller needs the full matrix).  This is
    the multi-GPU layout for config 5, whose m x d partial (419 MB) would
    dwarf each GPU's share of the input under row sharding.  Within a bucket
    the rows are still summed in ascending order, so every rank's block is
    bit-identical to the same rows of the single-GPU (and reference) SA.

    ``block_fn(a, out_dtype, (b0, b1)) -> (b1 - b0) x d`` is injectable so the
    partition and the gather run on CPU with gloo in tests."""

    family = "sparse"

    def __init__(self, n: int, t: int, seed: int, group=None, device=None, block_fn=None):
        self.input_dim, self.output_dim, self.seed = int(n), int(t), int(seed)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.bucket_begin, self.bucket_end = shard_rows(self.output_dim, self.world, self.rank)
        self.local = None
        if block_fn is None:
            from .sketch import SparseEmbedding

            self.local = SparseEmbedding(n, t, seed, device=device)
            block_fn = self._gpu_block
        self.block_fn = block_fn

    def _gpu_block(self, a, out_dtype, buckets, deterministic=True):
        b0, b1 = buckets
        op = self.local
        if isinstance(a, torch.Tensor) and a.layout == torch.sparse_csr:
            ip, ix, vv = (x.to(op.device) for x in (a.crow_indices(), a.col_indices(), a.values()))
            out = op._apply_csr_device(ip, ix, vv, a.shape[1], out_dtype, canonical=True,
                                       deterministic=deterministic, buckets=buckets)
        else:
            x = a.to(op.device)
            out = op._apply_dense_device(x, out_dtype, check_finite=True, buckets=buckets)
        return out[b0:b1]

    def apply(self, a, out_dtype=torch.float64, **kw):
        """This rank's SA rows [bucket_begin, bucket_end) from the full input."""
        if a.shape[0] != self.input_dim:
            raise ValueError(f"operator expects {self.input_dim} rows, got {a.shape[0]}")
        return self.block_fn(a, out_dtype, (self.bucket_begin, self.bucket_end), **kw)

    def gather(self, block):
        """All ranks' blocks -> the full t x d SA on every rank (all-gather)."""
        rows = [b1 - b0 for b0, b1 in (shard_rows(self.output_dim, self.world, r) for r in range(self.world))]
        mx = max(rows)  # equal-size exchange (blocks differ by at most one row)
        pad = torch.zeros((mx,) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
        pad[: block.shape[0]] = block
        parts = [torch.empty_like(pad) for _ in rows]
        dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:r] for p, r in zip(parts, rows)], 0)

    def descriptor(self) -> dict:
        return {"family": self.family, "n": self.input_dim, "t": self.output_dim, "seed": self.seed}
