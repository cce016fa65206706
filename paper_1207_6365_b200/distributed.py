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

import ctypes

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

    def _gpu_partial(self, a_local, out_dtype, buckets=None, out=None, flag=None):
        if buckets is None:
            return self.local.apply(a_local, out_dtype=out_dtype)
        if out is None:
            out = torch.empty((self.output_dim, a_local.shape[1]), dtype=out_dtype, device=a_local.device)
        # the fused non-finite scan lands in ``flag`` (no host sync inside the
        # pipeline); apply() checks every range's flag once at the end
        self.local._apply_dense_device(a_local, out_dtype, out=out, buckets=buckets, flag=flag)
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
        ranges = self.bucket_chunks(chunks)
        flags = torch.zeros(len(ranges), dtype=torch.int32, device=device)
        works = []
        for k, (b0, b1) in enumerate(ranges):
            piece = self.partial_fn(a_local, out_dtype, buckets=(b0, b1), out=out, flag=flags[k:k + 1])
            if piece.data_ptr() != out[b0:b1].data_ptr():
                out[b0:b1].copy_(piece)
            works.append(dist.all_reduce(out[b0:b1], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        # non-finite input on any rank raises on every rank (as_dense,
        # _validation.py:25-26), checked once after the pipeline is issued
        bad = flags.amax().reshape(1)
        works.append(dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=self.group, async_op=True))
        if async_op:
            return out, works
        for w in works:
            w.wait()
        if int(bad.item()) != 0:
            raise ValueError("matrix contains non-finite entries")
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

    def _gpu_block(self, a, out_dtype, buckets, deterministic=True, canonical=False):
        """``canonical=True`` asserts that no row of a sparse CSR ``a`` repeats
        a column (as_csr output, _validation.py:30-41) and unlocks the faster
        canonical kernels; torch CSR tensors carry no such guarantee, so the
        default serialises duplicates like SparseEmbedding.apply does."""
        b0, b1 = buckets
        op = self.local
        if isinstance(a, torch.Tensor) and a.layout == torch.sparse_csr:
            ip, ix, vv = (x.to(op.device) for x in (a.crow_indices(), a.col_indices(), a.values()))
            out = op._apply_csr_device(ip, ix, vv, a.shape[1], out_dtype, canonical=canonical,
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


# ---------------------------------------------------------------------------
# Fused exchange: K3 pushes partial rows into the owner ranks' receive buffers
# ---------------------------------------------------------------------------
def owner_bounds(t: int, world: int) -> list[int]:
    """Owner g of the fused exchange holds buckets [b_g, b_{g+1})."""
    return [g * t // world for g in range(world + 1)]


def _push(op, a_local, out_dtype, peers, bounds, me, cap, ldr, flag=None):
    """skt_apply_dense_push for one rank's shard operator ``op``; the fused
    non-finite scan lands in ``flag`` (1-element int32 device tensor)."""
    from . import _lib
    from .sketch import _TORCH_TO_SKT, _ptr, _stream_ptr, dense_operand

    a_local = dense_operand(a_local)
    n, d = a_local.shape
    P = ctypes.c_void_p * len(peers)
    B = ctypes.c_int64 * len(bounds)
    with torch.cuda.device(a_local.device):
        _lib.check(_lib.lib().skt_apply_dense_push(
            _ptr(op.plan_indptr), _ptr(op.plan_rows), op.output_dim, n, _ptr(a_local), _TORCH_TO_SKT[a_local.dtype],
            d, max(a_local.stride(0), d, 1) if n > 1 else max(d, 1), _TORCH_TO_SKT[out_dtype], P(*peers),
            B(*bounds), len(peers), me, cap, ldr, 0, _ptr(flag), _stream_ptr(a_local.device)))


def _slot_sum(recv, nslots, rows, d, cap, out):
    from . import _lib
    from .sketch import _TORCH_TO_SKT, _ptr, _stream_ptr

    with torch.cuda.device(recv.device):
        _lib.check(_lib.lib().skt_slot_sum(_ptr(recv), _TORCH_TO_SKT[recv.dtype], nslots, rows, d, cap * d, d,
                                           _ptr(out), d, _stream_ptr(recv.device)))


def fused_apply_emulated(ops, a_shards, out_dtype=torch.float64):
    """The fused exchange with all ranks' data on ONE device (the way to test
    it with one GPU: the ranks never wait on one another -- every push lands in
    a local buffer, then every owner sums its slots): returns the full t x d SA.
    ``ops[g]`` is rank g's shard operator, ``a_shards[g]`` its rows."""
    world = len(ops)
    t, d = ops[0].output_dim, a_shards[0].shape[1]
    bounds = owner_bounds(t, world)
    cap = max(bounds[g + 1] - bounds[g] for g in range(world))
    dev = a_shards[0].device
    recv = [torch.zeros((world * cap, d), dtype=out_dtype, device=dev) for _ in range(world)]
    peers = [r.data_ptr() for r in recv]
    for g, (op, a) in enumerate(zip(ops, a_shards)):
        _push(op, a, out_dtype, peers, bounds, g, cap, d)
    out = torch.empty((t, d), dtype=out_dtype, device=dev)
    for g in range(world):
        rows = bounds[g + 1] - bounds[g]
        if rows:
            _slot_sum(recv[g], world, rows, d, cap, out[bounds[g]:bounds[g + 1]])
    return out


class FusedShardedSparseEmbedding(ShardedSparseEmbedding):
    """Row-sharded S.A whose exchange is fused into K3: each rank's kernel
    stores its partial bucket rows straight into the owner rank's receive
    buffer over NVLink (torch symmetric memory: every rank maps every other
    rank's buffer), so the transfer overlaps the compute of the remaining
    buckets; after a cross-rank barrier each owner sums its N slots in rank
    order (deterministic) and the SA row blocks are all-gathered (NCCL).
    Dense input with rows the gather4 kernel takes (512 B .. 2 KB).  The data
    path is tested on one GPU by fused_apply_emulated; the symmetric-memory
    plumbing needs >= 2 GPUs (bench.py --fused)."""

    def __init__(self, n, t, seed, group=None, device=None):
        super().__init__(n, t, seed, group=group, device=device)
        self.bounds = owner_bounds(self.output_dim, self.world)
        self.cap = max(self.bounds[g + 1] - self.bounds[g] for g in range(self.world))
        self._bufs = {}

    def _buffers(self, d, dtype, device):
        key = (d, dtype)
        if key not in self._bufs:
            import torch.distributed._symmetric_memory as symm_mem

            recv = symm_mem.empty((self.world * self.cap, d), dtype=dtype, device=device)
            hdl = symm_mem.rendezvous(recv, group=self.group if self.group is not None else dist.group.WORLD)
            peers = [hdl.get_buffer(g, (self.world * self.cap, d), dtype).data_ptr() for g in range(self.world)]
            self._bufs[key] = (recv, hdl, peers)
        return self._bufs[key]

    def apply(self, a_local, out_dtype=torch.float64, async_op: bool = False, chunks: int = 1,
              check_finite: bool = True):
        """Same contract as ShardedSparseEmbedding.apply: ``a_local`` holds this
        rank's rows, non-finite input on any rank raises ValueError on every
        rank (after the exchange, one flag all-reduce)."""
        if not isinstance(a_local, torch.Tensor) or not a_local.is_cuda:
            raise ValueError("the fused exchange takes this rank's rows as a CUDA tensor")
        if a_local.shape[0] != self.row_end - self.row_begin:
            raise ValueError(
                f"rank {self.rank} expects rows [{self.row_begin}, {self.row_end}), got {a_local.shape[0]} rows"
            )
        from .sketch import dense_operand

        a_local = dense_operand(a_local)
        d = a_local.shape[1]
        recv, hdl, peers = self._buffers(d, out_dtype, a_local.device)
        flag = torch.zeros(1, dtype=torch.int32, device=a_local.device) if check_finite else None
        hdl.barrier()  # every owner has summed the previous apply's slots
        _push(self.local, a_local, out_dtype, peers, self.bounds, self.rank, self.cap, d, flag)
        hdl.barrier()  # every rank's pushes have landed
        block = torch.empty((self.cap, d), dtype=out_dtype, device=a_local.device)
        mine = self.bounds[self.rank + 1] - self.bounds[self.rank]
        if mine:
            _slot_sum(recv, self.world, mine, d, self.cap, block[:mine])
        gathered = torch.empty((self.world * self.cap, d), dtype=out_dtype, device=a_local.device)
        dist.all_gather_into_tensor(gathered, block, group=self.group)
        out = torch.cat([gathered[g * self.cap: g * self.cap + self.bounds[g + 1] - self.bounds[g]]
                         for g in range(self.world)])
        if flag is not None:
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
            if int(flag.item()) != 0:
                raise ValueError("matrix contains non-finite entries")
        return out
