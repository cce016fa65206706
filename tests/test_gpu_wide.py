"""The wide-CSR kernels behind skt_apply_csr_wide (csrc/csr_fine.cuh, the
default; csrc/csr_partition.cuh and csrc/csr_colblock.cuh, opt-in) for CSR A
with SA rows too wide for on-chip accumulators (BASELINE config 5's shape):
bit-exact against the oracle (sketch.py:155-164: per output, ascending row
order from +0.0) on the edge cases of their design -- several column blocks and
a partial last one, buckets of more than 32 / 512 rows (several pieces, more
than 32 pieces), pieces too large for the shared-memory image, empty buckets
and empty rows,
rows with thousands of entries in one block, a column shared by every row of a
bucket (chains longer than 32 and lists over 2048 entries: the ordered
fallback), int64 index arrays, fp64 values, fp32 / fp64 output, bucket
ranges."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import oracle as O
from paper_1207_6365_b200 import SparseEmbedding

pytestmark = pytest.mark.gpu


def _dev(a, itype=None):
    parts = [np.ascontiguousarray(a.indptr), np.ascontiguousarray(a.indices), np.ascontiguousarray(a.data)]
    if itype is not None:
        parts[0], parts[1] = parts[0].astype(itype), parts[1].astype(itype)
    return tuple(torch.from_numpy(x).cuda() for x in parts)


def _random_csr(rng, n, d, per, dtype):
    rows = [np.sort(rng.choice(d, size=min(d, int(rng.integers(0, 2 * per + 1))), replace=False)) for _ in range(n)]
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows])
    indices = np.concatenate(rows).astype(np.int32) if indptr[-1] else np.zeros(0, np.int32)
    data = rng.standard_normal(indptr[-1]).astype(dtype)
    return sp.csr_array((data, indices, indptr), shape=(n, d))


def _check(op, a, t, seed, d, itype=None):
    h, s = O.hash_signs(a.shape[0], t, seed)
    ref = O.apply_csr(h, s, t, a)
    ip, ix, vv = _dev(a, itype)
    for out in (torch.float64, torch.float32):
        got = op._apply_csr_device(ip, ix, vv, d, out, canonical=True).cpu().numpy()
        want = ref if out == torch.float64 else ref.astype(np.float32)
        assert np.array_equal(got, want), (out, np.argwhere(got != want)[:5])
    return ref


@pytest.mark.parametrize("n,d,t,per,dtype", [
    (3_000, 70_001, 37, 60, np.float32),    # 9 super-steps, partial last one, several column blocks
    (2_500, 262_144, 5, 40, np.float64),    # config 5's width; buckets of ~500 rows, fp64 values
    (5_000, 30_000, 2, 20, np.float32),     # buckets of ~2500 rows: cursors in the workspace
    (300, 50_000, 250, 30, np.float32),     # many empty buckets
])
def test_colsweep_bit_exact(n, d, t, per, dtype):
    rng = np.random.default_rng(n + d + t)
    a = _random_csr(rng, n, d, per, dtype)
    _check(SparseEmbedding(n, t, 3), a, t, 3, d)


def test_colsweep_dense_runs_and_shared_columns():
    """Rows with thousands of entries inside one super-step (continuation loads
    of 16), and one column set shared by all rows (same-column adds of one
    bucket serialised in row order)."""
    rng = np.random.default_rng(1)
    n, d, t = 1_500, 40_000, 3
    a = _random_csr(rng, n, d, 10, np.float64).tolil()
    shared = np.sort(rng.choice(d, size=50, replace=False))
    for r in range(0, n, 3):
        a[r, shared] = rng.standard_normal(50)
    for r in (0, 7, 1499):
        a[r, 100:9000] = rng.standard_normal(8900)  # dense run across two super-steps
    a = sp.csr_array(a)
    a.sort_indices()
    _check(SparseEmbedding(n, t, 9), a, t, 9, d)


def test_fine_blocks_over_256_and_unstaged_piece():
    """More than 256 column blocks (d > 262,144) and an fp32 piece with more
    entries than the shared-memory image holds (placed directly in the
    workspace), next to ordinary pieces."""
    rng = np.random.default_rng(11)
    n, d, t = 1_200, 300_001, 3
    a = _random_csr(rng, n, d, 30, np.float32).tolil()
    for r in (5, 600):
        a[r, 1000:21_000] = rng.standard_normal(20_000).astype(np.float32)
    a = sp.csr_array(a)
    a.sort_indices()
    _check(SparseEmbedding(n, t, 13), a, t, 13, d)


def test_colsweep_int64_indices_and_empty_rows():
    rng = np.random.default_rng(2)
    n, d, t = 4_000, 33_000, 29
    a = _random_csr(rng, n, d, 3, np.float32)  # many empty rows (row length 0..6)
    _check(SparseEmbedding(n, t, 4), a, t, 4, d, itype=np.int64)


def test_colsweep_bucket_ranges():
    rng = np.random.default_rng(3)
    n, d, t = 2_000, 45_000, 41
    a = _random_csr(rng, n, d, 25, np.float32)
    op = SparseEmbedding(n, t, 5)
    ip, ix, vv = _dev(a)
    full = op._apply_csr_device(ip, ix, vv, d, torch.float32, canonical=True)
    pieced = torch.full_like(full, float("nan"))
    for b0, b1 in [(0, 1), (1, 17), (17, 40), (40, 41)]:
        op._apply_csr_device(ip, ix, vv, d, torch.float32, canonical=True, out=pieced, buckets=(b0, b1))
    assert torch.equal(pieced, full)


_COLSWEEP_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from tests.test_gpu_wide import _check, _random_csr
from paper_1207_6365_b200 import SparseEmbedding
for n, d, t, per in [(3000, 70001, 37, 60), (5000, 30000, 2, 20)]:
    rng = np.random.default_rng(n + d)
    a = _random_csr(rng, n, d, per, np.float32)
    _check(SparseEmbedding(n, t, 3), a, t, 3, d)
print("ok")
"""


@pytest.mark.parametrize("kernel", ["colblock", "partition"])
def test_wide_kernel_opt_in(kernel):
    """The opt-in wide paths (SKT_CSR_WIDE=colblock: csr_colblock.cuh, one
    kernel; SKT_CSR_WIDE=partition: csr_partition.cuh, 16384-column blocks; the
    default is the fine-block path, csr_fine.cuh),
    run in a child process (the selector is read once per process): bit-exact
    against the oracle."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SKT_CSR_WIDE=kernel)
    out = subprocess.run([sys.executable, "-c", _COLSWEEP_SCRIPT, root], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
