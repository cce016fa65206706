"""Seeded synthetic inputs with BASELINE.json's shapes and value distributions
(numpy default_rng; regenerated bit-identically on the GPU box from the seeds).

No public dataset is named by BASELINE.json; the paper's UF-collection corpus
is not in this container and is not recreated.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

SKETCH_SEED = 1  # SparseEmbedding(n, m, seed=1) as in BASELINE.md's CPU baseline


def csr_fixed_nnz(rng, n: int, d: int, per_row: int, dtype=np.float64, scale: float = 1.0):
    """n x d CSR with exactly `per_row` distinct uniform columns per row (sorted),
    values N(0, scale^2)."""
    cols = np.empty((n, per_row), dtype=np.int32)
    chunk = 1 << 17
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        keys = rng.random((r1 - r0, d))
        cols[r0:r1] = np.sort(np.argpartition(keys, per_row - 1, axis=1)[:, :per_row], axis=1)
    vals = (scale * rng.standard_normal(n * per_row)).astype(dtype)
    indptr = np.arange(0, (n + 1) * per_row, per_row, dtype=np.int64)
    if indptr[-1] < 2**31:
        indptr = indptr.astype(np.int32)
    return sp.csr_array((vals, cols.ravel(), indptr), shape=(n, d))


def matvec_fixed_order(a: np.ndarray, x: np.ndarray) -> np.ndarray:
    """A @ x with a fixed summation order (elementwise ufuncs, no BLAS), so the
    generated right-hand side is bit-identical on every host CPU."""
    acc = a[:, 0] * x[0, 0]
    for j in range(1, a.shape[1]):
        acc = acc + a[:, j] * x[j, 0]
    return acc.reshape(-1, 1)


def config1():
    """C1: dense fp64 100,000 x 20 ~ N(0,1); b = A x* + 0.1 N(0,1); m = 4,000."""
    rng = np.random.default_rng(101)
    a = rng.standard_normal((100_000, 20))
    x = rng.standard_normal((20, 1))
    b = matvec_fixed_order(a, x) + 0.1 * rng.standard_normal((100_000, 1))
    return a, b, SKETCH_SEED


def config2():
    """C2: CSR fp64 1e6 x 50, exactly 5 distinct uniform columns per row, N(0,1);
    b = A x* + 0.01 N(0,1); m = 25,000."""
    rng = np.random.default_rng(102)
    a = csr_fixed_nnz(rng, 1_000_000, 50, 5)
    x = rng.standard_normal((50, 1))
    b = np.asarray(a @ x) + 0.01 * rng.standard_normal((1_000_000, 1))
    return a, b, SKETCH_SEED


def lowrank_case():
    """Config-5 shaped low-rank case at oracle size: square CSR n = 3,000 with
    2% density, values (U V^T)_ij + 0.01 N(0,1), U, V ~ N(0,1)^{n x 5};
    k = 5, column sketch t_r = 20, row sketch t_s = 300."""
    rng = np.random.default_rng(105)
    n, r = 3_000, 5
    u = rng.standard_normal((n, r))
    v = rng.standard_normal((n, r))
    a = csr_fixed_nnz(rng, n, n, 60)
    rows = np.repeat(np.arange(n), 60)
    a.data = matvec_rows(u[rows], v[a.indices]) + 0.01 * rng.standard_normal(a.nnz)
    return a, r, 3, 20, 300


def matvec_rows(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Row-wise dot products with a fixed summation order (no BLAS)."""
    acc = x[:, 0] * y[:, 0]
    for j in range(1, x.shape[1]):
        acc = acc + x[:, j] * y[:, j]
    return acc


def lev_case():
    """Config-4 shaped leverage case, scaled to oracle size: CSR fp64 n=20,000,
    d=16, 6 random columns per row, 1% of rows fully dense with N(0, 100)
    values; sketch m = 2,000; JL probe k = 32."""
    rng = np.random.default_rng(104)
    n, d = 20_000, 16
    a = csr_fixed_nnz(rng, n, d, 6).tolil()
    dense_rows = rng.choice(n, size=n // 100, replace=False)
    for r in dense_rows:
        a[r, :] = 10.0 * rng.standard_normal(d)
    a = sp.csr_array(a)
    a.sort_indices()
    return a, 2_000, 32, 7


def csr_matvec_fixed_order(a: sp.csr_array, x: np.ndarray, per_row: int) -> np.ndarray:
    """A @ x for a CSR with exactly `per_row` entries per row, summed slot by
    slot with elementwise ufuncs (bit-identical on every host)."""
    v = a.data.reshape(-1, per_row) * x[a.indices, 0].reshape(-1, per_row)
    acc = v[:, 0]
    for j in range(1, per_row):
        acc = acc + v[:, j]
    return acc.reshape(-1, 1)


def precond_cases():
    """Inputs of the preconditioned-iteration cases (regress.py:159-283):
    name -> (A, b, eps0, seed).  Ill-conditioned columns (scaled 1 .. 1e3),
    a two-column right-hand side, a rank-deficient A, a CSR A."""
    rng = np.random.default_rng(41)
    n, d = 20_000, 12
    a = rng.standard_normal((n, d)) * (10.0 ** np.linspace(0.0, 3.0, d))
    x = rng.standard_normal((d, 1))
    b = matvec_fixed_order(a, x) + 0.01 * rng.standard_normal((n, 1))
    b2 = np.hstack([b, 0.5 * b + rng.standard_normal((n, 1))])
    a_def = a.copy()
    a_def[:, 5] = 2.0 * a_def[:, 2]
    s = csr_fixed_nnz(rng, 50_000, 20, 6)
    xs = rng.standard_normal((20, 1))
    bs = csr_matvec_fixed_order(s, xs, 6) + 0.01 * rng.standard_normal((50_000, 1))
    return {
        "dense": (a, b, 0.5, 3),
        "dense_2col": (a, b2, 0.5, 4),
        "rank_deficient": (a_def, b, 0.5, 5),
        "csr": (s, bs, 0.5, 6),
    }


def gram_cases():
    """Inputs of the rank-k Gram residual (lowrank.py:100-108) above the 4M
    entry limit: name -> A (CSR 3000 x 2000 at 1%, dense 2100 x 2000)."""
    rng = np.random.default_rng(43)
    s = sp.csr_array(sp.random_array((3000, 2000), density=0.01, rng=rng, format="csr"))
    dense = rng.standard_normal((2100, 2000))
    return {"csr": s, "dense": dense}


def nnls_cases():
    """Inputs of nonneg_regression (regress.py:330-370): name -> (A, b, eps, seed)."""
    rng = np.random.default_rng(47)
    n, d = 30_000, 8
    a = rng.standard_normal((n, d))
    x = np.array([[1.5], [-0.7], [0.3], [2.0], [-1.2], [0.0], [0.8], [-0.1]])
    b = matvec_fixed_order(a, x) + 0.05 * rng.standard_normal((n, 1))
    b2 = np.hstack([b, -b + 0.05 * rng.standard_normal((n, 1))])
    s = csr_fixed_nnz(rng, 40_000, 10, 5)
    xs = np.abs(rng.standard_normal((10, 1))) * np.where(np.arange(10) % 3 == 0, -1.0, 1.0)[:, None]
    bs = csr_matvec_fixed_order(s, xs, 5) + 0.05 * rng.standard_normal((40_000, 1))
    return {"dense": (a, b, 0.5, 7), "dense_2col": (a, b2, 0.5, 8), "csr": (s, bs, 0.5, 9)}


def lowrank_default_case():
    """A 3000 x 2500 CSR at 2% density sampled from a rank-5 product plus
    0.01 N(0,1) (config 5's construction, small): k = 5, eps = 0.5, seed = 11."""
    rng = np.random.default_rng(53)
    n, m, r = 3000, 2500, 5
    u = rng.standard_normal((n, r))
    v = rng.standard_normal((m, r))
    pat = sp.random_array((n, m), density=0.02, rng=rng, format="coo")
    vals = u[pat.row, 0] * v[pat.col, 0]
    for j in range(1, r):
        vals = vals + u[pat.row, j] * v[pat.col, j]
    vals = vals + 0.01 * rng.standard_normal(vals.size)
    return sp.csr_array((vals, (pat.row, pat.col)), shape=(n, m))
