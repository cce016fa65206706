"""Rank-k approximation with the sketches on the GPU -- mirror of the
reference's ``low_rank_approx`` (lowrank.py:111-222): the default
"srht_compose" strategy (each sketch an SRHT composed with a sparse
embedding) and explicit sparse-embedding sketches ``r_op`` / ``s_op`` (BASELINE
config 5).

GPU: the column sketch Y = A R^T (transpose-free kernel, sketch.py:445-448,
then the SRHT of the small sketch), S U and S A (K3 / K4 + SRHT), and the
Gram-identity residual (one fused pass over A, csrc/lsq.cu).  Host: the thin
SVDs / truncations of the small sketched problems -- the reference's own
numpy calls, so the factors match to LAPACK rounding.  "leverage_sample"
(leverage-score row samplers, another sketch family) is delegated to the
reference package when it is importable."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from .sketch import ComposedSketch, apply_right, check_count, check_eps, default_sparse_dim
from .sketch import sparse_embedding_or_identity
from .solvers import as_matrix, srht_or_identity

RANK_REL_TOL = 1e-10
DENSE_RESIDUAL_LIMIT = 4_000_000  # lowrank.py:41
LOWRANK_TR_C, LOWRANK_V_C, LOWRANK_VP_C = 0.5, 1.0, 1.0  # _constants.py


@dataclass(frozen=True)
class LowRankFactors:
    l: np.ndarray
    d: np.ndarray
    w: np.ndarray
    k: int


@dataclass(frozen=True)
class LowRankResult:
    factors: LowRankFactors
    err: float
    cond_su: float
    t_r: int
    t_s: int
    strategy: str
    seed: int
    capped: bool = False


def _affine_dims(t_r: int, eps: float):
    y = t_r / eps
    v = max(t_r + 1, math.ceil(LOWRANK_V_C * y * y * max(1.0, math.log(y))))
    v_prime = max(t_r + 1, math.ceil(LOWRANK_VP_C * y * max(1.0, math.log(y)) ** 2))
    return v, min(v_prime, v)


def sketch_dims_lowrank(k: int, eps: float):
    """lowrank.py:68-75."""
    k = check_count(k, "k")
    eps = check_eps(eps)
    x = k / eps
    t_r = max(k + 1, math.ceil(LOWRANK_TR_C * x * max(1.0, math.log(x))))
    return (t_r,) + _affine_dims(t_r, eps)


def _thin_svd(a):
    u, s, vt = np.linalg.svd(np.asarray(a, dtype=np.float64), full_matrices=False)
    rank = 0 if s.size == 0 or s[0] == 0.0 else int(np.count_nonzero(s > RANK_REL_TOL * s[0]))
    return u, s, vt.T, rank


def _orthonormal_basis(a):
    u, _, _, rank = _thin_svd(a)
    return u[:, :rank]


def _condition_number(a) -> float:
    s = np.linalg.svd(np.asarray(a, dtype=np.float64), compute_uv=False)
    if s.size == 0 or s[0] == 0.0 or s[-1] <= RANK_REL_TOL * s[0]:
        return float("inf")
    return float(s[0] / s[-1])


def _truncate_rank_k(m, k: int):
    u, s, v, _ = _thin_svd(m)
    return (u[:, :k] * s[:k]) @ v[:, :k].T


def _pad_orthonormal(q: np.ndarray, k: int, seed: int) -> np.ndarray:
    n, have = q.shape
    if have >= k:
        return q[:, :k]
    rng = np.random.default_rng(seed)
    extra = rng.standard_normal((n, k - have))
    extra -= q @ (q.T @ extra)
    extra, _ = np.linalg.qr(extra)
    return np.hstack([q, extra[:, : k - have]])


def _frobenius_norm(a) -> float:
    if sp.issparse(a):
        return float(np.sqrt(np.sum(a.data**2)))
    return float(np.linalg.norm(a, "fro"))


def _residual_norm(a, l, d, w) -> float:
    """lowrank.py:100-108 (dense below 4M entries, Gram identity above).  The
    Gram branch's two passes over A (a @ (w d) with the row dot against L, and
    ||A||_F^2) are one fused GPU pass (skt_gram_cross_*, precond.gram_residual_sq)."""
    n, n_cols = a.shape
    if n * n_cols <= DENSE_RESIDUAL_LIMIT:
        dense = a.toarray() if sp.issparse(a) else a
        return float(np.linalg.norm(dense - (l * d) @ w.T, "fro"))
    from .precond import gram_residual_sq  # noqa: PLC0415

    cross, fro2 = gram_residual_sq(a, l, d, w)
    val = fro2 - 2.0 * cross + float(np.sum(d**2))
    return float(math.sqrt(max(val, 0.0)))


STRATEGIES = ("srht_compose", "leverage_sample")  # lowrank.py:39


def low_rank_approx(a, k: int, eps: float, seed: int = 0, strategy: str = "srht_compose",
                    t_r: int | None = None, r_op=None, s_op=None, **kw) -> LowRankResult:
    """lowrank.py:111-222.  The default strategy ("srht_compose": SRHT o sparse
    embedding for both sketches) and explicit sparse-embedding sketches run
    here with every sketch on the GPU; "leverage_sample" (leverage-score row
    samplers, another sketch family) raises -- this package never runs the
    reference's CPU code."""
    if strategy not in STRATEGIES:
        raise ValueError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
    if strategy != "srht_compose" and (r_op is None or s_op is None):
        # leverage-score row samplers are another sketch family (out
        # of scope); the reference's own low_rank_approx with shim.install()
        # runs that strategy with its sparse-embedding column sketch on the GPU
        raise ValueError(
            "low_rank_approx(strategy='leverage_sample') samples rows by leverage scores "
            "(outside this package); use 'srht_compose', pass r_op and s_op, or call "
            "sketchnla.lowrank.low_rank_approx after paper_1207_6365_b200.install()"
        )
    a = as_matrix(a)
    n, n_cols = a.shape
    k = check_count(k, "k")
    if k > min(n, n_cols):
        raise ValueError(f"k={k} out of range for shape {a.shape}")
    eps = check_eps(eps)
    dims_t_r, v, v_prime = sketch_dims_lowrank(k, eps)
    if t_r is None:
        t_r = dims_t_r
    else:
        t_r = check_count(t_r, "t_r")
        v, v_prime = _affine_dims(t_r, eps)

    def stream(j):
        return int(np.random.SeedSequence(int(seed), spawn_key=(7, j)).generate_state(1)[0])

    if r_op is None:  # srht_compose (lowrank.py:154-157)
        t_hat = min(max(2 * t_r, default_sparse_dim(k, eps)), n_cols)
        inner = sparse_embedding_or_identity(n_cols, t_hat, stream(1))
        r_op = ComposedSketch(srht_or_identity(inner.output_dim, t_r, stream(0)), inner)
    if s_op is None:  # srht_compose (lowrank.py:180-184)
        inner = sparse_embedding_or_identity(n, min(v, n), stream(3))
        s_op = ComposedSketch(srht_or_identity(inner.output_dim, v_prime, stream(2)), inner)

    # step 1: row-space sketch Y = A R^T on the GPU, orthonormal basis on the host
    y = apply_right(a, r_op)
    u = _orthonormal_basis(y)
    if u.shape[1] == 0:
        factors = LowRankFactors(l=_pad_orthonormal(np.zeros((n, 0)), k, stream(9)), d=np.zeros(k),
                                 w=_pad_orthonormal(np.zeros((n_cols, 0)), k, stream(10)), k=k)
        return LowRankResult(factors, _frobenius_norm(a), 1.0, t_r, 0, strategy, int(seed))
    # step 2: affine sketch of (U, A) on the GPU
    su = np.asarray(s_op.apply(u))
    sa = np.asarray(s_op.apply(a))
    t_s = s_op.output_dim
    cond_su = _condition_number(su)
    # steps 3-5 on the host (small)
    fu, fs, fv, frank = _thin_svd(su)
    ut_sa = fu[:, :frank].T @ sa
    x_hat = _truncate_rank_k(ut_sa, min(k, min(ut_sa.shape)))
    t_mat = (fv[:, :frank] / fs[:frank]) @ x_hat
    gu, gs, gv, grank = _thin_svd(t_mat)
    k_eff = min(k, grank)
    l = _pad_orthonormal(u @ gu[:, :k_eff], k, stream(9))
    w = _pad_orthonormal(gv[:, :k_eff], k, stream(10))
    d = np.zeros(k)
    d[:k_eff] = gs[:k_eff]
    err = _residual_norm(a, l, d, w)
    return LowRankResult(LowRankFactors(l=l, d=d, w=w, k=k), err, float(cond_su), t_r, t_s, strategy,
                         int(seed))


def best_rank_k_error_gpu(a, k: int, oversample: int = 20, power_iters: int = 10, seed: int = 0,
                          device=None) -> float:
    """Delta_k = ||A - [A]_k||_F for a large sparse A, by randomized subspace
    iteration on the GPU.  SUBSTITUTE for the reference's best_rank_k_error
    (lowrank.py:225-230), which densifies A (550 GB at config 5)."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    m = sp.csr_array(a, dtype=np.float64)
    A = torch.sparse_csr_tensor(torch.from_numpy(m.indptr.astype(np.int64)),
                                torch.from_numpy(m.indices.astype(np.int64)),
                                torch.from_numpy(m.data), size=m.shape).to(device)
    At = A.t().to_sparse_csr()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    q = torch.randn((m.shape[1], k + oversample), generator=g, device=device, dtype=torch.float64)
    y = A @ q
    q, _ = torch.linalg.qr(y)
    for _ in range(power_iters):
        z, _ = torch.linalg.qr(At @ q)
        q, _ = torch.linalg.qr(A @ z)
    b = (At @ q).t()  # (k+p) x n_cols = Q^T A
    sig = torch.linalg.svdvals(b)
    fro2 = float(np.sum(m.data**2))
    return float(math.sqrt(max(fro2 - float((sig[:k] ** 2).sum()), 0.0)))
