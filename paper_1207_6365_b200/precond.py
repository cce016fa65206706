"""Randomized preconditioning and the preconditioned iterations -- mirrors of
the reference's ``precondition``, ``richardson_solve`` and ``cgnr_solve``
(regress.py:159-283) with every pass over the data on the GPU.

* ``precondition``: the sparse embedding S.A (K1-K4) and the SRHT of the
  sketch (csrc/srht.cu) on the GPU -- both bit-identical to the reference --
  then the two pivoted QRs of the small sketches on the host with the
  reference's own LAPACK calls, so ``r_inv`` is identical.
* ``_iterate``: M = A R formed on the device by the library's own products
  (``skt_gemm_dense`` for dense A, ``skt_spmm_csr`` for CSR), then each iteration is one or two
  fused passes over M (csrc/lsq.cu): Richardson needs one
  (``skt_lsq_residual_grad``: the residual of the current iterate that
  ``_iterate`` records and M^T (b - M y) for the next step, where the
  reference makes three products), CGNR two (``skt_lsq_matvec_norm`` for
  M p and its norm, ``skt_lsq_update_grad`` for r - alpha M p, M^T r and the
  residual of the new iterate).  The r-sized vector algebra and the stopping
  rule run on the host exactly as in the reference; the residual on the
  original data is the fused GPU pass of ``residual_fro``.

The iterates agree with the reference to fp64 rounding (different summation
order in the products), so iteration counts and histories match on
non-degenerate problems (tests/test_gpu_precond.py, golden vectors from the
reference).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from ._lib import check
from .sketch import _ITYPE, _TORCH_TO_SKT, _ptr, _stream_ptr, check_eps, default_sparse_dim
from .sketch import sparse_embedding_or_identity
from .solvers import (  # noqa: F401  (SolverError re-exported)
    RegressionSolution,
    SolverError,
    _seed_stream,
    as_dense,
    as_matrix,
    default_srht_dim,
    pivoted_qr_rank,
    residual_fro,
    srht_apply,
)


@dataclass(frozen=True)
class Preconditioner:
    """regress.py:67-73."""

    r_inv: np.ndarray  # d x rank
    eps0: float
    seed: int
    rank: int
    sketch_dim: int


def precondition(a, eps0: float, seed: int = 0) -> Preconditioner:
    """regress.py:159-189: R with kappa(A R) <= (1 + eps0) / (1 - eps0)."""
    a = as_matrix(a)
    if not (0.0 < eps0 <= 0.5):
        raise ValueError(f"eps0 must be in (0, 0.5], got {eps0}")
    n, d = a.shape
    t1 = default_sparse_dim(d, eps0 / 2)
    s = sparse_embedding_or_identity(n, t1, _seed_stream(seed, 0))
    sa = np.asarray(s.apply(a), dtype=np.float64)
    _, _, _, rank = pivoted_qr_rank(sa)
    if rank == 0:
        raise ValueError("cannot precondition a zero matrix")
    rows = sa.shape[0]
    t2 = default_srht_dim(rank, eps0 / 2, rows)
    if t2 >= rows:  # srht_or_identity (sketch.py:429-433)
        sketched, sketch_dim = sa.copy(), rows
    else:
        sketched, sketch_dim = srht_apply(sa, t2, _seed_stream(seed, 1)), t2
    _, r_mat, perm, rank2 = pivoted_qr_rank(sketched)
    r11_inv = np.linalg.inv(r_mat[:rank2, :rank2])
    r_inv = np.zeros((d, rank2))
    r_inv[perm[:rank2]] = r11_inv
    return Preconditioner(r_inv=r_inv, eps0=eps0, seed=int(seed), rank=rank2, sketch_dim=sketch_dim)


# ---------------------------------------------------------------- GPU passes
class _Passes:
    """M = A R on the device and the fused passes over it (one b column at a time)."""

    def __init__(self, a, r_inv: np.ndarray, b: np.ndarray, device):
        self.dev = device
        self.L = _lib.lib()
        n, d = a.shape
        rank = r_inv.shape[1]
        self.n, self.r = n, rank
        r_dev = torch.from_numpy(np.ascontiguousarray(r_inv, dtype=np.float64)).to(device)
        with torch.cuda.device(device):
            self.stream = _stream_ptr(device)
            if sp.issparse(a):
                ip, ix, vv = (torch.from_numpy(np.ascontiguousarray(t)).to(device) for t in (a.indptr, a.indices, a.data))
                self.m = torch.empty((n, rank), dtype=torch.float64, device=device)
                check(self.L.skt_spmm_csr(n, d, _ptr(ip), _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype], _ptr(vv),
                                          _TORCH_TO_SKT[vv.dtype], vv.numel(), _ptr(r_dev), rank, _ptr(self.m),
                                          max(rank, 1), self.stream))
            else:
                ad = torch.from_numpy(np.ascontiguousarray(a)).to(device)
                self.m = torch.empty((n, rank), dtype=torch.float64, device=device)
                check(self.L.skt_gemm_dense(n, d, _ptr(ad), _TORCH_TO_SKT[ad.dtype], max(ad.stride(0), d, 1),
                                            _ptr(r_dev), rank, _ptr(self.m), max(rank, 1), self.stream))
            self.m = self.m.contiguous()
        self.b = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).to(device)  # n x cols
        nb = ctypes.c_size_t()
        check(self.L.skt_lsq_workspace(rank, ctypes.byref(nb)))
        self.ws = torch.empty(nb.value, dtype=torch.uint8, device=device)
        self.out = torch.empty(rank + 2, dtype=torch.float64, device=device)

    def _col(self, t: torch.Tensor, c: int) -> int:
        return _ptr(t) + 8 * c  # column c of a row-major n x cols tensor (ld = cols)

    def residual_grad(self, y: np.ndarray, want_grad: bool = True):
        """sum_c ||b_c - M y_c||^2 and M^T (b - M y) (rank x cols)."""
        cols = self.b.shape[1]
        g = np.zeros((self.r, cols))
        res2 = 0.0
        with torch.cuda.device(self.dev):
            for c in range(cols):
                yc = torch.from_numpy(np.ascontiguousarray(y[:, c])).to(self.dev)
                check(self.L.skt_lsq_residual_grad(self.n, self.r, _ptr(self.m), max(self.r, 1), _ptr(yc),
                                                   self._col(self.b, c), cols, _ptr(self.out) if want_grad else None,
                                                   _ptr(self.out) + 8 * (self.r + 1), _ptr(self.ws),
                                                   self.ws.numel(), self.stream))
                o = self.out.cpu().numpy()
                if want_grad:
                    g[:, c] = o[: self.r]
                res2 += float(o[self.r + 1])
        return res2, g

    def matvec_norm(self, p: np.ndarray):
        """q = M p (kept on the device, n x cols) and ||q_c||^2 per column."""
        cols = p.shape[1]
        q = torch.empty((self.n, cols), dtype=torch.float64, device=self.dev)
        qq = np.zeros(cols)
        with torch.cuda.device(self.dev):
            for c in range(cols):
                pc = torch.from_numpy(np.ascontiguousarray(p[:, c])).to(self.dev)
                check(self.L.skt_lsq_matvec_norm(self.n, self.r, _ptr(self.m), max(self.r, 1), _ptr(pc),
                                                 self._col(q, c), cols, _ptr(self.out), _ptr(self.ws),
                                                 self.ws.numel(), self.stream))
                qq[c] = float(self.out[0].item())
        return q, qq

    def update_grad(self, q: torch.Tensor, alpha: np.ndarray, rvec: torch.Tensor, y: np.ndarray):
        """rvec <- rvec - q alpha (in place), z = M^T rvec, sum_c ||M y_c - b_c||^2."""
        cols = rvec.shape[1]
        z = np.zeros((self.r, cols))
        res2 = 0.0
        with torch.cuda.device(self.dev):
            for c in range(cols):
                yc = torch.from_numpy(np.ascontiguousarray(y[:, c])).to(self.dev)
                check(self.L.skt_lsq_update_grad(self.n, self.r, _ptr(self.m), max(self.r, 1), self._col(q, c), cols,
                                                 float(alpha[c]), self._col(rvec, c), cols, _ptr(yc),
                                                 self._col(self.b, c), cols, _ptr(self.out),
                                                 _ptr(self.out) + 8 * (self.r + 1), _ptr(self.ws), self.ws.numel(),
                                                 self.stream))
                o = self.out.cpu().numpy()
                z[:, c] = o[: self.r]
                res2 += float(o[self.r + 1])
        return res2, z


def _richardson_steps(passes: _Passes):
    """regress.py:237-241: y <- y + M^T (b - M y); yields (y, ||M y - b||_F)."""
    cols = passes.b.shape[1]
    y = np.zeros((passes.r, cols))
    _, g = passes.residual_grad(y)
    while True:
        y = y + g
        res2, g = passes.residual_grad(y)  # residual of y, and the next step
        yield y, math.sqrt(res2)


def _cgnr_steps(passes: _Passes):
    """regress.py:267-283 (CG on the normal equations of M)."""
    cols = passes.b.shape[1]
    y = np.zeros((passes.r, cols))
    rvec = passes.b.clone()  # r = b - M 0
    _, z = passes.residual_grad(y)  # z = M^T r
    p = z.copy()
    zz = np.einsum("ij,ij->j", z, z)
    while True:
        q, denom = passes.matvec_norm(p)
        alpha = np.where(denom > 0, zz / np.maximum(denom, 1e-300), 0.0)
        y = y + p * alpha
        res2, z = passes.update_grad(q, alpha, rvec, y)
        zz_new = np.einsum("ij,ij->j", z, z)
        beta = np.where(zz > 0, zz_new / np.maximum(zz, 1e-300), 0.0)
        p = z + p * beta
        zz = zz_new
        yield y, math.sqrt(res2)


def _iterate(a, pre: Preconditioner, b, eps: float, max_iter: int, steps, method: str,
             device=None) -> RegressionSolution:
    """regress.py:192-234: iterate in preconditioned coordinates, map back."""
    a = as_matrix(a)
    b = as_dense(b)
    if a.shape[0] != b.shape[0]:
        raise ValueError(f"operands must have the same number of rows: {a.shape[0]} vs {b.shape[0]}")
    eps = check_eps(eps)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    passes = _Passes(a, pre.r_inv, b, device)
    y = np.zeros((pre.rank, b.shape[1]))
    res = float(np.linalg.norm(b, "fro"))
    history = [res]
    floor = 1e-14 * max(res, 1.0)
    grew = 0
    iterations = 0
    for y, new_res in steps(passes):
        iterations += 1
        history.append(new_res)
        if new_res > floor and new_res > history[-2] * (1 + 1e-9):
            grew += 1
            if grew >= 2:
                raise SolverError(
                    f"{method} diverged: residual grew twice in a row; "
                    "the preconditioner did not capture the column space",
                    best=pre.r_inv @ y,
                )
        else:
            grew = 0
        if new_res <= floor:
            break
        if history[-2] > 0 and abs(new_res - history[-2]) <= (eps / 10) * history[-2]:
            break
        if iterations >= max_iter:
            break
    x = pre.r_inv @ y
    return RegressionSolution(
        x=x,
        residual_norm=residual_fro(a, x, b, device),
        method=method,
        sketch_dim=pre.sketch_dim,
        seed=pre.seed,
        iterations=iterations,
        residual_history=tuple(history),
    )


def richardson_solve(a, pre: Preconditioner, b, eps: float, max_iter: int = 100) -> RegressionSolution:
    """regress.py:226-243."""
    return _iterate(a, pre, b, eps, max_iter, _richardson_steps, "richardson")


def cgnr_solve(a, pre: Preconditioner, b, eps: float, max_iter: int = 100) -> RegressionSolution:
    """regress.py:246-285."""
    return _iterate(a, pre, b, eps, max_iter, _cgnr_steps, "cgnr")


# ---------------------------------------------------------------- rank-k residual
def gram_residual_sq(a, l: np.ndarray, d: np.ndarray, w: np.ndarray, device=None):
    """(cross, ||A||_F^2) of the Gram identity (lowrank.py:104-107) in one fused
    pass over A on the GPU: cross = sum_i <A_i (W diag d), L_i>."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    L = _lib.lib()
    n, ncols = a.shape
    k = l.shape[1]
    mw = torch.from_numpy(np.ascontiguousarray(w * d, dtype=np.float64)).to(device)
    lt = torch.from_numpy(np.ascontiguousarray(l, dtype=np.float64)).to(device)
    nb = ctypes.c_size_t()
    check(L.skt_lsq_workspace(0, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=device)
    out = torch.zeros(2, dtype=torch.float64, device=device)
    with torch.cuda.device(device):
        stream = _stream_ptr(device)
        if sp.issparse(a):
            m = sp.csr_array(a)
            ip, ix, vv = (torch.from_numpy(np.ascontiguousarray(t)).to(device) for t in (m.indptr, m.indices, m.data))
            if vv.dtype not in _TORCH_TO_SKT:
                vv = vv.to(torch.float64)
            check(L.skt_gram_cross_csr(n, ncols, _ptr(ip), _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype], _ptr(vv),
                                       _TORCH_TO_SKT[vv.dtype], _ptr(mw), k, k, _ptr(lt), k, _ptr(out), _ptr(ws),
                                       nb.value, stream))
        else:
            at = torch.from_numpy(np.ascontiguousarray(a)).to(device)
            if at.dtype not in _TORCH_TO_SKT:
                at = at.to(torch.float64)
            check(L.skt_gram_cross_dense(n, ncols, _ptr(at), _TORCH_TO_SKT[at.dtype], max(ncols, 1), _ptr(mw), k,
                                         k, _ptr(lt), k, _ptr(out), _ptr(ws), nb.value, stream))
        o = out.cpu().numpy()
    return float(o[0]), float(o[1])
