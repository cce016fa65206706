"""Callers of the hot path, mirroring the reference's entry points.

* ``sketch_solve_ls``  -- regress.py:85-116: two GPU sketch applies (A, b), the
  thin SVD-pseudoinverse solve of (SA, Sb) on the host (linalg.py:75-90, the
  reference's own LAPACK path, so x is bit-identical when SA is), and the
  residual on the original data recomputed on the GPU.
* ``lev_rownorms``     -- leverage.py:90-91 fused on the GPU (K5).
* ``leverage_scores_sketched`` -- the config-4 pipeline of leverage.py:74-91
  with an explicit sketch size and probe width: S.A (GPU) -> pivoted QR /
  basis change (host, leverage.py:36-47) -> probe = N G^T -> scores (GPU).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import torch

from . import _constants as _C
from . import _lib
from ._lib import check
from .sketch import (
    ComposedSketch,
    IdentityOperator,
    SparseEmbedding,
    _ITYPE,
    _TORCH_TO_SKT,
    _host,
    _ptr,
    _stream_ptr,
    check_count,
    check_eps,
    default_sparse_dim,
    pcg64_state,
    seed_words,
    sparse_embedding_or_identity,
)

RANK_REL_TOL = 1e-10  # linalg.py:20-32 Tolerances.rank_rel_tol


def as_dense(a, name: str = "matrix") -> np.ndarray:
    """_validation.py:16-27."""
    if sp.issparse(a):
        a = a.toarray()
    out = np.asarray(a, dtype=np.float64)
    if out.ndim == 1:
        out = out.reshape(-1, 1)
    if out.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {out.shape}")
    if not np.all(np.isfinite(out)):
        raise ValueError(f"{name} contains non-finite entries")
    return out


def as_csr(a, name: str = "matrix") -> sp.csr_array:
    """_validation.py:30-41."""
    out = sp.csr_array(a, dtype=np.float64) if sp.issparse(a) else sp.csr_array(as_dense(a, name))
    out.sum_duplicates()
    out.eliminate_zeros()
    out.sort_indices()
    if not np.all(np.isfinite(out.data)):
        raise ValueError(f"{name} contains non-finite entries")
    return out


def as_matrix(a, name: str = "matrix"):
    return as_csr(a, name) if sp.issparse(a) else as_dense(a, name)


def pseudoinverse_solve(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """linalg.py:75-90 (thin SVD, singular values below 1e-10 sigma_1 dropped)."""
    u, sigma, vt = np.linalg.svd(a, full_matrices=False)
    if sigma.size == 0 or sigma[0] == 0.0:
        return np.zeros((a.shape[1], b.shape[1]))
    rank = int(np.count_nonzero(sigma > RANK_REL_TOL * sigma[0]))
    if rank == 0:
        return np.zeros((a.shape[1], b.shape[1]))
    ur, sr, vr = u[:, :rank], sigma[:rank], vt.T[:, :rank]
    return vr @ ((ur.T @ b) / sr[:, None])


@dataclass(frozen=True)
class RegressionSolution:
    """regress.py:54-64 (fields used by sketch_solve_ls)."""

    x: np.ndarray
    residual_norm: float
    method: str
    sketch_dim: int
    seed: int
    iterations: int = 0
    residual_history: tuple = ()
    coreset: object = None


def residual_fro(a, x, b, device=None) -> float:
    """||A x - b||_F (regress.py:81-82) in one fused pass over A on the GPU
    (skt_residual_dense / skt_residual_csr).  ``a``: numpy / scipy CSR / torch;
    ``x``: d x k (or d); ``b``: n x k (or n)."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    L = _lib.lib()
    n, d = a.shape[0], a.shape[1]
    xt = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64) if not isinstance(x, torch.Tensor) else x)
    xt = xt.to(device=device, dtype=torch.float64).reshape(d, -1).contiguous()
    k = xt.shape[1]
    bt = torch.as_tensor(np.ascontiguousarray(b) if not isinstance(b, torch.Tensor) else b).to(device)
    if bt.dtype not in _TORCH_TO_SKT:
        bt = bt.to(torch.float64)
    bt = bt.reshape(n, -1).contiguous()
    if bt.shape[1] != k:
        raise ValueError(f"x has {k} columns, b has {bt.shape[1]}")
    ws_bytes = ctypes.c_size_t()
    check(L.skt_residual_workspace(ctypes.byref(ws_bytes)))
    ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device=device)
    out = torch.empty(1, dtype=torch.float64, device=device)
    with torch.cuda.device(device):
        stream = _stream_ptr(device)
        if sp.issparse(a) or (isinstance(a, torch.Tensor) and a.layout == torch.sparse_csr):
            if isinstance(a, torch.Tensor):
                ip, ix, vv = (t.to(device) for t in (a.crow_indices(), a.col_indices(), a.values()))
            else:
                m = sp.csr_array(a)
                ip, ix, vv = (torch.from_numpy(np.ascontiguousarray(t)).to(device)
                              for t in (m.indptr, m.indices, m.data))
            if vv.dtype not in _TORCH_TO_SKT:
                vv = vv.to(torch.float64)
            check(L.skt_residual_csr(n, d, _ptr(ip), _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype], _ptr(vv),
                                     _TORCH_TO_SKT[vv.dtype], _ptr(xt), k, _ptr(bt), _TORCH_TO_SKT[bt.dtype],
                                     k, _ptr(out), _ptr(ws), ws_bytes.value, stream))
        else:
            at = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            at = at.to(device)
            if at.dtype not in _TORCH_TO_SKT:
                at = at.to(torch.float64)
            at = at.reshape(n, -1).contiguous()
            check(L.skt_residual_dense(n, d, _ptr(at), _TORCH_TO_SKT[at.dtype], max(d, 1), _ptr(xt), k, _ptr(bt),
                                       _TORCH_TO_SKT[bt.dtype], k, _ptr(out), _ptr(ws), ws_bytes.value, stream))
    return math.sqrt(float(out.item()))


def _residual_fro_gpu(a, x: np.ndarray, b: np.ndarray, device) -> float:
    return residual_fro(a, x, b, device)


def sketch_solve_ls(a, b, eps: float, seed: int = 0, operator=None) -> RegressionSolution:
    """regress.py:85-116 with the sketch applied on the GPU."""
    a = as_matrix(a)
    b = as_dense(b)
    if a.shape[0] != b.shape[0]:
        raise ValueError(f"operands must have the same number of rows: {a.shape[0]} vs {b.shape[0]}")
    eps = check_eps(eps)
    if operator is None:
        t = default_sparse_dim(a.shape[1] + b.shape[1], eps)
        operator = sparse_embedding_or_identity(a.shape[0], t, seed)
    sa = operator.apply(a)
    sb = operator.apply(b)
    x = pseudoinverse_solve(np.asarray(sa), np.asarray(sb))
    device = getattr(operator, "device", None) or torch.device("cuda", torch.cuda.current_device())
    return RegressionSolution(
        x=x,
        residual_norm=_residual_fro_gpu(a, x, b, device),
        method="sketch",
        sketch_dim=operator.output_dim,
        seed=int(seed),
    )


# ---------------------------------------------------------------------------
# leverage scores
# ---------------------------------------------------------------------------
def pivoted_qr_rank(a: np.ndarray):
    """linalg.py:142-155."""
    q, r, perm = scipy.linalg.qr(a, mode="economic", pivoting=True)
    diag = np.abs(np.diag(r))
    rank = 0 if diag.size == 0 or diag[0] == 0.0 else int(np.count_nonzero(diag > RANK_REL_TOL * diag[0]))
    return q, r, perm, rank


def basis_change(sketched: np.ndarray):
    """leverage.py:36-47: N (d x rank) with sketched @ N orthonormal."""
    _, r, perm, rank = pivoted_qr_rank(sketched)
    if rank == 0:
        return np.zeros((sketched.shape[1], 0)), 0
    n_mat = np.zeros((sketched.shape[1], rank))
    n_mat[perm[:rank]] = np.linalg.inv(r[:rank, :rank])
    return n_mat, rank


def gaussian_jl_entries(rows: int, cols: int, seed: int) -> np.ndarray:
    """GaussianJl.entries (sketch.py:344-355): _rng(seed, 4, 0) normals / sqrt(rows)."""
    rng = np.random.default_rng(np.random.SeedSequence(int(seed), spawn_key=(4, 0)))
    return rng.standard_normal((rows, cols)) / math.sqrt(rows)


def lev_rownorms(a, probe, device=None, out_dtype=torch.float64):
    """scores_i = ||A_i probe||^2 (leverage.py:90-91) fused on the GPU (K5).

    ``a``: scipy CSR / numpy dense / torch (CUDA) dense or sparse-CSR tensor;
    ``probe``: d x k (fp64).  Returns numpy for host input, torch otherwise.
    """
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    L = _lib.lib()
    host = not isinstance(a, torch.Tensor)
    p = torch.as_tensor(np.ascontiguousarray(probe, dtype=np.float64) if not isinstance(probe, torch.Tensor) else probe)
    p = p.to(device=device, dtype=torch.float64).contiguous()
    d, k = p.shape
    with torch.cuda.device(device):
        stream = _stream_ptr(device)
        if sp.issparse(a) or (isinstance(a, torch.Tensor) and a.layout == torch.sparse_csr):
            if isinstance(a, torch.Tensor):
                ip, ix, vv = (x.to(device) for x in (a.crow_indices(), a.col_indices(), a.values()))
                n = a.shape[0]
            else:
                m = sp.csr_array(a)
                if m.data.dtype not in (np.float32, np.float64):
                    m = sp.csr_array(m, dtype=np.float64)
                n = m.shape[0]
                ip, ix, vv = (torch.from_numpy(np.ascontiguousarray(x)).to(device) for x in (m.indptr, m.indices, m.data))
            if a.shape[1] != d:
                raise ValueError(f"probe has {d} rows, matrix has {a.shape[1]} columns")
            if vv.dtype not in _TORCH_TO_SKT:
                vv = vv.to(torch.float64)
            out = torch.empty(n, dtype=out_dtype, device=device)
            check(
                L.skt_lev_rownorms_csr(
                    n, d, _ptr(ip), _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype], _ptr(vv),
                    _TORCH_TO_SKT[vv.dtype], _ptr(p), k, _ptr(out), _TORCH_TO_SKT[out_dtype], stream,
                )
            )
        else:
            x = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(a)))
            x = x.to(device)
            if x.dtype not in _TORCH_TO_SKT:
                x = x.to(torch.float64)
            x = x.reshape(x.shape[0], -1).contiguous()
            if x.shape[1] != d:
                raise ValueError(f"probe has {d} rows, matrix has {x.shape[1]} columns")
            out = torch.empty(x.shape[0], dtype=out_dtype, device=device)
            flag = torch.empty(1, dtype=torch.int32, device=device)
            check(
                L.skt_lev_rownorms_dense(
                    x.shape[0], d, _ptr(x), _TORCH_TO_SKT[x.dtype], max(d, 1), _ptr(p), k, _ptr(out),
                    _TORCH_TO_SKT[out_dtype], _ptr(flag), stream,
                )
            )
            if x.shape[0] > 0 and int(flag.item()) != 0:
                raise ValueError("matrix contains non-finite entries")
    if host:
        return _host(out).numpy()
    return out if a.is_cuda else _host(out)


@dataclass(frozen=True)
class LeverageRun:
    scores: np.ndarray
    rank: int
    sa: np.ndarray
    probe: np.ndarray


def leverage_scores_sketched(a, m: int, k: int, seed: int, rep: int = 0) -> LeverageRun:
    """One repetition of leverage.py:71-91 with sketch size ``m`` and JL width
    ``k`` chosen by the caller (the SRHT stage is the identity when m does not
    exceed _srht_rows(rank), as in BASELINE config 4)."""
    sub = np.random.SeedSequence(int(seed), spawn_key=(100 + rep,)).generate_state(3)
    n = a.shape[0]
    s = SparseEmbedding(n, m, int(sub[0]))
    sa = s.apply(a)
    n_mat, rank = basis_change(sa)
    if rank == 0:
        return LeverageRun(np.zeros(n), 0, sa, np.zeros((a.shape[1], 0)))
    g = gaussian_jl_entries(k, rank, int(sub[2]))
    probe = n_mat @ g.T
    scores = lev_rownorms(a, probe)
    return LeverageRun(scores, rank, sa, probe)


def _srht_draws(n_pad: int, seed: int, device):
    """The SRHT's sign vector (stream (2, 0) .choice over n_pad) and its row
    draws (stream (2, 1) .integers(0, n_pad)), one K1 call: bucket stream
    (2, 1) with t = n_pad, sign stream (2, 0) -- n_pad row draws; an operator
    with t samples uses the first t (sketch.py:276-281)."""
    L = _lib.lib()
    hs, ss = pcg64_state(seed, (2, 1)), pcg64_state(seed, (2, 0))
    rows = torch.empty(n_pad, dtype=torch.int32, device=device)
    sign = torch.empty(n_pad, dtype=torch.int8, device=device)
    kb = ctypes.c_size_t()
    check(L.skt_hash_signs_workspace(n_pad, n_pad, ctypes.byref(kb)))
    kws = torch.empty(max(kb.value, 8), dtype=torch.uint8, device=device)
    with torch.cuda.device(device):
        check(L.skt_hash_signs(ctypes.byref(hs), ctypes.byref(ss), 0, n_pad, n_pad, _ptr(rows), _ptr(sign),
                               _ptr(kws), kb.value, _stream_ptr(device)))
        torch.cuda.current_stream(device).synchronize()
    return rows, sign


def srht_apply(a, t: int, seed: int, device=None, all_rows: bool = False):
    """SrhtOperator(n, t, seed).apply(a) (sketch.py:255-291) on the GPU
    (skt_srht_apply: sign flip + padding, the reference's _fwht butterflies
    stage by stage, sampling + scaling), bit-identical to the reference.  The
    sign vector and the sampled rows are the reference's streams (2, 0) and
    (2, 1) of SeedSequence(seed), drawn on the GPU by K1 (``all_rows``: every
    padded row in order, t = n_pad).  ``a``: numpy or torch (n x d or n);
    returns the same kind (torch on ``a``'s device)."""
    if device is None:
        device = a.device if isinstance(a, torch.Tensor) and a.is_cuda else torch.device(
            "cuda", torch.cuda.current_device())
    host = not isinstance(a, torch.Tensor)
    x = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64) if host else a)
    x = x.to(device=device, dtype=torch.float64)
    one_d = x.dim() == 1
    x = x.reshape(x.shape[0], -1).contiguous()
    n, d = x.shape
    if n < 1 or t < 1:
        raise ValueError("n and t must be >= 1")
    n_pad = 1 << (n - 1).bit_length()
    if all_rows:
        t = n_pad
    if t > n_pad:
        raise ValueError(f"t={t} exceeds padded dimension {n_pad}")

    scale = math.sqrt(n_pad / t) / math.sqrt(n_pad)
    out = torch.empty((t, d), dtype=torch.float64, device=device)
    L = _lib.lib()
    rows, sign = _srht_draws(n_pad, seed, device)
    if all_rows:
        rows = torch.arange(n_pad, dtype=torch.int32, device=device)
    with torch.cuda.device(device):
        stream = _stream_ptr(device)
        wsb = ctypes.c_size_t()
        check(L.skt_srht_workspace(n, d, ctypes.byref(wsb)))
        ws = torch.empty(max(wsb.value, 8), dtype=torch.uint8, device=device)
        check(L.skt_srht_apply(_ptr(x), n, d, max(d, 1), _ptr(sign), _ptr(rows), t, scale, _ptr(out), max(d, 1),
                               _ptr(ws), wsb.value, stream))
        torch.cuda.current_stream(device).synchronize()  # workspaces freed after the stream consumed them
    if one_d:
        out = out.reshape(-1)
    return _host(out).numpy() if host else out


class SrhtOperator:
    """sketch.py:255-302: subsampled randomized Hadamard transform, applied on
    the GPU (srht_apply).  ``sign`` / ``sampled_rows`` are host views of the
    K1 draws (the reference's arrays, bit for bit)."""

    family = "srht"

    def __init__(self, n: int, t: int, seed: int, all_rows: bool = False, device=None):
        self.input_dim = check_count(n, "n")
        self.n_pad = 1 << (self.input_dim - 1).bit_length()
        self.seed = int(seed)
        self.all_rows = bool(all_rows)
        if all_rows:
            t = self.n_pad
        self.output_dim = check_count(t, "t")
        if self.output_dim > self.n_pad:
            raise ValueError(f"t={t} exceeds padded dimension {self.n_pad}")
        self.scale = math.sqrt(self.n_pad / self.output_dim) / math.sqrt(self.n_pad)
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._views = None

    def _draws(self):
        if self._views is None:
            rows, sign = _srht_draws(self.n_pad, self.seed, self.device)
            picks = np.arange(self.n_pad) if self.all_rows else rows[: self.output_dim].cpu().numpy().astype(np.int64)
            self._views = (sign.cpu().numpy().astype(np.float64), picks)
        return self._views

    @property
    def sign(self) -> np.ndarray:
        return self._draws()[0]

    @property
    def sampled_rows(self) -> np.ndarray:
        return self._draws()[1]

    def apply(self, a):
        if a.shape[0] != self.input_dim:
            raise ValueError(f"operator expects {self.input_dim} rows, got {a.shape[0]}")
        if isinstance(a, torch.Tensor):
            x = a.to_dense() if a.layout != torch.strided else a
            return srht_apply(x.to(self.device), self.output_dim, self.seed, self.device, self.all_rows)
        return srht_apply(as_dense(a), self.output_dim, self.seed, self.device, self.all_rows)

    def dense(self) -> np.ndarray:
        return self.apply(np.eye(self.input_dim))

    def descriptor(self) -> dict:
        return {"family": self.family, "n": self.input_dim, "t": self.output_dim, "seed": self.seed,
                "all_rows": self.all_rows}


def default_srht_dim(r: int, eps: float, n: int) -> int:
    """sketch.py:83-94."""
    r = check_count(r, "r")
    n = check_count(n, "n")
    eps = check_eps(eps)
    t = _C.SRHT_DIM_C * (math.sqrt(r) + math.sqrt(math.log(max(n, 2)))) ** 2 * math.log(r + 1.0) / eps**2
    return max(r + 1, math.ceil(t))


def srht_or_identity(n: int, t: int, seed: int):
    """sketch.py:429-433."""
    if t >= n:
        return IdentityOperator(n)
    return SrhtOperator(n, t, seed)


# ---------------------------------------------------------------------------
# nonnegative regression (regress.py:288-370)
# ---------------------------------------------------------------------------
class SolverError(RuntimeError):
    """regress.py:36-41: an iterative / active-set solve that failed; ``best``
    is the last iterate."""

    def __init__(self, message, best=None):
        super().__init__(message)
        self.best = best


def lawson_hanson_nnls(m, y, dual_tol: float = 1e-8, max_passes: int | None = None) -> np.ndarray:
    """Lawson-Hanson active-set NNLS, min ||m x - y|| s.t. x >= 0 (regress.py:
    288-327): add the inactive coordinate with the largest dual value, solve
    least squares on the passive set, and step back to the feasible boundary
    while the passive solution has non-positive entries.  Stops when every
    inactive dual value is <= dual_tol * max(max |w_0|, 1); raises SolverError
    after max_passes (default 10 d + 50) additions.  Host code on the small
    sketched problem, as in the reference."""
    m = as_dense(m)
    y = np.asarray(y, dtype=np.float64).ravel()
    d = m.shape[1]
    cap = 10 * d + 50 if max_passes is None else max_passes
    x = np.zeros(d)
    passive = np.zeros(d, dtype=bool)
    w = m.T @ (y - m @ x)
    scale = max(np.abs(w).max(initial=0.0), 1.0)
    added = 0
    while True:
        free = ~passive
        if not free.any() or w[free].max(initial=-np.inf) <= dual_tol * scale:
            return x
        added += 1
        if added > cap:
            raise SolverError("NNLS did not converge within the pass cap", best=x)
        candidates = np.flatnonzero(free)
        passive[candidates[np.argmax(w[free])]] = True
        while True:
            cols = np.flatnonzero(passive)
            z = np.zeros(d)
            z[cols] = np.linalg.lstsq(m[:, cols], y, rcond=None)[0]
            if z[cols].min(initial=np.inf) > 0:
                x = z
                break
            blocking = cols[z[cols] <= 0]  # passive coordinates the full step would push to <= 0
            step = np.min(x[blocking] / np.maximum(x[blocking] - z[blocking], 1e-300))
            x = x + step * (z - x)
            passive &= x > 1e-14
        w = m.T @ (y - m @ x)


def nonneg_regression(a, b, eps: float, seed: int = 0, operator=None) -> RegressionSolution:
    """regress.py:330-370: min_{X >= 0} ||A X - B|| on an affine-embedding
    sketch -- SRHT o sparse embedding, each at eps / 3 -- applied on the GPU
    (K1-K4, then the SRHT of the small sketch), Lawson-Hanson per column on
    the host, the residual on the original data by the fused GPU pass."""
    a = as_matrix(a)
    b = as_dense(b)
    if a.shape[0] != b.shape[0]:
        raise ValueError(f"operands must have the same number of rows: {a.shape[0]} vs {b.shape[0]}")
    eps = check_eps(eps)
    if operator is None:
        joint = a.shape[1] + b.shape[1]
        n = a.shape[0]
        t1 = min(default_sparse_dim(joint, eps / 3), n)
        inner = sparse_embedding_or_identity(n, t1, _seed_stream(seed, 0))
        t2 = default_srht_dim(joint, eps / 3, inner.output_dim)
        operator = ComposedSketch(srht_or_identity(inner.output_dim, t2, _seed_stream(seed, 1)), inner)
    sa = np.asarray(_host_array(operator.apply(a)))
    sb = np.asarray(_host_array(operator.apply(b)))
    x = np.column_stack([lawson_hanson_nnls(sa, sb[:, j]) for j in range(sb.shape[1])])
    device = getattr(getattr(operator, "inner", operator), "device", None) or torch.device(
        "cuda", torch.cuda.current_device())
    return RegressionSolution(
        x=x,
        residual_norm=_residual_fro_gpu(a, x, b, device),
        method="nnls",
        sketch_dim=operator.output_dim,
        seed=int(seed),
    )


def _host_array(x):
    return _host(x).numpy() if isinstance(x, torch.Tensor) else x


def _seed_stream(seed: int, *key: int) -> int:
    """regress.py:76-77."""
    return int(np.random.SeedSequence(int(seed), spawn_key=key).generate_state(1)[0])


@dataclass(frozen=True)
class LeverageScores:
    """leverage.py:26-32."""

    scores: np.ndarray
    eps: float
    repetitions: int
    seed: int
    rank: int


def approx_leverage_scores(a, eps: float, repetitions: int = 5, seed: int = 0) -> LeverageScores:
    """leverage.py:50-97 with the sketch (K3/K4), the SRHT of the sketch and
    the fused contraction + row norms (K5) on the GPU; the pivoted QR / basis
    change of the small sketch and the median stay on the host as in the
    reference."""
    from .sketch import check_count  # noqa: PLC0415

    eps = check_eps(eps)
    repetitions = check_count(repetitions, "repetitions")
    if repetitions % 2 == 0:
        raise ValueError("repetitions must be odd for a median to amplify")
    a = as_matrix(a)
    n, d = a.shape
    per_rep = np.zeros((repetitions, n))
    ranks = []
    t1 = default_sparse_dim(max(d, 1), 0.25)  # default_t1 (leverage.py:100-102)
    for rep in range(repetitions):
        sub = np.random.SeedSequence(int(seed), spawn_key=(100 + rep,)).generate_state(3)
        s = sparse_embedding_or_identity(n, t1, int(sub[0]))
        sa = np.asarray(s.apply(a))
        _, _, _, rank = pivoted_qr_rank(sa)
        if rank == 0:
            ranks.append(0)
            continue
        log_r = math.log(max(rank, 2))
        t_f = max(rank + 1, math.ceil(40.0 * rank * log_r * log_r))  # _srht_rows (leverage.py:105-107)
        fsa = sa if t_f >= sa.shape[0] else srht_apply(sa, t_f, int(sub[1]))
        n_mat, rank2 = basis_change(fsa)
        ranks.append(rank2)
        if rank2 == 0:
            continue
        m = max(1, math.ceil(16.0 * math.log(max(n, 2)) / eps**2))
        probe = n_mat @ gaussian_jl_entries(m, rank2, int(sub[2])).T
        per_rep[rep] = lev_rownorms(a, probe)
    rank = int(np.median(ranks)) if ranks else 0
    return LeverageScores(scores=np.median(per_rep, axis=0), eps=eps, repetitions=repetitions,
                          seed=int(seed), rank=rank)


__all__ = [
    "as_dense",
    "as_csr",
    "as_matrix",
    "pseudoinverse_solve",
    "RegressionSolution",
    "sketch_solve_ls",
    "pivoted_qr_rank",
    "basis_change",
    "gaussian_jl_entries",
    "lev_rownorms",
    "leverage_scores_sketched",
    "approx_leverage_scores",
    "LeverageScores",
    "residual_fro",
    "srht_apply",
    "seed_words",
]
