"""Generalized sparse embedding on the GPU: the reference's
GeneralizedSparseEmbedding (sketch.py:176-238), the operator lp.py's block
embeddings are made of (§8f rank 4).

Every input row j contributes to k_blocks output rows
    h_b(j) = outer(j) * (k v) + b v + inner_b(j),  weight sign_b(j) / sqrt(k),
one per block b.  The device build reuses the CountSketch machinery on the
k n "virtual rows" vid = b n + j (the reference draws its (k, n)-shaped inner
streams in that order): K1 draws the three streams bit-exactly, a combine
kernel forms h(vid), K2 stably sorts the virtual rows by output row and the
plan words are folded back to j.  ``apply`` runs the weighted kernels of
csrc/gse.cu, which reproduce scipy's csr_matvecs / csr_matmat element order
and rounding (bit-identical to the reference).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import scipy.sparse as sp
import torch

from . import _constants as C
from . import _lib
from ._lib import check
from .sketch import (
    _ITYPE,
    _TORCH_TO_SKT,
    SketchOperator,
    _host,
    _ptr,
    _stream_ptr,
    _workspace,
    check_count,
    check_eps,
    pcg64_state,
)


def generalized_dims(r: int, eps: float, delta: float) -> tuple[int, int, int, int]:
    """(q, k_blocks, v, t), sketch.py:69-80."""
    r = check_count(r, "r")
    eps = check_eps(eps)
    delta = check_eps(delta, name="delta")
    k_blocks = max(1, math.ceil(C.GEN_K_C * math.log(r / (eps * delta)) / eps))
    v = max(1, math.ceil(C.GEN_V_C / eps))
    q = max(1, math.ceil(C.GEN_Q_C * r * (r + math.log(1.0 / (delta * eps))) / eps**2))
    return q, k_blocks, v, q * k_blocks * v


class GeneralizedSparseEmbedding(SketchOperator):
    """GeneralizedSparseEmbedding(n, r, eps, delta, seed) on the GPU."""

    family = "generalized"

    def __init__(self, n: int, r: int, eps: float, delta: float, seed: int, device=None):
        self.input_dim = check_count(n, "n")
        self.r = check_count(r, "r")
        self.eps = check_eps(eps)
        self.delta = check_eps(delta, name="delta")
        self.seed = int(seed)
        self.q, self.k_blocks, self.v, self.output_dim = generalized_dims(r, self.eps, self.delta)
        self.scale = 1.0 / math.sqrt(self.k_blocks)
        self.dense_fallback = self.output_dim > self.input_dim
        if self.output_dim >= 2**32 or self.k_blocks * self.input_dim >= 2**31:
            raise ValueError("generalized embedding too large for the 32-bit plan")
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._mat_cache = None
        self._build()

    def _build(self):
        L = _lib.lib()
        n, k, v, q, t = self.input_dim, self.k_blocks, self.v, self.q, self.output_dim
        dev = self.device
        with torch.cuda.device(dev):
            stream = _stream_ptr(dev)
            # outer buckets: stream (1, 0) .integers(0, q, n)
            self.outer = torch.empty(n, dtype=torch.int32, device=dev)
            nb = ctypes.c_size_t()
            check(L.skt_hash_signs_workspace(n, q, ctypes.byref(nb)))
            ws1 = _workspace(nb.value, dev)
            ho = pcg64_state(self.seed, (1, 0))
            check(L.skt_hash_signs(ctypes.byref(ho), ctypes.byref(ho), 0, n, q, _ptr(self.outer), None,
                                   _ptr(ws1), nb.value, stream))
            # inner buckets / signs: streams (1, 1) / (1, 2) over the (k, n) draws
            kn = k * n
            self.inner = torch.empty(kn, dtype=torch.int32, device=dev)
            self.inner_s = torch.empty(kn, dtype=torch.int8, device=dev)
            check(L.skt_hash_signs_workspace(kn, v, ctypes.byref(nb)))
            ws2 = _workspace(nb.value, dev)
            hi, si = pcg64_state(self.seed, (1, 1)), pcg64_state(self.seed, (1, 2))
            check(L.skt_hash_signs(ctypes.byref(hi), ctypes.byref(si), 0, kn, v, _ptr(self.inner),
                                   _ptr(self.inner_s), _ptr(ws2), nb.value, stream))
            # h(vid) and the plan over the k n virtual rows
            self.h = torch.empty(kn, dtype=torch.int32, device=dev)
            check(L.skt_gse_buckets(_ptr(self.outer), _ptr(self.inner), n, k, v, q, _ptr(self.h), stream))
            self.plan_indptr = torch.empty(t + 1, dtype=torch.int64, device=dev)
            self.plan_rows = torch.empty(kn, dtype=torch.int32, device=dev)
            check(L.skt_plan_workspace(kn, t, 0, ctypes.byref(nb)))
            ws3 = _workspace(nb.value, dev)
            check(L.skt_plan_build(_ptr(self.h), _ptr(self.inner_s), kn, t, 0, _ptr(self.plan_indptr),
                                   _ptr(self.plan_rows), None, _ptr(ws3), nb.value, stream))
            check(L.skt_gse_fold_rows(_ptr(self.plan_rows), kn, n, stream))
            torch.cuda.current_stream(dev).synchronize()  # workspaces released after use
            del ws1, ws2, ws3

    # ---- host views (API / test compatibility; sketch.py:201-218) ----------
    @property
    def outer_bucket(self) -> np.ndarray:
        return self.outer.cpu().numpy().view(np.uint32).astype(np.int64)

    @property
    def inner_bucket(self) -> np.ndarray:
        return self.inner.cpu().numpy().view(np.uint32).astype(np.int64).reshape(self.k_blocks, self.input_dim)

    @property
    def inner_sign(self) -> np.ndarray:
        return self.inner_s.cpu().numpy().astype(np.float64).reshape(self.k_blocks, self.input_dim)

    @property
    def _mat(self) -> sp.csr_array:
        if self._mat_cache is None:
            words = self.plan_rows.cpu().numpy().view(np.uint32)
            data = np.where(words >> 31, -1.0, 1.0) * self.scale
            self._mat_cache = sp.csr_array(
                (data, (words & 0x7FFFFFFF).astype(np.int32), self.plan_indptr.cpu().numpy()),
                shape=(self.output_dim, self.input_dim))
        return self._mat_cache

    def descriptor(self) -> dict:
        return {"family": self.family, "n": self.input_dim, "r": self.r, "eps": self.eps,
                "delta": self.delta, "seed": self.seed}

    # ---- apply ---------------------------------------------------------------
    def apply(self, a):
        """self._mat @ a (sketch.py:222-227): fp64 (t, d); numpy in -> numpy
        out, torch in -> torch on the input's device."""
        self._check_rows(a)
        L = _lib.lib()
        dev = self.device
        is_torch = isinstance(a, torch.Tensor)
        with torch.cuda.device(dev):
            stream = _stream_ptr(dev)
            if sp.issparse(a) or (is_torch and a.layout == torch.sparse_csr):
                if is_torch:
                    ip, ix, vv = (x.to(dev) for x in (a.crow_indices(), a.col_indices(), a.values()))
                else:
                    m = sp.csr_array(a)
                    ip, ix, vv = (torch.from_numpy(np.ascontiguousarray(x)).to(dev)
                                  for x in (m.indptr, m.indices, m.data))
                if vv.dtype not in _TORCH_TO_SKT:
                    vv = vv.to(torch.float64)
                d = a.shape[1]
                out = torch.empty((self.output_dim, d), dtype=torch.float64, device=dev)
                check(L.skt_gse_apply_csr(_ptr(self.plan_indptr), _ptr(self.plan_rows), self.output_dim, _ptr(ip),
                                          _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype], _ptr(vv),
                                          _TORCH_TO_SKT[vv.dtype], d, self.scale, _ptr(out), max(d, 1), stream))
            else:
                x = a if is_torch else torch.from_numpy(np.ascontiguousarray(np.asarray(a)))
                x = x.to(dev)
                if x.dtype not in _TORCH_TO_SKT:
                    x = x.to(torch.float64)
                one_d = x.dim() == 1
                x = x.reshape(x.shape[0], -1).contiguous()
                d = x.shape[1]
                out = torch.empty((self.output_dim, d), dtype=torch.float64, device=dev)
                check(L.skt_gse_apply_dense(_ptr(self.plan_indptr), _ptr(self.plan_rows), self.output_dim,
                                            x.shape[0], _ptr(x),
                                            _TORCH_TO_SKT[x.dtype], d, max(d, 1), self.scale, _ptr(out), max(d, 1),
                                            None, stream))
                if one_d:
                    out = out.reshape(-1)
        if is_torch:
            return out if a.is_cuda else _host(out)
        return _host(out).numpy()


def make_generalized_sparse_embedding(n: int, r: int, eps: float, delta: float, seed: int):
    """sketch.py make_generalized_sparse_embedding."""
    return GeneralizedSparseEmbedding(n, r, eps, delta, seed)


__all__ = ["GeneralizedSparseEmbedding", "generalized_dims", "make_generalized_sparse_embedding"]
