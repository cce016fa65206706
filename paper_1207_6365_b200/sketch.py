"""CountSketch / sparse-embedding operator on B200 -- the drop-in boundary.

Mirrors the reference's ``SketchOperator`` protocol (sketch.py:97-119) and
``SparseEmbedding`` (sketch.py:138-173): same constructor ``(n, t, seed)``,
``family == "sparse"``, ``input_dim``/``output_dim``/``seed``, ``apply``,
``dense``, ``descriptor``, plus the host attributes tests read (``bucket``,
``sign``, ``_mat``), materialised lazily from the device plan.

Construction runs K1 (bit-exact h/s from the seed's PCG64 streams) and K2 (the
bucket-sorted plan) on the GPU; ``apply`` runs K3 (dense) or K4 (CSR).  Inputs
may be numpy arrays / scipy sparse matrices (copied to the device and back, the
reference's calling convention: a new float64 ndarray) or torch tensors (CUDA
tensors stay on the device; CPU tensors are copied in and the result copied
out).  There is no CPU fallback: without the native library or a CUDA device
every entry point raises.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np
import scipy.sparse as sp
import torch

from . import _constants as C
from . import _lib
from ._lib import SktPcg64, check

__all__ = [
    "SparseEmbedding",
    "IdentityOperator",
    "ComposedSketch",
    "make_sparse_embedding",
    "sparse_embedding_or_identity",
    "apply_left",
    "apply_right",
    "compose",
    "default_sparse_dim",
    "to_descriptor",
    "from_descriptor",
    "seed_words",
    "pcg64_state",
    "derived_seed",
]

_TORCH_TO_SKT = {torch.float32: _lib.SKT_F32, torch.float64: _lib.SKT_F64}
_ITYPE = {torch.int32: _lib.SKT_I32, torch.int64: _lib.SKT_I64}


# --------------------------------------------------------------------------
# validation helpers (restating _validation.py:16-27, 71-75)
# --------------------------------------------------------------------------
def check_count(k, name: str = "count", minimum: int = 1) -> int:
    k = int(k)
    if k < minimum:
        raise ValueError(f"{name} must be >= {minimum}, got {k}")
    return k


def check_eps(eps: float, lo: float = 0.0, hi: float = 1.0, name: str = "eps") -> float:
    eps = float(eps)
    if not (lo < eps < hi):
        raise ValueError(f"{name} must be in ({lo}, {hi}), got {eps}")
    return eps


def default_sparse_dim(r: int, eps: float) -> int:
    """sketch.py:56-66: max(FLOOR, ceil(C (r/eps)^2 max(1, ln(r/eps))))."""
    r = check_count(r, "r")
    eps = check_eps(eps)
    x = r / eps
    t = C.SPARSE_DIM_C * x * x * max(1.0, math.log(x))
    return max(C.SPARSE_DIM_FLOOR, math.ceil(t))


# --------------------------------------------------------------------------
# seeding (sketch.py:51-53) through the C ABI
# --------------------------------------------------------------------------
def seed_words(seed: int) -> np.ndarray:
    """Little-endian uint32 words of a non-negative int (numpy's coercion)."""
    seed = int(seed)
    if seed < 0:
        raise ValueError("expected non-negative integer")
    words = []
    while True:
        words.append(seed & 0xFFFFFFFF)
        seed >>= 32
        if seed == 0:
            break
    return np.asarray(words, dtype=np.uint32)


def pcg64_state(seed: int, spawn_key=()) -> SktPcg64:
    """PCG64(SeedSequence(seed, spawn_key)) state, computed by the library."""
    ent = seed_words(seed)
    key = np.asarray([int(k) for k in spawn_key], dtype=np.uint32)
    st = SktPcg64()
    check(
        _lib.lib().skt_pcg64_seed(
            ent.ctypes.data, len(ent), key.ctypes.data if len(key) else None, len(key), ctypes.byref(st)
        )
    )
    return st


def derived_seed(seed: int, *key: int) -> int:
    """SeedSequence(seed, spawn_key=key).generate_state(1)[0] (regress.py:77-78)."""
    ent = seed_words(seed)
    k = np.asarray([int(x) for x in key], dtype=np.uint32)
    out = np.zeros(1, dtype=np.uint32)
    check(
        _lib.lib().skt_seedseq_generate(
            ent.ctypes.data, len(ent), k.ctypes.data if len(k) else None, len(k), out.ctypes.data, 1
        )
    )
    return int(out[0])


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _workspace(nbytes: int, device) -> torch.Tensor | None:
    if nbytes == 0:
        return None
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _host(t: torch.Tensor) -> torch.Tensor:
    """Device result -> a new host tensor in page-locked memory (torch's caching
    host allocator): the read-back runs at PCIe speed instead of the ~2 GB/s
    of a copy into freshly faulted pageable pages (15 ms for config 3's SA)."""
    try:
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    except RuntimeError:  # page-locked memory exhausted
        return t.cpu()
    out.copy_(t)
    return out


_STAGE_MIN = 1 << 20  # host arrays below this go through torch's own copy


def _to_device(x: np.ndarray, device) -> torch.Tensor:
    """numpy array (pageable host memory) -> new device tensor, through the
    library's page-locked staging ring (skt_memcpy_staged) for large arrays."""
    x = np.ascontiguousarray(x)
    if x.nbytes < _STAGE_MIN:
        return torch.from_numpy(x).to(device)
    out = torch.empty(x.shape, dtype=torch.from_numpy(x[:0]).dtype, device=device)
    with torch.cuda.device(device):
        check(_lib.lib().skt_memcpy_staged(_ptr(out), x.ctypes.data, x.nbytes, 0, _stream_ptr(device)))
    return out


def csr_is_canonical_device(indptr: torch.Tensor, indices: torch.Tensor, n: int) -> bool:
    """Strictly increasing column indices in every row (skt_csr_check_sorted);
    one 4-byte device->host read."""
    flag = torch.empty(1, dtype=torch.int32, device=indptr.device)
    with torch.cuda.device(indptr.device):
        check(_lib.lib().skt_csr_check_sorted(n, _ptr(indptr), _ITYPE[indptr.dtype], _ptr(indices),
                                              _ITYPE[indices.dtype], _ptr(flag), _stream_ptr(indptr.device)))
    return int(flag.item()) == 0


def dense_operand(a: torch.Tensor) -> torch.Tensor:
    """A device matrix in the layout K3 reads: 2-D (1-D -> one column), f32 or
    f64 (other dtypes -> f64, as_dense's upcast), unit column stride, and rows
    that do not overlap (a broadcast view such as ``x[None].expand(n, d)`` has
    row stride 0 and is materialised)."""
    if a.dim() == 1:
        a = a.reshape(-1, 1)
    if a.dim() != 2:
        raise ValueError(f"matrix must be 2-D, got shape {tuple(a.shape)}")
    if a.dtype not in _TORCH_TO_SKT:
        a = a.to(torch.float64)
    n, d = a.shape
    if d > 0 and (a.stride(1) != 1 or (n > 1 and a.stride(0) < d)):
        a = a.contiguous()
    return a


class SketchOperator:
    """Duck-typed protocol of the reference (sketch.py:97-119)."""

    input_dim: int
    output_dim: int
    family: str

    def apply(self, a):
        raise NotImplementedError

    def dense(self) -> np.ndarray:
        return self.apply(np.eye(self.input_dim))

    def descriptor(self) -> dict:
        raise NotImplementedError

    def _check_rows(self, a) -> None:
        if a.shape[0] != self.input_dim:
            raise ValueError(f"operator expects {self.input_dim} rows, got {a.shape[0]}")


class IdentityOperator(SketchOperator):
    """sketch.py:122-135: what a pipeline uses when a sketch would not shrink."""

    family = "identity"

    def __init__(self, n: int):
        self.input_dim = self.output_dim = check_count(n, "n")

    def apply(self, a):
        self._check_rows(a)
        if isinstance(a, torch.Tensor):
            return (a.to_dense() if a.layout != torch.strided else a).to(torch.float64).reshape(a.shape[0], -1).clone()
        if sp.issparse(a):
            return a.toarray()
        out = np.asarray(a, dtype=np.float64)
        if out.ndim == 1:
            out = out.reshape(-1, 1)
        if not np.all(np.isfinite(out)):
            raise ValueError("matrix contains non-finite entries")
        return out

    def descriptor(self) -> dict:
        return {"family": self.family, "n": self.input_dim}


class SparseEmbedding(SketchOperator):
    """CountSketch: one +-1 per input coordinate, hashed to t buckets (GPU).

    Device state (on ``self.device``): ``h`` (uint32 bucket per row, stored as
    int32), ``s`` (int8 sign), ``plan_indptr`` (int64[t+1]) and ``plan_rows``
    (row ids stably sorted by bucket, sign in bit 31) -- the reference's
    ``_mat`` (sketch.py:149-151) in device form.
    """

    family = "sparse"

    def __init__(self, n: int, t: int, seed: int, device=None, row_range=None):
        self.input_dim = check_count(n, "n")
        self.output_dim = check_count(t, "t")
        self.seed = int(seed)
        if self.output_dim > 1 << 32:
            raise ValueError("t must be <= 2^32 (numpy's 32-bit bounded-integer path)")
        if self.input_dim >= 1 << 31:
            raise ValueError("n must be < 2^31")
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("SparseEmbedding runs on a CUDA device only (no CPU fallback)")
        # rows [r0, r1) of the operator held on this device (row sharding, §8e)
        r0, r1 = (0, self.input_dim) if row_range is None else (int(row_range[0]), int(row_range[1]))
        if not (0 <= r0 <= r1 <= self.input_dim):
            raise ValueError(f"bad row_range {row_range!r}")
        self.row_begin, self.row_end = r0, r1
        self._bucket = self._sign = self._mat_cache = None
        self._plan_lock = threading.Lock()
        self._build()

    # ---- K1 + K2 ----------------------------------------------------------
    def _build(self) -> None:
        L = _lib.lib()
        dev, t = self.device, self.output_dim
        r0, r1 = self.row_begin, self.row_end
        m = r1 - r0
        with torch.cuda.device(dev):
            stream = _stream_ptr(dev)
            hs = pcg64_state(self.seed, (0, 0))
            ss = pcg64_state(self.seed, (0, 1))
            self.h = torch.empty(m, dtype=torch.int32, device=dev)
            self.s = torch.empty(m, dtype=torch.int8, device=dev)
            nb = ctypes.c_size_t()
            check(L.skt_hash_signs_workspace(r1, t, ctypes.byref(nb)))
            ws = _workspace(nb.value, dev)
            check(
                L.skt_hash_signs(
                    ctypes.byref(hs), ctypes.byref(ss), r0, r1, t, _ptr(self.h), _ptr(self.s),
                    _ptr(ws), nb.value, stream,
                )
            )
            self.plan_indptr, self.plan_rows, _, ws2 = self._build_plan(0, stream)
            # keep the workspaces alive until the stream has consumed them
            self._build_ws = (ws, ws2)
            self._grouped = {0: (self.plan_indptr, self.plan_rows, None)}

    def _build_plan(self, shift: int, stream):
        """K2: rows stably sorted by bucket (shift 0) or bucket group h >> shift."""
        L = _lib.lib()
        dev, t = self.device, self.output_dim
        m = self.row_end - self.row_begin
        ngroups = ((t - 1) >> shift) + 1
        indptr = torch.empty(ngroups + 1, dtype=torch.int64, device=dev)
        rows = torch.empty(m, dtype=torch.int32, device=dev)
        blo = torch.empty(m, dtype=torch.uint8, device=dev) if shift > 0 else None
        nb = ctypes.c_size_t()
        check(L.skt_plan_workspace(m, t, shift, ctypes.byref(nb)))
        ws = _workspace(nb.value, dev)
        check(
            L.skt_plan_build(
                _ptr(self.h), _ptr(self.s), m, t, shift, _ptr(indptr), _ptr(rows), _ptr(blo),
                _ptr(ws), nb.value, stream,
            )
        )
        return indptr, rows, blo, ws

    def grouped_plan(self, shift: int):
        """Plan with rows sorted by bucket group h >> shift (cached per shift;
        built once even when several host threads apply the operator)."""
        with self._plan_lock:
            if shift not in self._grouped:
                with torch.cuda.device(self.device):
                    indptr, rows, blo, ws = self._build_plan(shift, _stream_ptr(self.device))
                    self._grouped[shift] = (indptr, rows, blo)
                    self._grouped_ws = ws
            return self._grouped[shift]

    def window_plan(self, d: int):
        """Plan of the row-window CSR kernel (csrc/csr_window.cuh): ``(W, pos,
        wpi)`` -- rows per window, every row's slot inside its window (sign in
        bit 31) and the first slot of every bucket per window -- or None when
        (t, d) is outside the kernel's range on this device.  Built once from
        the per-bucket plan and cached."""
        L = _lib.lib()
        m = self.row_end - self.row_begin
        w, nwin = ctypes.c_int32(), ctypes.c_int32()
        with torch.cuda.device(self.device):
            check(L.skt_csr_window_config(m, self.output_dim, d, ctypes.byref(w), ctypes.byref(nwin)))
        if w.value == 0:
            return None
        with self._plan_lock:
            cached = getattr(self, "_window", None)
            if cached is None or cached[0] != w.value:
                pos = torch.empty(m, dtype=torch.int32, device=self.device)
                wpi = torch.empty((nwin.value, self.output_dim + 1), dtype=torch.int32, device=self.device)
                with torch.cuda.device(self.device):
                    check(L.skt_plan_window_build(_ptr(self.plan_indptr), _ptr(self.plan_rows), self.output_dim,
                                                  m, w.value, _ptr(pos), _ptr(wpi), _stream_ptr(self.device)))
                self._window = cached = (w.value, pos, wpi)
            return cached

    def cta_plan(self, d: int):
        """Plan of the window gather kernel (csrc/csr_cta.cuh): ``(W, wrows,
        wpi)`` -- rows per window, the rows of every window stably sorted by
        bucket (sign in bit 31) and every bucket's first rank per window -- or
        None when (t, d) is outside the kernel's range.  Cached."""
        L = _lib.lib()
        m = self.row_end - self.row_begin
        w, nwin = ctypes.c_int32(), ctypes.c_int32()
        with torch.cuda.device(self.device):
            check(L.skt_csr_cta_config(m, self.output_dim, d, ctypes.byref(w), ctypes.byref(nwin)))
        if w.value == 0:
            return None
        with self._plan_lock:
            cached = getattr(self, "_cta_plan", None)
            if cached is None or cached[0] != w.value:
                pos = torch.empty(m, dtype=torch.int32, device=self.device)
                wrows = torch.empty(m, dtype=torch.int32, device=self.device)
                wpi = torch.empty((nwin.value, self.output_dim + 1), dtype=torch.int32, device=self.device)
                with torch.cuda.device(self.device):
                    st = _stream_ptr(self.device)
                    check(L.skt_plan_window_build(_ptr(self.plan_indptr), _ptr(self.plan_rows), self.output_dim,
                                                  m, w.value, _ptr(pos), _ptr(wpi), st))
                    check(L.skt_plan_window_rows(_ptr(pos), m, w.value, _ptr(wrows), st))
                self._cta_plan = cached = (w.value, wrows, wpi)
                self._cta_plan_ws = pos  # alive until the stream has consumed it
            return cached

    def _window_mode(self, indptr, indices, vals) -> str:
        """Which row-window CSR kernel takes this input: ``SKT_CSR_WINDOW`` =
        ``cta`` (window gather, csr_cta.cuh), ``1`` (slot ring through L2,
        csr_window.cuh) or unset / ``0`` (the per-bucket kernels).  Both take
        fp32 values and int32 column indices."""
        mode = os.environ.get("SKT_CSR_WINDOW", "0")
        if mode not in ("1", "cta") or self.row_end - self.row_begin <= 0:
            return ""
        if vals.dtype != torch.float32 or indices.dtype != torch.int32:
            return ""
        if mode == "1" and any(x.data_ptr() % 16 for x in (vals, indices, indptr)):
            return ""
        return mode

    def _window_eligible(self, indptr, indices, vals, d: int, nnz: int) -> bool:
        return self._window_mode(indptr, indices, vals) != ""

    def _apply_csr_cta(self, plan, indptr, indices, vals, d: int, out):
        w, wrows, wpi = plan
        with torch.cuda.device(self.device):
            check(
                _lib.lib().skt_apply_csr_cta(
                    _ptr(wrows), _ptr(wpi), w, self.output_dim, self.row_end - self.row_begin, _ptr(indptr),
                    _ITYPE[indptr.dtype], _ptr(indices), _ptr(vals), vals.numel(), d, _ptr(out),
                    _TORCH_TO_SKT[out.dtype], max(out.stride(0), 1), _stream_ptr(self.device),
                )
            )
        return out

    def _apply_csr_window(self, plan, indptr, indices, vals, d: int, out):
        L = _lib.lib()
        w, pos, wpi = plan
        m = self.row_end - self.row_begin
        nb = ctypes.c_size_t()
        check(L.skt_apply_csr_window_workspace(m, w, ctypes.byref(nb)))
        ws = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            check(
                L.skt_apply_csr_window(
                    _ptr(pos), _ptr(wpi), w, self.output_dim, m, _ptr(indptr), _ITYPE[indptr.dtype],
                    _ptr(indices), _ptr(vals), vals.numel(), d, _ptr(out), _TORCH_TO_SKT[out.dtype],
                    max(out.stride(0), 1), _ptr(ws), nb.value, _stream_ptr(self.device),
                )
            )
        return out

    def csr_group_shift(self, d: int, canonical: bool, nnz: int | None = None) -> int:
        """Plan granularity for the CSR kernels.  Short canonical rows (mean
        <= 8 nonzeros) use the grouped sweep: 2^shift buckets per warp, about
        one warp per group across the chip (148 SMs x 32 warps), group
        accumulators <= 24 KB.  Everything else sweeps the per-bucket plan."""
        m = self.row_end - self.row_begin
        if not canonical or nnz is None or m == 0 or os.environ.get("SKT_CSR_KERNEL") in ("lane", "tile"):
            return 0
        if os.environ.get("SKT_CSR_SHIFT"):  # A/B override
            return int(os.environ["SKT_CSR_SHIFT"])
        if nnz > 8 * m:
            return 0
        shift, resident = 0, 148 * 32
        while shift < 8 and (self.output_dim >> shift) > resident and (2 << shift) * d * 8 <= 24 * 1024:
            shift += 1
        return shift

    # ---- host views (lazy; for API / test compatibility) -------------------
    @property
    def bucket(self) -> np.ndarray:
        if self._bucket is None:
            self._bucket = self.h.cpu().numpy().view(np.uint32).astype(np.int64)
        return self._bucket

    @property
    def sign(self) -> np.ndarray:
        if self._sign is None:
            self._sign = self.s.cpu().numpy().astype(np.float64)
        return self._sign

    @property
    def _mat(self) -> sp.csr_array:
        """S as a t x n scipy CSR, read back from the device plan."""
        if self._mat_cache is None:
            rows = self.plan_rows.cpu().numpy().view(np.uint32)
            indices = (rows & 0x7FFFFFFF).astype(np.int32) + self.row_begin
            data = np.where(rows >> 31, -1.0, 1.0)
            indptr = self.plan_indptr.cpu().numpy()
            self._mat_cache = sp.csr_array(
                (data, indices, indptr), shape=(self.output_dim, self.input_dim)
            )
        return self._mat_cache

    def descriptor(self) -> dict:
        return {"family": self.family, "n": self.input_dim, "t": self.output_dim, "seed": self.seed}

    # ---- apply -------------------------------------------------------------
    def _check_shard_rows(self, nrows: int) -> None:
        want = self.row_end - self.row_begin
        if nrows != want:
            raise ValueError(f"operator expects {want} rows, got {nrows}")

    def apply(self, a, out_dtype=None, check_finite: bool = True, deterministic: bool = True):
        """S @ a (sketch.py:153-165).  Returns float64 unless ``out_dtype``.

        numpy / scipy input -> new numpy array; torch input -> torch tensor on
        the input's device (CPU tensors are staged through the GPU).
        ``deterministic=False`` lets sparse input use unordered atomics (equal
        to the reference up to rounding, not bit-for-bit).
        """
        if self.row_begin == 0 and self.row_end == self.input_dim:
            self._check_rows(a)
        else:
            self._check_shard_rows(a.shape[0])
        if isinstance(a, torch.Tensor):
            out_t = torch.float64 if out_dtype is None else out_dtype
            if a.layout == torch.sparse_csr:
                parts = (a.crow_indices(), a.col_indices(), a.values())
                if not a.is_cuda:
                    parts = tuple(x.to(self.device, non_blocking=True) for x in parts)
                res = self._apply_csr_device(*parts, a.shape[1], out_t,
                                             canonical=csr_is_canonical_device(parts[0], parts[1], a.shape[0]),
                                             deterministic=deterministic)
                return res if a.is_cuda else _host(res)
            if a.is_cuda:
                return self._apply_dense_device(a, out_t, check_finite)
            dev_a = a.to(self.device, non_blocking=a.is_pinned())
            return _host(self._apply_dense_device(dev_a, out_t, check_finite))
        out_t = torch.float64 if out_dtype is None else out_dtype
        if sp.issparse(a):
            m = a if a.format == "csr" else sp.csr_array(a)
            if m.data.dtype not in (np.float32, np.float64):
                m = sp.csr_array(m, dtype=np.float64)
            dev = self.device
            ip, ix, vv = (_to_device(x, dev) for x in (m.indptr, m.indices, m.data))
            # canonical form: scipy's cached flag when it has one (set by its
            # conversions), else checked on the device (scipy's
            # has_canonical_format is an O(nnz) host scan on every new object)
            known = getattr(m, "_has_canonical_format", None)
            if known is None:
                known = csr_is_canonical_device(ip, ix, m.shape[0])
                m.has_canonical_format = known  # cached on the object, as scipy's own check does
            canonical = bool(known)
            return _host(self._apply_csr_device(ip, ix, vv, m.shape[1], out_t, canonical,
                                                deterministic=deterministic)).numpy()
        arr = np.asarray(a)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        if arr.ndim == 1:
            arr = arr.reshape(-1, 1)
        if arr.ndim != 2:
            raise ValueError(f"matrix must be 2-D, got shape {arr.shape}")
        dev_a = _to_device(arr, self.device)
        return _host(self._apply_dense_device(dev_a, out_t, check_finite)).numpy()

    def _apply_dense_device(self, a: torch.Tensor, out_dtype, check_finite=True, out=None, buckets=None,
                            flag=None):
        """K3 on a device tensor.  ``buckets=(b0, b1)`` computes only SA rows
        [b0, b1) (the multi-GPU pipeline reduces finished bucket ranges while
        the next range is computed).  ``flag`` (a 1-element int32 device
        tensor) receives the fused non-finite scan without a host sync -- the
        caller checks it (once, after a batch of calls); otherwise
        ``check_finite`` syncs and raises ValueError like as_dense
        (_validation.py:25-26)."""
        if a.device != self.device:
            raise ValueError(f"input on {a.device}, operator on {self.device}")
        a = dense_operand(a)
        n, d = a.shape
        lda = max(a.stride(0), d, 1) if n > 1 else max(d, 1)
        if out is None:
            out = torch.empty((self.output_dim, d), dtype=out_dtype, device=self.device)
        sync_check = check_finite and flag is None
        if sync_check:
            flag = torch.empty(1, dtype=torch.int32, device=self.device)
        b0, b1 = (0, self.output_dim) if buckets is None else (int(buckets[0]), int(buckets[1]))
        if not (0 <= b0 < b1 <= self.output_dim):
            raise ValueError(f"bad bucket range {buckets!r}")
        with torch.cuda.device(self.device):
            check(
                _lib.lib().skt_apply_dense(
                    _ptr(self.plan_indptr) + 8 * b0, _ptr(self.plan_rows), b1 - b0, n, _ptr(a),
                    _TORCH_TO_SKT[a.dtype], d, lda, _ptr(out) + b0 * out.stride(0) * out.element_size(),
                    _TORCH_TO_SKT[out.dtype], out.stride(0) if d > 0 else 1, _ptr(flag),
                    _stream_ptr(self.device),
                )
            )
        if sync_check and d > 0 and int(flag.item()) != 0:
            raise ValueError("matrix contains non-finite entries")
        return out

    # widest d the shared-memory CSR kernels accumulate on chip (fp64 per warp)
    _CSR_SMEM_MAX_D = (200 * 1024 - 3328) // 8

    def _apply_csr_device(self, indptr, indices, vals, d: int, out_dtype, canonical: bool, out=None,
                          shift=None, deterministic: bool = True, buckets=None):
        """K4 on device CSR arrays.  ``buckets=(b0, b1)`` computes only SA rows
        [b0, b1) (bucket-ownership sharding); the returned tensor is the full
        t x d ``out`` with those rows written."""
        if vals.dtype not in _TORCH_TO_SKT:
            vals = vals.to(torch.float64)
        if out is None:
            out = torch.empty((self.output_dim, d), dtype=out_dtype, device=self.device)
        b0, b1 = (0, self.output_dim) if buckets is None else (int(buckets[0]), int(buckets[1]))
        if not (0 <= b0 < b1 <= self.output_dim):
            raise ValueError(f"bad bucket range {buckets!r}")
        if deterministic and canonical and d > self._CSR_SMEM_MAX_D:
            # wide SA rows (config 5): entries ordered by 1024-column block, then a warp per
            # (bucket, block) adds in row order into shared-memory fp64 accumulators; no atomics
            return self._apply_csr_wide(indptr, indices, vals, d, out, b0, b1)
        if shift is None and deterministic and canonical and b0 == 0 and b1 == self.output_dim and d > 0:
            mode = self._window_mode(indptr, indices, vals)
            if mode == "cta":  # opt-in: window gather, buckets owned by SMs (csr_cta.cuh)
                plan = self.cta_plan(d)
                if plan is not None:
                    return self._apply_csr_cta(plan, indptr, indices, vals, d, out)
            elif mode == "1":  # opt-in: A streamed once in row order (csr_window.cuh)
                plan = self.window_plan(d)
                if plan is not None:
                    try:
                        return self._apply_csr_window(plan, indptr, indices, vals, d, out)
                    except _lib.SketchError as e:
                        if "status 3" not in str(e):  # SKT_ENOTSUP: CTAs not co-resident -> default kernel
                            raise
        if shift is None:
            shift = self.csr_group_shift(d, canonical, vals.numel()) if deterministic else 0
        if b0 % (1 << shift):
            shift = 0  # a grouped plan serves ranges starting on a group boundary
        gptr, grows, gblo = self.grouped_plan(shift)
        flags = (_lib.SKT_CSR_CANONICAL if canonical else 0) | (0 if deterministic else _lib.SKT_CSR_FAST)
        with torch.cuda.device(self.device):
            check(
                _lib.lib().skt_apply_csr(
                    _ptr(gptr) + 8 * (b0 >> shift), _ptr(grows), _ptr(gblo), shift, b1 - b0,
                    self.row_end - self.row_begin, _ptr(indptr), _ITYPE[indptr.dtype], _ptr(indices),
                    _ITYPE[indices.dtype], _ptr(vals), _TORCH_TO_SKT[vals.dtype], vals.numel(), d,
                    _ptr(out) + b0 * out.stride(0) * out.element_size(), _TORCH_TO_SKT[out.dtype], max(d, 1),
                    flags, _stream_ptr(self.device),
                )
            )
        return out

    def _apply_csr_wide(self, indptr, indices, vals, d: int, out, b0: int, b1: int):
        """skt_apply_csr_wide: rows [b0, b1) of SA for canonical CSR A with
        wide rows (csrc/csr_fine.cuh); writes ``out`` directly in its dtype."""
        L = _lib.lib()
        m = self.row_end - self.row_begin
        nb = ctypes.c_size_t()
        check(L.skt_apply_csr_wide_workspace(m, b1 - b0, d, vals.numel(), _TORCH_TO_SKT[vals.dtype], ctypes.byref(nb)))
        ws = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            check(
                L.skt_apply_csr_wide(
                    _ptr(self.plan_indptr) + 8 * b0, _ptr(self.plan_rows), b1 - b0, m, _ptr(indptr),
                    _ITYPE[indptr.dtype], _ptr(indices), _ITYPE[indices.dtype], _ptr(vals),
                    _TORCH_TO_SKT[vals.dtype], vals.numel(), d,
                    _ptr(out) + b0 * out.stride(0) * out.element_size(), _TORCH_TO_SKT[out.dtype],
                    max(d, 1), _ptr(ws), nb.value, _stream_ptr(self.device),
                )
            )
        return out

    # ---- column sketch: A @ S^T (sketch.py:445-448), transpose-free ---------
    def apply_right(self, a, out_dtype=None):
        if self.row_begin != 0 or self.row_end != self.input_dim:
            raise ValueError("apply_right needs the full operator")
        out_t = torch.float64 if out_dtype is None else out_dtype
        L = _lib.lib()
        dev = self.device
        to_numpy = not isinstance(a, torch.Tensor)
        if sp.issparse(a) or (isinstance(a, torch.Tensor) and a.layout == torch.sparse_csr):
            if isinstance(a, torch.Tensor):
                ip, ix, vv = (x.to(dev) for x in (a.crow_indices(), a.col_indices(), a.values()))
                n_rows, ncols = a.shape
            else:
                m = sp.csr_array(a)
                if m.data.dtype not in (np.float32, np.float64):
                    m = sp.csr_array(m, dtype=np.float64)
                if not m.has_sorted_indices:
                    m = m.copy()
                    m.sort_indices()
                n_rows, ncols = m.shape
                ip, ix, vv = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (m.indptr, m.indices, m.data))
            if ncols != self.input_dim:
                raise ValueError(f"operator expects {self.input_dim} rows, got {ncols}")
            if vv.dtype not in _TORCH_TO_SKT:
                vv = vv.to(torch.float64)
            y = torch.empty((n_rows, self.output_dim), dtype=out_t, device=dev)
            with torch.cuda.device(dev):
                check(
                    L.skt_apply_right_csr(
                        _ptr(self.h), _ptr(self.s), self.output_dim, n_rows, ncols, _ptr(ip),
                        _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype], _ptr(vv), _TORCH_TO_SKT[vv.dtype],
                        _ptr(y), _TORCH_TO_SKT[out_t], self.output_dim, _stream_ptr(dev),
                    )
                )
        else:
            if isinstance(a, torch.Tensor):
                x = a.to(dev)
            else:
                arr = np.asarray(a)
                if arr.dtype not in (np.float32, np.float64):
                    arr = arr.astype(np.float64)
                if arr.ndim == 1:
                    arr = arr.reshape(-1, 1)
                x = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
            if x.dtype not in _TORCH_TO_SKT:
                x = x.to(torch.float64)
            if x.dim() == 1:
                x = x.reshape(-1, 1)
            x = x.contiguous()
            n_rows, ncols = x.shape
            if ncols != self.input_dim:
                raise ValueError(f"operator expects {self.input_dim} rows, got {ncols}")
            y = torch.empty((n_rows, self.output_dim), dtype=out_t, device=dev)
            flag = torch.empty(1, dtype=torch.int32, device=dev)
            with torch.cuda.device(dev):
                check(
                    L.skt_apply_right_dense(
                        _ptr(self.h), _ptr(self.s), self.output_dim, n_rows, ncols, _ptr(x),
                        _TORCH_TO_SKT[x.dtype], max(ncols, 1), _ptr(y), _TORCH_TO_SKT[out_t],
                        self.output_dim, _ptr(flag), _stream_ptr(dev),
                    )
                )
            if n_rows > 0 and int(flag.item()) != 0:
                raise ValueError("matrix contains non-finite entries")
        if to_numpy:
            return _host(y).numpy()
        return y if (isinstance(a, torch.Tensor) and a.is_cuda) else _host(y)


class ComposedSketch(SketchOperator):
    """sketch.py:372-396: outer @ inner; apply runs inner first."""

    family = "composed"

    def __init__(self, outer, inner):
        if outer.input_dim != inner.output_dim:
            raise ValueError(
                f"cannot compose: outer expects {outer.input_dim} rows, "
                f"inner produces {inner.output_dim}"
            )
        self.outer, self.inner = outer, inner
        self.input_dim, self.output_dim = inner.input_dim, outer.output_dim

    def apply(self, a):
        return self.outer.apply(self.inner.apply(a))

    def descriptor(self) -> dict:
        return {"family": self.family, "outer": self.outer.descriptor(), "inner": self.inner.descriptor()}


def make_sparse_embedding(n: int, t: int, seed: int) -> SparseEmbedding:
    """sketch.py:399-400."""
    return SparseEmbedding(n, t, seed)


def sparse_embedding_or_identity(n: int, t: int, seed: int):
    """sketch.py:422-426: the identity when t >= n."""
    if t >= n:
        return IdentityOperator(n)
    return SparseEmbedding(n, t, seed)


def compose(outer, inner) -> ComposedSketch:
    return ComposedSketch(outer, inner)


def apply_left(s, a):
    """sketch.py:440-442."""
    return s.apply(a)


def apply_right(a, s):
    """sketch.py:445-448: A @ S^T.  Transpose-free on the GPU for SparseEmbedding;
    other operator families keep the reference formula (S @ A^T)^T."""
    if isinstance(s, SparseEmbedding):
        return s.apply_right(a)
    if getattr(s, "family", None) == "composed" and isinstance(getattr(s, "inner", None), SparseEmbedding):
        # (outer inner A^T)^T = apply_right(A inner^T, outer): the sparse
        # embedding's column sketch stays transpose-free on the GPU
        y = s.inner.apply_right(a)
        return apply_right(y, s.outer)
    if sp.issparse(a):
        at = a.T
    else:
        at = np.asarray(a, dtype=np.float64)
        if at.ndim == 1:
            at = at.reshape(-1, 1)
        at = at.T
    return s.apply(at).T


def to_descriptor(s) -> dict:
    return s.descriptor()


def from_descriptor(d: dict):
    """sketch.py:460-478 for every family this package owns: the sparse
    embedding, the generalized embedding and the SRHT come back as this
    package's GPU classes.  The leverage sampler and Gaussian JL are other
    sketch families outside the hot path; they raise instead of
    silently running the reference's CPU code."""
    family = d.get("family")
    if family == "identity":
        return IdentityOperator(d["n"])
    if family == "sparse":
        return SparseEmbedding(d["n"], d["t"], d["seed"])
    if family == "generalized":
        from .generalized import GeneralizedSparseEmbedding  # noqa: PLC0415 (import cycle)

        return GeneralizedSparseEmbedding(d["n"], d["r"], d["eps"], d["delta"], d["seed"])
    if family == "srht":
        from .solvers import SrhtOperator  # noqa: PLC0415 (import cycle)

        return SrhtOperator(d["n"], d["t"], d["seed"], all_rows=d.get("all_rows", False))
    if family == "composed":
        return ComposedSketch(from_descriptor(d["outer"]), from_descriptor(d["inner"]))
    if family in ("leverage", "gaussian"):
        raise ValueError(
            f"sketch family {family!r} is not provided by this package (outside the "
            "CountSketch hot path); build it with sketchnla.sketch.from_descriptor"
        )
    raise ValueError(f"unknown sketch family {family!r}")
