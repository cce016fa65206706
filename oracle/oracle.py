"""CPU oracle for the CountSketch hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module; it
is the checker, never the thing measured on the GPU path or shipped.  The
product package ``paper_1207_6365_b200`` has no import of it and no CPU
fallback.

Two restatements of the reference (``/root/reference/pkg/src/sketchnla``):

* ``liboracle_skt.so`` (``skt_oracle.c``): scalar C restatement of numpy's
  SeedSequence + PCG64 + bounded-integer draws (sketch.py:51-53,147-148), the
  counting-sort plan (sketch.py:149-151), and the two apply branches
  (sketch.py:155-165), all sequential fp64.
* numpy/scipy restatements below (``np_*``): the same algorithm written with
  the reference's own primitives (``bincount`` for CSR, scipy CSR @ dense for
  dense, ``csr @ probe`` + einsum for the leverage contraction); this is the
  "reference CPU path" timed by ``bench.py --impl reference``.

Pinned against the reference itself by ``tests/golden/make_golden.py``
(reference imported in the build container) and ``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_skt.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "skt_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
        L.oracle_seedseq_generate.argtypes = [P, i32, P, i32, P, i32]
        L.oracle_pcg64_seed.argtypes = [P, i32, P, i32, P]
        L.oracle_pcg64_raw.argtypes = [P, i64, P]
        L.oracle_hash_signs.argtypes = [P, P, i64, u64, P, P]
        L.oracle_plan.argtypes = [P, i64, i64, P, P]
        L.oracle_apply_dense.argtypes = [P, P, P, i64, P, i32, i64, i64, P]
        L.oracle_apply_csr.argtypes = [P, P, i64, i64, P, P, P, i32, i64, P]
        L.oracle_lev_rownorms_csr.argtypes = [i64, P, P, P, i32, P, i64, P]
        L.oracle_apply_dense_mt.argtypes = [P, P, P, i64, P, i32, i64, i64, P, i32]
        L.oracle_apply_csr_mt.argtypes = [P, P, P, i64, P, P, P, i32, i64, P, i32]
        L.oracle_lev_rownorms_csr_mt.argtypes = [i64, P, P, P, i32, P, i64, P, i32]
        for f in ("oracle_apply_dense_mt", "oracle_apply_csr_mt", "oracle_lev_rownorms_csr_mt"):
            getattr(L, f).restype = i32
        for f in ("oracle_seedseq_generate", "oracle_pcg64_seed", "oracle_hash_signs"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def int_to_words(x: int) -> np.ndarray:
    """numpy's _coerce_to_uint32_array for a non-negative Python int."""
    x = int(x)
    if x < 0:
        raise ValueError("expected non-negative integer")
    words = []
    while True:
        words.append(x & 0xFFFFFFFF)
        x >>= 32
        if x == 0:
            break
    return np.asarray(words, dtype=np.uint32)


def seedseq_generate(seed: int, spawn_key=(), n_words: int = 4) -> np.ndarray:
    ent = int_to_words(seed)
    sk = np.asarray([int(k) for k in spawn_key], dtype=np.uint32)
    out = np.zeros(n_words, dtype=np.uint32)
    rc = lib().oracle_seedseq_generate(_ptr(ent), len(ent), _ptr(sk), len(sk), _ptr(out), n_words)
    assert rc == 0
    return out


def pcg64_seed(seed: int, spawn_key=()) -> np.ndarray:
    """(state_hi, state_lo, inc_hi, inc_lo) of PCG64(SeedSequence(seed, spawn_key))."""
    ent = int_to_words(seed)
    sk = np.asarray([int(k) for k in spawn_key], dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint64)
    assert lib().oracle_pcg64_seed(_ptr(ent), len(ent), _ptr(sk), len(sk), _ptr(out)) == 0
    return out


def pcg64_raw(state: np.ndarray, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().oracle_pcg64_raw(_ptr(np.ascontiguousarray(state, dtype=np.uint64)), n, _ptr(out))
    return out


def hash_signs(n: int, t: int, seed: int):
    """(bucket uint32[n], sign int8[n]) exactly as SparseEmbedding(n, t, seed)."""
    hs = pcg64_seed(seed, (0, 0))
    ss = pcg64_seed(seed, (0, 1))
    h = np.zeros(n, dtype=np.uint32)
    s = np.zeros(n, dtype=np.int8)
    rc = lib().oracle_hash_signs(_ptr(hs), _ptr(ss), n, t, _ptr(h), _ptr(s))
    if rc != 0:
        raise ValueError("bad (n, t)")
    return h, s


def plan(h: np.ndarray, t: int):
    """S in CSR: (indptr int64[t+1], rows int32[n]) -- stable counting sort."""
    h = np.ascontiguousarray(h, dtype=np.uint32)
    indptr = np.zeros(t + 1, dtype=np.int64)
    rows = np.zeros(len(h), dtype=np.int32)
    lib().oracle_plan(_ptr(h), len(h), t, _ptr(indptr), _ptr(rows))
    return indptr, rows


def _threads(threads: int) -> int:
    """0 = every core this process may run on."""
    if threads and threads > 0:
        return int(threads)
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def apply_dense(h, s, t: int, a: np.ndarray, threads: int = 1) -> np.ndarray:
    """Dense branch; ``threads != 1`` splits the buckets over host threads
    (bit-identical: each SA element is summed by one thread in row order)."""
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    a = np.ascontiguousarray(a)
    indptr, rows = plan(h, t)
    d = a.shape[1]
    out = np.zeros((t, d), dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.int8)
    if threads == 1:
        lib().oracle_apply_dense(
            _ptr(indptr), _ptr(rows), _ptr(s), t, _ptr(a), int(a.dtype == np.float32), d, d, _ptr(out)
        )
    else:
        rc = lib().oracle_apply_dense_mt(
            _ptr(indptr), _ptr(rows), _ptr(s), t, _ptr(a), int(a.dtype == np.float32), d, d, _ptr(out),
            _threads(threads),
        )
        assert rc == 0, "pthread_create failed"
    return out


def _csr_parts(a):
    a = sp.csr_array(a)
    if a.data.dtype not in (np.float32, np.float64):
        a = sp.csr_array(a, dtype=np.float64)
    indptr = np.ascontiguousarray(a.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(a.indices, dtype=np.int32)
    vals = np.ascontiguousarray(a.data)
    return a.shape, indptr, indices, vals


def apply_csr(h, s, t: int, a, threads: int = 1) -> np.ndarray:
    """CSR branch; ``threads != 1`` walks each bucket's rows (the plan) on
    its own thread -- per element the same order as the nnz-order bincount."""
    (n, d), indptr, indices, vals = _csr_parts(a)
    out = np.zeros((t, d), dtype=np.float64)
    hh = np.ascontiguousarray(h, dtype=np.uint32)
    ss = np.ascontiguousarray(s, dtype=np.int8)
    if threads == 1:
        lib().oracle_apply_csr(
            _ptr(hh), _ptr(ss), n, t, _ptr(indptr), _ptr(indices), _ptr(vals), int(vals.dtype == np.float32), d,
            _ptr(out),
        )
    else:
        pptr, prow = plan(hh, t)
        rc = lib().oracle_apply_csr_mt(
            _ptr(pptr), _ptr(prow), _ptr(ss), t, _ptr(indptr), _ptr(indices), _ptr(vals),
            int(vals.dtype == np.float32), d, _ptr(out), _threads(threads),
        )
        assert rc == 0, "pthread_create failed"
    return out


def apply(h, s, t: int, a) -> np.ndarray:
    """SparseEmbedding.apply restated (sketch.py:153-165)."""
    if sp.issparse(a):
        return apply_csr(h, s, t, a)
    return apply_dense(h, s, t, a)


def lev_rownorms_csr(a, p: np.ndarray, threads: int = 1) -> np.ndarray:
    (n, d), indptr, indices, vals = _csr_parts(a)
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.zeros(n, dtype=np.float64)
    args = (n, _ptr(indptr), _ptr(indices), _ptr(vals), int(vals.dtype == np.float32), _ptr(p), p.shape[1],
            _ptr(out))
    if threads == 1:
        lib().oracle_lev_rownorms_csr(*args)
    else:
        assert lib().oracle_lev_rownorms_csr_mt(*args, _threads(threads)) == 0, "pthread_create failed"
    return out


# ---------------------------------------------------------------------------
# numpy / scipy restatement: the reference CPU path with its own primitives.
# ---------------------------------------------------------------------------


def np_sketch_matrix(h, s, t: int, n: int):
    """_mat of sketch.py:149-151 (scipy COO->CSR: stable by bucket)."""
    return sp.csr_array(
        (np.asarray(s, dtype=np.float64), (np.asarray(h, dtype=np.int64), np.arange(n))),
        shape=(t, n),
    )


def np_apply_dense(mat, a: np.ndarray) -> np.ndarray:
    """sketch.py:165: as_dense (fp64 upcast + finiteness scan) then CSR @ dense."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix contains non-finite entries")
    return np.asarray(mat @ a, dtype=np.float64)


def np_apply_csr(h, s, t: int, a) -> np.ndarray:
    """sketch.py:155-164: repeat + bincount scatter."""
    a = sp.csr_array(a)
    d = a.shape[1]
    counts = np.diff(a.indptr)
    flat = np.repeat(np.asarray(h, dtype=np.int64) * d, counts) + a.indices
    weights = np.repeat(np.asarray(s, dtype=np.float64), counts) * a.data
    return np.bincount(flat, weights=weights, minlength=t * d).reshape(t, d)


def np_lev_rownorms(a, probe: np.ndarray) -> np.ndarray:
    """leverage.py:90-91."""
    rows = np.asarray(a @ probe)
    return np.einsum("ij,ij->i", rows, rows)


def residual_fro(a, x, b) -> float:
    """||a @ x - b||_F exactly as regress.py:79-80 (_residual_fro) computes it:
    the reference's own numpy / scipy product, then the Frobenius norm."""
    return float(np.linalg.norm(np.asarray(a @ x) - b, "fro"))


def srht_apply(a: np.ndarray, t: int, seed: int) -> np.ndarray:
    """SrhtOperator(n, t, seed).apply(a) restated (sketch.py:241-252 _fwht,
    sketch.py:266-291 __init__ / apply): zero-pad to n_pad = 2^ceil(log2 n),
    sign flip from stream (2, 0), unnormalised Walsh-Hadamard along rows, t rows
    sampled from stream (2, 1), scaled by sqrt(n_pad/t)/sqrt(n_pad)."""
    import math

    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    n = a.shape[0]
    n_pad = 1 << (n - 1).bit_length()
    rng = lambda k: np.random.default_rng(np.random.SeedSequence(int(seed), spawn_key=(2, k)))  # noqa: E731
    sign = rng(0).choice(np.array([-1.0, 1.0]), size=n_pad)
    rows = rng(1).integers(0, n_pad, size=t)
    scale = math.sqrt(n_pad / t) / math.sqrt(n_pad)
    out = np.zeros((n_pad, a.shape[1]))
    out[:n] = a
    out *= sign[:, None]
    h = 1
    while h < n_pad:
        out = out.reshape(n_pad // (2 * h), 2, h, -1)
        out = np.stack((out[:, 0] + out[:, 1], out[:, 0] - out[:, 1]), axis=1).reshape(n_pad, -1)
        h *= 2
    return scale * out[rows]


def gse_operator(n: int, r: int, eps: float, delta: float, seed: int):
    """GeneralizedSparseEmbedding's hashes and matrix restated (sketch.py:69-80
    generalized_dims, sketch.py:186-220 __init__): returns (q, k, v, t, outer,
    inner, sign, mat) with mat the t x n scipy CSR the reference multiplies by."""
    import math

    k = max(1, math.ceil(1.0 * math.log(r / (eps * delta)) / eps))
    v = max(1, math.ceil(1.0 / eps))
    q = max(1, math.ceil(1.0 * r * (r + math.log(1.0 / (delta * eps))) / eps**2))
    t = q * k * v
    rng = lambda s: np.random.default_rng(np.random.SeedSequence(int(seed), spawn_key=(1, s)))  # noqa: E731
    outer = rng(0).integers(0, q, size=n)
    inner = rng(1).integers(0, v, size=(k, n))
    sign = rng(2).choice(np.array([-1.0, 1.0]), size=(k, n))
    rows = outer[None, :] * (k * v) + np.arange(k)[:, None] * v + inner
    cols = np.broadcast_to(np.arange(n), (k, n))
    mat = sp.csr_array(((sign / math.sqrt(k)).ravel(), (rows.ravel(), cols.ravel())), shape=(t, n))
    return q, k, v, t, outer, inner, sign, mat


def gse_apply(mat, a) -> np.ndarray:
    """sketch.py:222-227: the reference's own product (scipy csr_matvecs /
    csr_matmat), fp64."""
    out = mat @ a
    if sp.issparse(out):
        out = out.toarray()
    return np.asarray(out, dtype=np.float64)
