"""Matrix Market ingest feeding device CSR (reference io.py:37-104,
load_matrix_market; §8f rank 4).

The coordinate entries are parsed natively on all host cores
(csrc/mm_ingest.cpp: mmapped file split at line boundaries, count pass,
prefix sum, parse pass; the reference's "path:line: reason" errors) and
canonicalised on the GPU (csrc/coo_csr.cu: stable (row, col) sort with the
plan builder, duplicates summed, zero sums dropped) -- the reference's
as_csr(coo) contract, with the CSR left on the device for S.A.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from ._lib import SktMmInfo
from .sketch import _host, _ptr, _stream_ptr


class MatrixMarketError(ValueError):
    """Raised for malformed or unsupported Matrix Market input (io.py:17-18)."""


def _check_mm(status: int) -> None:
    if status != 0:
        msg = _lib.last_error()
        if status == 1:
            raise MatrixMarketError(msg)
        raise _lib.SketchError(msg)


def read_coo(path, n_threads: int = 0):
    """Parse a coordinate .mtx on the host: (shape, rows, cols, vals), 0-based,
    symmetric storage expanded, in the reference's entry order."""
    L = _lib.lib()
    p = os.fsencode(str(path))
    info = SktMmInfo()
    _check_mm(L.skt_mm_probe(p, ctypes.byref(info)))
    cap = info.n_entries * (2 if info.symmetric else 1)
    rows = torch.empty(cap, dtype=torch.int64, pin_memory=torch.cuda.is_available())
    cols = torch.empty(cap, dtype=torch.int64, pin_memory=torch.cuda.is_available())
    vals = torch.empty(cap, dtype=torch.float64, pin_memory=torch.cuda.is_available())
    count = ctypes.c_int64()
    _check_mm(L.skt_mm_read_coo(p, cap, _ptr(rows), _ptr(cols), _ptr(vals), ctypes.byref(count), int(n_threads)))
    k = count.value
    return (int(info.n_rows), int(info.n_cols)), rows[:k], cols[:k], vals[:k]


def load_matrix_market_device(path, device=None, n_threads: int = 0):
    """Coordinate .mtx -> canonical CSR on the GPU: (indptr int64, indices
    int32, values fp64) torch tensors and the shape."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    (n_rows, n_cols), rows, cols, vals = read_coo(path, n_threads)
    L = _lib.lib()
    count = rows.numel()
    with torch.cuda.device(device):
        stream = _stream_ptr(device)
        r = rows.to(device, non_blocking=True)
        c = cols.to(device, non_blocking=True)
        v = vals.to(device, non_blocking=True)
        indptr = torch.empty(n_rows + 1, dtype=torch.int64, device=device)
        indices = torch.empty(max(count, 1), dtype=torch.int32, device=device)
        out = torch.empty(max(count, 1), dtype=torch.float64, device=device)
        nnz = torch.zeros(1, dtype=torch.int64, device=device)
        bad = torch.zeros(1, dtype=torch.int32, device=device)
        wsb = ctypes.c_size_t()
        _lib.check(L.skt_coo_to_csr_workspace(count, n_rows, n_cols, ctypes.byref(wsb)))
        ws = torch.empty(max(wsb.value, 8), dtype=torch.uint8, device=device)
        _lib.check(L.skt_coo_to_csr(_ptr(r), _ptr(c), _ptr(v), count, n_rows, n_cols, _ptr(indptr), _ptr(indices),
                                    _ptr(out), _ptr(nnz), _ptr(bad), _ptr(ws), wsb.value, stream))
        k = int(nnz.item())
        if int(bad.item()) != 0:  # as_csr(coo, path) (io.py:103, _validation.py:39-40)
            raise ValueError(f"{path} contains non-finite entries")
    return (n_rows, n_cols), indptr, indices[:k], out[:k]


def load_matrix_market(path, device=None, n_threads: int = 0) -> sp.csr_array:
    """io.py:37-104: a coordinate .mtx as canonical scipy CSR (built on the GPU)."""
    shape, indptr, indices, values = load_matrix_market_device(path, device, n_threads)
    return sp.csr_array((_host(values).numpy(), _host(indices).numpy(), _host(indptr).numpy()), shape=shape)


def as_torch_csr(shape, indptr, indices, values) -> torch.Tensor:
    """The device CSR as a torch sparse_csr tensor (accepted by SparseEmbedding.apply)."""
    return torch.sparse_csr_tensor(indptr, indices, values, size=shape)


__all__ = ["MatrixMarketError", "read_coo", "load_matrix_market", "load_matrix_market_device", "as_torch_csr"]
