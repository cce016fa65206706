"""ctypes binding of the C ABI in ``include/sketch_b200.h`` (libsketch_b200.so).

This is the one place Python touches native code.  There is no CPU fallback:
if the shared library is missing or fails to load, or no CUDA device is
present when a device entry point is called, the call raises.  ctypes releases
the GIL for the duration of each foreign call, so operators may be applied
concurrently from several host threads (the reference CLI's ThreadPoolExecutor,
cli.py:227-231).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKT_LIB_PATH") or os.path.join(_HERE, "libsketch_b200.so")
CSRC = os.path.join(_HERE, "csrc")

SKT_OK, SKT_EINVAL, SKT_ECUDA, SKT_ENOTSUP, SKT_EWORKSPACE = range(5)
SKT_F32, SKT_F64 = 0, 1
SKT_I32, SKT_I64 = 0, 1
SKT_CSR_CANONICAL = 1
SKT_CSR_FAST = 2

# Every symbol include/sketch_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "skt_version",
    "skt_last_error",
    "skt_launch_count",
    "skt_seedseq_generate",
    "skt_pcg64_seed",
    "skt_pcg64_advance",
    "skt_hash_signs_workspace",
    "skt_hash_signs",
    "skt_plan_workspace",
    "skt_plan_build",
    "skt_apply_dense",
    "skt_apply_csr",
    "skt_memcpy_staged",
    "skt_csr_check_sorted",
    "skt_apply_csr_wide_workspace",
    "skt_apply_csr_wide",
    "skt_csr_window_config",
    "skt_plan_window_build",
    "skt_apply_csr_window_workspace",
    "skt_apply_csr_window",
    "skt_csr_cta_config",
    "skt_plan_window_rows",
    "skt_apply_csr_cta",
    "skt_apply_dense_push",
    "skt_slot_sum",
    "skt_apply_right_dense",
    "skt_apply_right_csr",
    "skt_lev_rownorms_csr",
    "skt_lev_rownorms_dense",
    "skt_residual_workspace",
    "skt_residual_dense",
    "skt_residual_csr",
    "skt_lsq_workspace",
    "skt_lsq_residual_grad",
    "skt_lsq_matvec_norm",
    "skt_lsq_update_grad",
    "skt_gemm_dense",
    "skt_spmm_csr",
    "skt_gram_cross_csr",
    "skt_gram_cross_dense",
    "skt_srht_workspace",
    "skt_srht_apply",
    "skt_gse_buckets",
    "skt_gse_fold_rows",
    "skt_gse_apply_dense",
    "skt_gse_apply_csr",
    "skt_mm_probe",
    "skt_mm_read_coo",
    "skt_coo_to_csr_workspace",
    "skt_coo_to_csr",
)


class SktMmInfo(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64),
        ("n_cols", ctypes.c_int64),
        ("n_entries", ctypes.c_int64),
        ("field", ctypes.c_int32),
        ("symmetric", ctypes.c_int32),
    ]


class SktPcg64(ctypes.Structure):
    _fields_ = [
        ("state_hi", ctypes.c_uint64),
        ("state_lo", ctypes.c_uint64),
        ("inc_hi", ctypes.c_uint64),
        ("inc_lo", ctypes.c_uint64),
    ]


class SketchError(RuntimeError):
    """CUDA / unsupported-shape failure reported by the native library."""


def build(verbose: bool = False) -> str:
    """Compile libsketch_b200.so for sm_100a in-tree (nvcc via make)."""
    cmd = ["make", "-C", CSRC, "-j8"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"building libsketch_b200.so failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)"
        )
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u32, u64, sz = (
        ctypes.c_void_p,
        ctypes.c_int32,
        ctypes.c_int64,
        ctypes.c_uint32,
        ctypes.c_uint64,
        ctypes.c_size_t,
    )
    PS = ctypes.POINTER(SktPcg64)
    sig = {
        "skt_version": ([], ctypes.c_char_p),
        "skt_last_error": ([], ctypes.c_char_p),
        "skt_launch_count": ([], u64),
        "skt_seedseq_generate": ([P, i32, P, i32, P, i32], i32),
        "skt_pcg64_seed": ([P, i32, P, i32, PS], i32),
        "skt_pcg64_advance": ([PS, u64], i32),
        "skt_hash_signs_workspace": ([i64, u64, ctypes.POINTER(sz)], i32),
        "skt_hash_signs": ([PS, PS, i64, i64, u64, P, P, P, sz, P], i32),
        "skt_plan_workspace": ([i64, u64, i32, ctypes.POINTER(sz)], i32),
        "skt_plan_build": ([P, P, i64, u64, i32, P, P, P, P, sz, P], i32),
        "skt_apply_dense": ([P, P, u64, i64, P, i32, i64, i64, P, i32, i64, P, P], i32),
        "skt_apply_csr": ([P, P, P, i32, u64, i64, P, i32, P, i32, P, i32, i64, i64, P, i32, i64, u32, P], i32),
        "skt_memcpy_staged": ([P, P, sz, i32, P], i32),
        "skt_csr_check_sorted": ([i64, P, i32, P, i32, P, P], i32),
        "skt_apply_csr_wide_workspace": ([i64, u64, i64, i64, i32, ctypes.POINTER(sz)], i32),
        "skt_apply_csr_wide": ([P, P, u64, i64, P, i32, P, i32, P, i32, i64, i64, P, i32, i64, P, sz, P], i32),
        "skt_csr_window_config": ([i64, u64, i64, ctypes.POINTER(i32), ctypes.POINTER(i32)], i32),
        "skt_plan_window_build": ([P, P, u64, i64, i32, P, P, P], i32),
        "skt_apply_csr_window_workspace": ([i64, i32, ctypes.POINTER(sz)], i32),
        "skt_apply_csr_window": ([P, P, i32, u64, i64, P, i32, P, P, i64, i64, P, i32, i64, P, sz, P], i32),
        "skt_csr_cta_config": ([i64, u64, i64, ctypes.POINTER(i32), ctypes.POINTER(i32)], i32),
        "skt_plan_window_rows": ([P, i64, i32, P, P], i32),
        "skt_apply_csr_cta": ([P, P, i32, u64, i64, P, i32, P, P, i64, i64, P, i32, i64, P], i32),
        "skt_apply_dense_push": ([P, P, u64, i64, P, i32, i64, i64, i32, P, P, i32, i32, i64, i64, i64, P, P], i32),
        "skt_slot_sum": ([P, i32, i32, i64, i64, i64, i64, P, i64, P], i32),
        "skt_apply_right_dense": ([P, P, u64, i64, i64, P, i32, i64, P, i32, i64, P, P], i32),
        "skt_apply_right_csr": ([P, P, u64, i64, i64, P, i32, P, i32, P, i32, P, i32, i64, P], i32),
        "skt_lev_rownorms_csr": ([i64, i64, P, i32, P, i32, P, i32, P, i64, P, i32, P], i32),
        "skt_lev_rownorms_dense": ([i64, i64, P, i32, i64, P, i64, P, i32, P, P], i32),
        "skt_residual_workspace": ([ctypes.POINTER(sz)], i32),
        "skt_residual_dense": ([i64, i64, P, i32, i64, P, i64, P, i32, i64, P, P, sz, P], i32),
        "skt_residual_csr": ([i64, i64, P, i32, P, i32, P, i32, P, i64, P, i32, i64, P, P, sz, P], i32),
        "skt_lsq_workspace": ([i64, ctypes.POINTER(sz)], i32),
        "skt_lsq_residual_grad": ([i64, i64, P, i64, P, P, i64, P, P, P, sz, P], i32),
        "skt_lsq_matvec_norm": ([i64, i64, P, i64, P, P, i64, P, P, sz, P], i32),
        "skt_lsq_update_grad": ([i64, i64, P, i64, P, i64, ctypes.c_double, P, i64, P, P, i64, P, P, P, sz, P], i32),
        "skt_gemm_dense": ([i64, i64, P, i32, i64, P, i64, P, i64, P], i32),
        "skt_spmm_csr": ([i64, i64, P, i32, P, i32, P, i32, i64, P, i64, P, i64, P], i32),
        "skt_gram_cross_csr": ([i64, i64, P, i32, P, i32, P, i32, P, i64, i64, P, i64, P, P, sz, P], i32),
        "skt_gram_cross_dense": ([i64, i64, P, i32, i64, P, i64, i64, P, i64, P, P, sz, P], i32),
        "skt_srht_workspace": ([i64, i64, ctypes.POINTER(sz)], i32),
        "skt_srht_apply": ([P, i64, i64, i64, P, P, i64, ctypes.c_double, P, i64, P, sz, P], i32),
        "skt_gse_buckets": ([P, P, i64, i32, u32, u64, P, P], i32),
        "skt_gse_fold_rows": ([P, i64, i64, P], i32),
        "skt_gse_apply_dense": ([P, P, u64, i64, P, i32, i64, i64, ctypes.c_double, P, i64, P, P], i32),
        "skt_gse_apply_csr": ([P, P, u64, P, i32, P, i32, P, i32, i64, ctypes.c_double, P, i64, P], i32),
        "skt_mm_probe": ([ctypes.c_char_p, ctypes.POINTER(SktMmInfo)], i32),
        "skt_mm_read_coo": ([ctypes.c_char_p, i64, P, P, P, ctypes.POINTER(i64), i32], i32),
        "skt_coo_to_csr_workspace": ([i64, i64, i64, ctypes.POINTER(sz)], i32),
        "skt_coo_to_csr": ([P, P, P, i64, i64, i64, P, P, P, P, P, P, sz, P], i32),
    }
    for name, (argtypes, restype) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = restype
    _lib = L
    return L


def last_error() -> str:
    msg = lib().skt_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status == SKT_OK:
        return
    msg = last_error()
    if status == SKT_EINVAL:
        raise ValueError(msg)
    raise SketchError(f"status {status}: {msg}")


def launch_count() -> int:
    return int(lib().skt_launch_count())
