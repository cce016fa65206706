"""Ceiling study for K3 (dense S.A) on config-3 shapes: the same kernel driven
by (a) the real bucket plan (random 512 B row gathers) and (b) an identity plan
(rows in order, 256 per bucket: sequential streaming), next to torch read-only
and copy bandwidth.  Prints one JSON line.  Not part of the product."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1207_6365_b200 import SparseEmbedding, _lib  # noqa: E402
from paper_1207_6365_b200.sketch import _TORCH_TO_SKT, _ptr  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n, d, t = 16_777_216, 128, 65_536
    dev = torch.device("cuda", 0)
    A = torch.randn((n, d), device=dev, dtype=torch.float32)
    op = SparseEmbedding(n, t, 1, device=dev)
    SA = torch.empty((t, d), device=dev, dtype=torch.float32)
    ident_rows = torch.arange(n, device=dev, dtype=torch.int32)
    ident_ptr = torch.arange(0, n + 1, n // t, device=dev, dtype=torch.int64)
    L = _lib.lib()
    stream = torch.cuda.current_stream().cuda_stream

    def run(indptr, rows):
        L.skt_apply_dense(_ptr(indptr), _ptr(rows), t, n, _ptr(A), _TORCH_TO_SKT[A.dtype], d, d, _ptr(SA),
                          _TORCH_TO_SKT[SA.dtype], d, None, stream)

    nbytes = A.numel() * 4 + SA.numel() * 4
    out = {}
    out["gather_ms"] = timeit(lambda: run(op.plan_indptr, op.plan_rows))
    out["sequential_ms"] = timeit(lambda: run(ident_ptr, ident_rows))
    out["torch_sum_ms"] = timeit(lambda: A.sum(dim=0))
    B = torch.empty_like(A)
    out["torch_copy_ms"] = timeit(lambda: B.copy_(A), reps=10)
    for k in ("gather_ms", "sequential_ms", "torch_sum_ms"):
        out[k.replace("_ms", "_GBps")] = nbytes / (out[k] / 1e3) / 1e9
    out["torch_copy_GBps"] = 2 * A.numel() * 4 / (out["torch_copy_ms"] / 1e3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
