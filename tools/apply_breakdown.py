"""Per-call cost breakdown of SparseEmbedding.apply(scipy CSR) at the sizes of
the reference's acceptance criterion 10 (n = 65536, d = 256, t = 512)."""
import sys
import time

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, ".")
from paper_1207_6365_b200 import make_sparse_embedding  # noqa: E402
from paper_1207_6365_b200.sketch import _host, _to_device, csr_is_canonical_device  # noqa: E402

n, d, t = 1 << 16, 256, 512
op = make_sparse_embedding(n, t, seed=77)
dev = op.device
g = np.random.default_rng(1010)


def tm(label, fn, reps=7):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"  {label:36s} {1e3 * best:8.3f} ms", flush=True)
    return r


for nnz in (1 << 19, 1 << 23):
    flat = g.permutation(n * d)[:nnz]
    rows, cols = np.divmod(flat, d)
    a = sp.csr_array(sp.coo_array((g.standard_normal(nnz), (rows, cols)), shape=(n, d)))
    print(f"nnz {nnz}: data {a.data.nbytes / 1e6:.1f} MB, indices {a.indices.nbytes / 1e6:.1f} MB", flush=True)
    tm("apply total", lambda: op.apply(a))
    tm("to_device indptr", lambda: _to_device(a.indptr, dev))
    tm("to_device indices", lambda: _to_device(a.indices, dev))
    tm("to_device data", lambda: _to_device(a.data, dev))
    tm("torch .to(dev) data (pageable)", lambda: torch.from_numpy(a.data).to(dev))
    ip, ix, vv = (_to_device(x, dev) for x in (a.indptr, a.indices, a.data))
    tm("canonical check (device + sync)", lambda: csr_is_canonical_device(ip, ix, n))
    res = tm("kernel fp64", lambda: op._apply_csr_device(ip, ix, vv, d, torch.float64, True))
    tm("_host(res)", lambda: _host(res))
    tm("_host(res).numpy()", lambda: _host(res).numpy())
