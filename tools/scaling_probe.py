"""The reference's acceptance criterion 10 (test_acceptance.py:264-291) on this
package's operator: apply time vs nnz (log-log slope), with a per-call
breakdown of the smallest size."""
import math
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from paper_1207_6365_b200 import make_sparse_embedding  # noqa: E402

n, d, t = 1 << 16, 256, 512
op = make_sparse_embedding(n, t, seed=77)
g = np.random.default_rng(1010)
sizes = [1 << p for p in range(19, 24)]
mats = []
for nnz in sizes:
    flat = g.permutation(n * d)[:nnz]
    rows, cols = np.divmod(flat, d)
    mats.append(sp.csr_array(sp.coo_array((g.standard_normal(nnz), (rows, cols)), shape=(n, d))))
best = [math.inf] * len(sizes)
for a in mats:
    op.apply(a)
for _ in range(7):
    for i, a in enumerate(mats):
        t0 = time.perf_counter()
        op.apply(a)
        best[i] = min(best[i], time.perf_counter() - t0)
slope = float(np.polyfit(np.log(sizes), np.log(best), 1)[0])
print("times ms", [round(1e3 * b, 3) for b in best], "slope", round(slope, 3))
