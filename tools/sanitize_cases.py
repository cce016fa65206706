"""Small invocations of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck).  Each case is also checked against the oracle, so a
sanitizer run doubles as a functional run.  Tools only (not a test)."""

import os
import sys

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1207_6365_b200 import SparseEmbedding, apply_right  # noqa: E402
from paper_1207_6365_b200.solvers import lev_rownorms  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    torch.cuda.set_device(0)
    checks = 0
    for n, t in [(3000, 211), (2000, 3 * 2**20 + 1), (500, 1), (4096, 256)]:
        op = SparseEmbedding(n, t, seed=7)
        h, s = O.hash_signs(n, t, 7)
        assert np.array_equal(op.bucket, h.astype(np.int64))
        for d, dt in [(1, np.float64), (20, np.float64), (128, np.float32), (256, np.float32), (33, np.float32),
                      (200, np.float32), (384, np.float32), (64, np.float64), (256, np.float64)]:  # gather4 rows
            a = rng.standard_normal((n, d)).astype(dt)
            assert np.array_equal(op.apply(a), O.apply_dense(h, s, t, a))
            checks += 1
        for d, dens, dt in [(50, 0.1, np.float64), (64, 0.25, np.float32), (700, 0.02, np.float32),
                            (30_000, 0.001, np.float64)]:
            if t * d > 50_000_000:
                continue
            a = sp.csr_array(sp.random_array((n, d), density=dens, rng=rng, format="csr"), dtype=dt)
            ref = O.np_apply_csr(h, s, t, a)
            assert np.array_equal(op.apply(a), ref)
            fast = op.apply(a, deterministic=False)
            assert np.linalg.norm(fast - ref) <= 1e-12 * max(np.linalg.norm(ref), 1e-300)
            checks += 2
        if t > 1 and t < n:
            for shift in (1, 3):
                a = sp.csr_array(sp.random_array((n, 40), density=0.1, rng=rng, format="csr"))
                dev = [torch.from_numpy(x).cuda() for x in (a.indptr, a.indices, a.data)]
                got = op._apply_csr_device(*dev, 40, torch.float64, canonical=True, shift=shift)
                assert np.array_equal(got.cpu().numpy(), O.np_apply_csr(h, s, t, a))
                checks += 1
    op = SparseEmbedding(900, 17, seed=3)
    h, s = O.hash_signs(900, 17, 3)
    a = rng.standard_normal((30, 900))
    assert np.array_equal(apply_right(a, op), O.apply_dense(h, s, 17, np.ascontiguousarray(a.T)).T)
    c = sp.csr_array(sp.random_array((30, 900), density=0.05, rng=rng, format="csr"))
    assert np.array_equal(apply_right(c, op), O.np_apply_csr(h, s, 17, sp.csr_array(c.T)).T)
    a32 = sp.csr_array(sp.random_array((1000, 64), density=0.25, rng=rng, format="csr"), dtype=np.float32)
    probe = rng.standard_normal((64, 32))
    ref = O.lev_rownorms_csr(a32, probe)
    got = lev_rownorms(a32, probe)
    assert np.max(np.abs(got - ref) / ref) <= 1e-5
    got64 = lev_rownorms(sp.csr_array(a32, dtype=np.float64), probe)
    assert np.max(np.abs(got64 - ref) / ref) <= 1e-12
    checks += 4
    # the passes after the sketch and the fused exchange
    from paper_1207_6365_b200 import cgnr_solve, precondition, richardson_solve
    from paper_1207_6365_b200.distributed import fused_apply_emulated, shard_rows
    from paper_1207_6365_b200.lowrank import _residual_norm

    am = rng.standard_normal((4000, 6))
    bm = am @ rng.standard_normal((6, 1)) + 0.01 * rng.standard_normal((4000, 1))
    pre = precondition(am, 0.5, seed=1)
    for fn in (richardson_solve, cgnr_solve):
        sol = fn(am, pre, bm, 1e-6, max_iter=20)
        assert sol.residual_norm <= 1.01 * np.linalg.norm(am @ np.linalg.lstsq(am, bm, rcond=None)[0] - bm)
    sa_ = sp.csr_array(sp.random_array((2100, 2000), density=0.01, rng=rng, format="csr"))
    lq, _ = np.linalg.qr(rng.standard_normal((2100, 3)))
    wq, _ = np.linalg.qr(rng.standard_normal((2000, 3)))
    _residual_norm(sa_, lq, np.ones(3), wq)
    at = torch.from_numpy(rng.standard_normal((3001, 128)).astype(np.float32)).cuda()
    ops = [SparseEmbedding(3001, 37, 2, row_range=shard_rows(3001, 3, g)) for g in range(3)]
    shards = [at[slice(*shard_rows(3001, 3, g))].contiguous() for g in range(3)]
    full = SparseEmbedding(3001, 37, 2).apply(at)
    assert float((fused_apply_emulated(ops, shards) - full).norm() / full.norm()) <= 1e-12
    checks += 5
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {checks} checks")


if __name__ == "__main__":
    main()
