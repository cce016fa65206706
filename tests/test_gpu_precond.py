"""Preconditioned iterations (regress.py:159-285) and the rank-k Gram
residual (lowrank.py:100-108) with their passes on the GPU (csrc/lsq.cu),
against golden vectors produced by the reference itself
(tests/golden/make_golden_precond.py)."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from paper_1207_6365_b200 import cgnr_solve, precondition, richardson_solve
from paper_1207_6365_b200.lowrank import _residual_norm
from paper_1207_6365_b200.precond import gram_residual_sq

from .conftest import GOLDEN
from .synth import gram_cases, precond_cases

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(GOLDEN, "precond_cases.npz"))
CASES = precond_cases()


@pytest.mark.parametrize("name", sorted(CASES))
def test_precondition_matches_reference(name):
    a, b, eps0, seed = CASES[name]
    pre = precondition(a, eps0, seed=seed)
    # S.A and the SRHT are bit-identical on the GPU, the QRs are the same
    # LAPACK calls: r_inv is the reference's to the bit
    assert pre.rank == int(G[f"{name}/rank"]) and pre.sketch_dim == int(G[f"{name}/sketch_dim"])
    assert np.array_equal(pre.r_inv, G[f"{name}/r_inv"])


@pytest.mark.parametrize("method,fn", [("richardson", richardson_solve), ("cgnr", cgnr_solve)])
@pytest.mark.parametrize("name", sorted(CASES))
def test_iterations_match_reference(name, method, fn):
    """Same iteration count, residual history to 1e-9 relative, x to 1e-9
    normwise: the fused passes sum in a different order than BLAS (fp64
    rounding), nothing else differs."""
    a, b, eps0, seed = CASES[name]
    pre = precondition(a, eps0, seed=seed)
    sol = fn(a, pre, b, 1e-6, max_iter=60)
    key = f"{name}/{method}"
    assert sol.method == method and sol.sketch_dim == pre.sketch_dim and sol.seed == seed
    assert sol.iterations == int(G[f"{key}/iterations"])
    hist = np.asarray(sol.residual_history)
    ref_hist = G[f"{key}/history"]
    assert hist.shape == ref_hist.shape
    assert np.max(np.abs(hist - ref_hist) / ref_hist) <= 1e-9
    ref_x = G[f"{key}/x"]
    assert np.linalg.norm(sol.x - ref_x) <= 1e-9 * np.linalg.norm(ref_x)
    assert abs(sol.residual_norm - float(G[f"{key}/residual"])) <= 1e-10 * float(G[f"{key}/residual"])


def test_precondition_errors():
    a, b, _, _ = CASES["dense"]
    with pytest.raises(ValueError):
        precondition(a, 0.75)
    with pytest.raises(ValueError):
        precondition(np.zeros((20_000, 4)), 0.5)
    pre = precondition(a, 0.5, seed=3)
    with pytest.raises(ValueError):
        richardson_solve(a, pre, b[:-1], 1e-6)


@pytest.mark.parametrize("name", ["csr", "dense"])
def test_gram_residual_matches_reference(name):
    a = gram_cases()[name]
    l, d, w = (G[f"gram_{name}/{k}"] for k in "ldw")
    got = _residual_norm(a, l, d, w)
    ref = float(G[f"gram_{name}/value"])
    assert abs(got - ref) <= 1e-10 * ref
    # one fused pass: cross and ||A||_F^2 against numpy, deterministic
    cross, fro2 = gram_residual_sq(a, l, d, w)
    dense = a.toarray() if sp.issparse(a) else a
    assert abs(cross - np.einsum("ij,ij->", dense @ (w * d), l)) <= 1e-12 * fro2
    assert abs(fro2 - np.sum(dense * dense)) <= 1e-13 * fro2
    assert gram_residual_sq(a, l, d, w) == (cross, fro2)
    # fp32 CSR values are upcast like the reference's fp64 arithmetic
    if name == "csr":
        a32 = sp.csr_array(a, dtype=np.float32)
        c32, f32 = gram_residual_sq(a32, l, d, w)
        d32 = a32.toarray().astype(np.float64)
        assert abs(c32 - np.einsum("ij,ij->", d32 @ (w * d), l)) <= 1e-12 * f32


NNLS = __import__("tests.synth", fromlist=["nnls_cases"]).nnls_cases()


@pytest.mark.parametrize("name", sorted(NNLS))
def test_nonneg_regression_matches_reference(name):
    """SRHT o sparse embedding on the GPU (bit-identical sketches), the same
    Lawson-Hanson steps on the host: x equal to the reference's up to LAPACK
    rounding, the same active set, residual by the fused GPU pass."""
    from paper_1207_6365_b200 import nonneg_regression

    a, b, eps, seed = NNLS[name]
    sol = nonneg_regression(a, b, eps, seed=seed)
    ref_x = G[f"nnls_{name}/x"]
    assert sol.method == "nnls" and sol.sketch_dim == int(G[f"nnls_{name}/sketch_dim"])
    assert np.array_equal(sol.x > 0, ref_x > 0)
    assert np.linalg.norm(sol.x - ref_x) <= 1e-10 * np.linalg.norm(ref_x)
    ref_res = float(G[f"nnls_{name}/residual"])
    assert abs(sol.residual_norm - ref_res) <= 1e-11 * ref_res


def test_nnls_pass_cap_and_feasibility():
    from paper_1207_6365_b200 import SolverError, lawson_hanson_nnls

    rng = np.random.default_rng(0)
    m = rng.standard_normal((50, 6))
    y = rng.standard_normal(50)
    x = lawson_hanson_nnls(m, y)
    w = m.T @ (y - m @ x)
    assert np.all(x >= 0) and np.all(w[x == 0] <= 1e-8 * max(np.abs(m.T @ y).max(), 1.0))
    with pytest.raises(SolverError):
        lawson_hanson_nnls(m, y @ np.zeros(50) + m @ np.ones(6), max_passes=0)


def test_low_rank_default_strategy_matches_reference():
    """low_rank_approx(a, k, eps) with the default srht_compose strategy:
    column sketch (transpose-free) + SRHT, S U / S A + SRHT, all on the GPU and
    bit-identical, so the factors equal the reference's; err from the fused
    Gram pass (7.5M entries > the dense limit) to 1e-10."""
    from paper_1207_6365_b200.lowrank import low_rank_approx

    from .synth import lowrank_default_case

    res = low_rank_approx(lowrank_default_case(), 5, 0.5, seed=11)
    for key in ("l", "d", "w"):
        assert np.array_equal(getattr(res.factors, key), G[f"lowrank_default/{key}"]), key
    assert res.t_r == int(G["lowrank_default/t_r"]) and res.t_s == int(G["lowrank_default/t_s"])
    assert res.cond_su == float(G["lowrank_default/cond_su"])
    assert abs(res.err - float(G["lowrank_default/err"])) <= 1e-10 * float(G["lowrank_default/err"])
    with pytest.raises(ValueError):
        low_rank_approx(lowrank_default_case(), 5, 0.5, strategy="bogus")


def test_srht_operator_views_and_apply():
    from paper_1207_6365_b200 import SrhtOperator, srht_or_identity

    z = np.load(os.path.join(GOLDEN, "srht_cases.npz"))
    meta = z["meta"]
    for k, (_, _, t, seed) in enumerate(meta):
        a = z[f"a{k}"]
        op = SrhtOperator(a.shape[0], int(t), int(seed))
        assert np.array_equal(op.apply(a), z[f"y{k}"])
        assert op.sign.shape == (op.n_pad,) and set(np.unique(op.sign)) <= {-1.0, 1.0}
        assert op.sampled_rows.shape == (int(t),) and op.sampled_rows.max() < op.n_pad
    op = SrhtOperator(1000, 300, 2)  # host views: the reference's arrays
    assert np.array_equal(op.sign, G["srht_views/sign"]) and np.array_equal(op.sampled_rows, G["srht_views/rows"])
    full = SrhtOperator(100, 1, 3, all_rows=True)  # exact isometry hook
    x = np.random.default_rng(1).standard_normal((100, 4))
    assert full.output_dim == 128
    assert np.allclose(np.linalg.norm(full.apply(x)), np.linalg.norm(x), rtol=1e-13)
    assert srht_or_identity(50, 60, 1).family == "identity"


@pytest.mark.parametrize("n,d,k,dtype,pad", [
    (100_000, 20, 20, np.float64, 0),   # config 1's M = A R
    (5_000, 300, 17, np.float32, 3),    # fp32 A, padded rows
    (2_000, 5_000, 9, np.float64, 0),   # X staged in several shared-memory chunks
    (7, 3, 1, np.float64, 1),
])
def test_gemm_dense_matches_numpy(n, d, k, dtype, pad):
    """skt_gemm_dense (M = A R for a dense A, regress.py:200): fp64 dot products,
    equal to numpy's BLAS product to rounding."""
    import torch

    from paper_1207_6365_b200 import _lib
    from paper_1207_6365_b200.sketch import _TORCH_TO_SKT

    rng = np.random.default_rng(n + d)
    a = rng.standard_normal((n, d + pad)).astype(dtype)
    x = rng.standard_normal((d, k))
    ad = torch.from_numpy(a).cuda()
    xd = torch.from_numpy(x).cuda()
    y = torch.empty((n, k), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().skt_gemm_dense(n, d, ad.data_ptr(), _TORCH_TO_SKT[ad.dtype], d + pad, xd.data_ptr(), k,
                                         y.data_ptr(), k, torch.cuda.current_stream().cuda_stream))
    ref = a[:, :d].astype(np.float64) @ x
    err = np.abs(y.cpu().numpy() - ref).max() / max(np.abs(ref).max(), 1e-300)
    assert err <= 1e-13, err
