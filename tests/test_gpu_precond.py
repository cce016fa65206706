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
