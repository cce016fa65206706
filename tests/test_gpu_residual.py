"""Fused residual pass (skt_residual_dense / _csr, regress.py:79-82) against
the oracle's restatement of the reference's `_residual_fro`."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import oracle as O
from paper_1207_6365_b200.solvers import residual_fro

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,k,adt,bdt", [
    (100_000, 20, 1, np.float64, np.float64),   # config-1 shape
    (5_003, 1, 1, np.float32, np.float64),
    (7_001, 33, 3, np.float32, np.float32),
    (3_000, 300, 2, np.float64, np.float64),    # d > 32 lanes
    (1, 5, 1, np.float64, np.float64),
])
def test_residual_dense(n, d, k, adt, bdt):
    rng = np.random.default_rng(n + d + k)
    a = rng.standard_normal((n, d)).astype(adt)
    x = rng.standard_normal((d, k))
    b = (a.astype(np.float64) @ x + 0.1 * rng.standard_normal((n, k))).astype(bdt)
    ref = O.residual_fro(a.astype(np.float64), x, b.astype(np.float64))
    got = residual_fro(a, x, b)
    assert abs(got - ref) <= 1e-12 * ref
    # deterministic: the same bits on a second run
    assert residual_fro(a, x, b) == got


@pytest.mark.parametrize("n,d,k,density,vdt", [
    (1_000_000, 50, 1, 0.1, np.float64),   # config-2 shape
    (20_000, 64, 2, 0.25, np.float32),
    (3_000, 5_000, 1, 0.01, np.float64),  # X in global memory (d*k*8 > 48 KB)
])
def test_residual_csr(n, d, k, density, vdt):
    rng = np.random.default_rng(n + d)
    a = sp.csr_array(sp.random_array((n, d), density=density, rng=rng, format="csr"), dtype=vdt)
    x = rng.standard_normal((d, k))
    b = a.astype(np.float64) @ x + 0.01 * rng.standard_normal((n, k))
    ref = O.residual_fro(a.astype(np.float64), x, b)
    got = residual_fro(a, x, b)
    assert abs(got - ref) <= 1e-12 * ref
    # empty rows and an all-zero row block are fine
    a2 = a.tolil()
    a2[: n // 3] = 0
    a2 = sp.csr_array(a2)
    assert abs(residual_fro(a2, x, b) - O.residual_fro(a2.astype(np.float64), x, b)) <= 1e-12 * ref


def test_residual_torch_inputs():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((4_000, 16))
    x = rng.standard_normal(16)
    b = rng.standard_normal(4_000)
    ref = O.residual_fro(a, x[:, None], b[:, None])  # the reference always passes 2-D operands
    got = residual_fro(torch.from_numpy(a).cuda(), torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda())
    assert abs(got - ref) <= 1e-12 * ref
