"""GPU SRHT (skt_srht_apply) against the reference's SrhtOperator.apply
(golden vectors from the reference itself, tests/golden/srht_cases.npz) and
the oracle restatement at a config-4 leverage-pipeline size: bit-identical
(the same fp64 butterflies in the same stage order)."""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1207_6365_b200.solvers import srht_apply

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_srht_golden_bit_exact():
    z = np.load(os.path.join(GOLDEN, "srht_cases.npz"))
    for k, (n, d, t, seed) in enumerate(z["meta"]):
        got = srht_apply(z[f"a{k}"], int(t), int(seed))
        assert np.array_equal(got, z[f"y{k}"]), (n, d, t, seed)


@pytest.mark.parametrize("n,d,t", [(363_409, 64, 20_000), (3, 1, 4), (1 << 14, 5, 1 << 14), (70_001, 17, 33)])
def test_srht_matches_oracle(n, d, t):
    """(363409 x 64: config 4's t1 x d sketch, n_pad = 2^19 -> three passes)."""
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, d))
    ref = O.srht_apply(a, t, 5)
    got = srht_apply(a, t, 5)
    assert np.array_equal(got, ref)
    gt = srht_apply(torch.from_numpy(a).cuda(), t, 5)  # device in, device out
    assert gt.is_cuda and np.array_equal(gt.cpu().numpy(), ref)


def test_srht_errors():
    with pytest.raises(ValueError):
        srht_apply(np.ones((5, 2)), 9, 0)  # t > n_pad = 8
