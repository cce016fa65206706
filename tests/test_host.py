"""Host-side logic that needs no GPU: sizing formulas, descriptors, the
rebinding shim, and the no-fallback guarantee."""

import importlib
import math

import numpy as np
import pytest
import torch

import paper_1207_6365_b200 as skb
from paper_1207_6365_b200 import sketch as S


def test_default_sparse_dim_matches_reference_formula():
    # sketch.py:56-66 with SPARSE_DIM_C = 1, SPARSE_DIM_FLOOR = 4
    for r in (1, 2, 3, 8, 20, 21, 64):
        for eps in (0.1, 0.25, 0.5, 0.75):
            x = r / eps
            want = max(4, math.ceil(x * x * max(1.0, math.log(x))))
            assert S.default_sparse_dim(r, eps) == want
    assert S.default_sparse_dim(21, 0.5) == 6594  # SURVEY §8d config-1 remark
    assert S.default_sparse_dim(64, 0.25) == 363409  # leverage.py default_t1(64)
    with pytest.raises(ValueError):
        S.default_sparse_dim(4, 1.5)
    with pytest.raises(ValueError):
        S.default_sparse_dim(0, 0.5)


def test_identity_operator_and_factories_without_gpu():
    op = S.sparse_embedding_or_identity(10, 10, seed=0)
    assert op.family == "identity"
    x = np.arange(20.0).reshape(10, 2)
    assert np.array_equal(op.apply(x), x)
    assert op.descriptor() == {"family": "identity", "n": 10}
    assert S.from_descriptor({"family": "identity", "n": 3}).input_dim == 3
    with pytest.raises(ValueError):
        op.apply(np.zeros((9, 2)))
    bad = x.copy()
    bad[3, 1] = np.nan
    with pytest.raises(ValueError):
        op.apply(bad)


def test_unknown_family_rejected():
    with pytest.raises(ValueError):
        S.from_descriptor({"family": "nope"})


def test_compose_dimension_check():
    with pytest.raises(ValueError):
        S.compose(S.IdentityOperator(4), S.IdentityOperator(5))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the CPU-only behaviour")
def test_no_cpu_fallback():
    with pytest.raises(Exception):
        skb.SparseEmbedding(100, 10, seed=1)
    with pytest.raises(ValueError):
        skb.SparseEmbedding(100, 10, seed=1, device="cpu")


def test_shim_rebinds_reference_module_globals():
    ref = pytest.importorskip("sketchnla.sketch")
    low = importlib.import_module("sketchnla.lowrank")
    orig = ref.SparseEmbedding
    skb.install()
    try:
        assert ref.SparseEmbedding is skb.SparseEmbedding
        assert ref.apply_right is skb.apply_right and low.apply_right is skb.apply_right
        lp = importlib.import_module("sketchnla.lp")
        assert ref.GeneralizedSparseEmbedding is skb.GeneralizedSparseEmbedding
        assert lp.GeneralizedSparseEmbedding is skb.GeneralizedSparseEmbedding
        assert ref.SrhtOperator is skb.SrhtOperator
        # the reference factories resolve the class at call time (sketch.py:400,426,465)
        if not torch.cuda.is_available():
            with pytest.raises(Exception):
                ref.make_sparse_embedding(50, 8, seed=1)
    finally:
        skb.uninstall()
    assert ref.SparseEmbedding is orig
    assert ref.SrhtOperator is not skb.SrhtOperator
