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


def test_no_reference_cpu_code_behind_the_package(monkeypatch):
    """The families this package does not own raise instead of being handed to
    the reference's CPU classes, and so does the leverage_sample low-rank
    strategy -- even when the reference package is importable."""
    import sys
    import types

    from paper_1207_6365_b200.lowrank import low_rank_approx

    trap = types.ModuleType("sketchnla")
    trap.__path__ = []  # any submodule import would fail loudly below

    def _boom(*a, **k):  # pragma: no cover - must not be reached
        raise AssertionError("product code reached the reference package")

    trap.__getattr__ = _boom
    monkeypatch.setitem(sys.modules, "sketchnla", trap)
    for d in ({"family": "leverage", "probs": [0.5, 0.5], "t": 2, "seed": 0},
              {"family": "gaussian", "rows": 2, "cols": 3, "seed": 0}):
        with pytest.raises(ValueError, match="not provided by this package"):
            S.from_descriptor(d)
    with pytest.raises(ValueError, match="leverage_sample"):
        low_rank_approx(np.ones((8, 6)), 2, 0.5, strategy="leverage_sample")


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


def test_srht_dims_and_nnls_match_reference():
    """Host pieces of the callers against the reference itself (build
    container; skipped where the reference is absent): default_srht_dim
    (sketch.py:83-94) and Lawson-Hanson NNLS (regress.py:288-327) -- the same
    numpy operations, so the same bits."""
    ref_sketch = pytest.importorskip("sketchnla.sketch")
    ref_regress = importlib.import_module("sketchnla.regress")
    from paper_1207_6365_b200.solvers import default_srht_dim, lawson_hanson_nnls

    for r in (1, 5, 12, 30):
        for eps in (0.1, 1 / 6, 0.25, 0.5):
            for n in (100, 8920, 10**6):
                assert default_srht_dim(r, eps, n) == ref_sketch.default_srht_dim(r, eps, n)
    rng = np.random.default_rng(5)
    for trial in range(20):
        m = rng.standard_normal((60, 7))
        y = m @ rng.standard_normal(7) + 0.1 * rng.standard_normal(60)
        assert np.array_equal(lawson_hanson_nnls(m, y), ref_regress.lawson_hanson_nnls(m, y))


def test_fused_exchange_owner_layout():
    """Owner ranges of the fused exchange cover the buckets once; every
    rank's slot fits the receive buffer."""
    from paper_1207_6365_b200.distributed import owner_bounds

    for t in (1, 7, 1001, 65536):
        for world in (1, 2, 3, 8):
            b = owner_bounds(t, world)
            assert b[0] == 0 and b[-1] == t and all(b[g] <= b[g + 1] for g in range(world))
            cap = max(b[g + 1] - b[g] for g in range(world))
            assert cap * world >= t and cap <= -(-t // world)
