"""Generalized sparse embedding (sketch.py:176-238): the oracle pinned to the
reference's golden vectors (CPU), and the GPU operator bit-identical to them."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import oracle as O

from .conftest import GOLDEN


def _cases():
    z = np.load(os.path.join(GOLDEN, "gse_cases.npz"))
    for k, row in enumerate(z["meta"]):
        n, r, eps, delta, seed, q, kb, v, t = row
        yield k, int(n), int(r), float(eps), float(delta), int(seed), (int(q), int(kb), int(v), int(t)), z


def _dup(n):
    return sp.csr_array((np.array([1.5, -2.0, 0.25, 3.0]), np.array([3, 3, 0, 3]), np.array([0, 2, 4] + [4] * (n - 2))),
                        shape=(n, 5))


def test_gse_oracle_matches_reference_golden():
    for k, n, r, eps, delta, seed, dims, z in _cases():
        q, kb, v, t, outer, inner, sign, mat = O.gse_operator(n, r, eps, delta, seed)
        assert (q, kb, v, t) == dims
        assert np.array_equal(outer.astype(np.uint32), z[f"outer{k}"])
        assert np.array_equal(inner.astype(np.uint32), z[f"inner{k}"])
        assert np.array_equal(sign.astype(np.int8), z[f"sign{k}"])
        assert np.array_equal(O.gse_apply(mat, z[f"a64_{k}"]), z[f"sa64_{k}"])
        assert np.array_equal(O.gse_apply(mat, z[f"a32_{k}"]), z[f"sa32_{k}"])
        ac = sp.csr_array((z[f"ac_data{k}"], z[f"ac_indices{k}"], z[f"ac_indptr{k}"]), shape=(n, 40))
        assert np.array_equal(O.gse_apply(mat, ac), z[f"sac_{k}"])


@pytest.mark.gpu
def test_gse_gpu_bit_exact():
    import torch

    from paper_1207_6365_b200.generalized import GeneralizedSparseEmbedding

    for k, n, r, eps, delta, seed, dims, z in _cases():
        op = GeneralizedSparseEmbedding(n, r, eps, delta, seed)
        assert (op.q, op.k_blocks, op.v, op.output_dim) == dims
        assert np.array_equal(op.outer_bucket.astype(np.uint32), z[f"outer{k}"])
        assert np.array_equal(op.inner_bucket.astype(np.uint32), z[f"inner{k}"])
        assert np.array_equal(op.inner_sign.astype(np.int8), z[f"sign{k}"])
        for key in ("a64", "a32", "a1"):
            assert np.array_equal(op.apply(z[f"{key}_{k}"]), z[f"sa{key[1:]}_{k}"]), (k, key)
        ac = sp.csr_array((z[f"ac_data{k}"], z[f"ac_indices{k}"], z[f"ac_indptr{k}"]), shape=(n, 40))
        assert np.array_equal(op.apply(ac), z[f"sac_{k}"])
        assert np.array_equal(op.apply(_dup(n)), z[f"sadup_{k}"])  # duplicate columns summed in order
        # the materialised matrix equals the reference's
        _, _, _, _, _, _, _, mat = O.gse_operator(n, r, eps, delta, seed)
        assert (op._mat != mat).nnz == 0
        # torch CUDA input stays on the device
        x = torch.from_numpy(z[f"a64_{k}"]).cuda()
        assert np.array_equal(op.apply(x).cpu().numpy(), z[f"sa64_{k}"])


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,d", [(np.float64, 64), (np.float64, 20), (np.float32, 64), (np.float32, 200),
                                     (np.float32, 384), (np.float64, 256)])
def test_gse_gpu_gather4_rows(dtype, d):
    """Rows of 512 B .. 2 KB take the K3 gather4 kernel with weighted terms:
    still scipy's order and rounding (fl(w x) then add), bit for bit."""
    from paper_1207_6365_b200.generalized import GeneralizedSparseEmbedding

    n = 6000
    op = GeneralizedSparseEmbedding(n, 5, 0.5, 0.1, 11)
    _, _, _, _, _, _, _, mat = O.gse_operator(n, 5, 0.5, 0.1, 11)
    a = np.random.default_rng(d).standard_normal((n, d)).astype(dtype)
    ref = mat @ a.astype(np.float64)
    assert np.array_equal(op.apply(a), ref)
