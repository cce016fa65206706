"""Matrix Market ingest (io.py:37-104): the native parser (CPU) against the
reference's outputs and error messages, and the GPU canonicalisation against
the reference's canonical CSR (golden vectors from the reference itself)."""

import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from .conftest import GOLDEN
from .golden.mm_cases import BAD, GOOD, NONFINITE


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_text(text)
    return str(p)


def _golden_csr(name):
    z = np.load(os.path.join(GOLDEN, "mm_cases.npz"))
    return sp.csr_array((z[f"{name}_data"], z[f"{name}_indices"], z[f"{name}_indptr"]),
                        shape=tuple(z[f"{name}_shape"]))


@pytest.mark.parametrize("name", sorted(GOOD))
def test_native_parse_matches_reference(tmp_path, name):
    """Host parse (C++) + host canonicalisation (scipy, the oracle side) ==
    the reference's canonical CSR."""
    from paper_1207_6365_b200.mmio import read_coo

    p = _write(tmp_path, name, GOOD[name])
    shape, r, c, v = read_coo(p, n_threads=3)
    m = sp.csr_array(sp.coo_array((v.numpy(), (r.numpy(), c.numpy())), shape=shape))
    m.sum_duplicates()
    m.eliminate_zeros()
    ref = _golden_csr(name)
    assert m.shape == ref.shape
    assert np.array_equal(m.indptr, ref.indptr) and np.array_equal(m.indices, ref.indices)
    assert np.array_equal(m.data, ref.data)


@pytest.mark.parametrize("name", sorted(BAD))
def test_native_errors_match_reference(tmp_path, name):
    from paper_1207_6365_b200.mmio import MatrixMarketError, read_coo

    want = json.load(open(os.path.join(GOLDEN, "mm_errors.json")))[name]
    p = _write(tmp_path, name, BAD[name])
    with pytest.raises(MatrixMarketError) as e:
        read_coo(p)
    assert str(e.value) == want.replace("{path}", p)


def test_native_parse_large_multithreaded(tmp_path):
    """A 300k-entry file parsed on many threads equals a single-thread parse
    and numpy's reading of the same text."""
    from paper_1207_6365_b200.mmio import read_coo

    rng = np.random.default_rng(3)
    n, m, k = 5000, 700, 300_000
    r = rng.integers(1, n + 1, k)
    c = rng.integers(1, m + 1, k)
    v = rng.standard_normal(k)
    lines = [f"%%MatrixMarket matrix coordinate real general\n% x\n{n} {m} {k}\n"]
    lines += [f"{a} {b} {float(x)!r}\n" if i % 1000 else f"% comment {i}\n{a} {b} {float(x)!r}\n" for i, (a, b, x) in
              enumerate(zip(r, c, v))]
    p = tmp_path / "big.mtx"
    p.write_text("".join(lines))
    shape, r1, c1, v1 = read_coo(str(p), n_threads=16)
    _, r2, c2, v2 = read_coo(str(p), n_threads=1)
    assert shape == (n, m)
    assert np.array_equal(r1.numpy(), r - 1) and np.array_equal(c1.numpy(), c - 1)
    assert np.array_equal(v1.numpy(), v)  # repr round-trips exactly through strtod
    assert np.array_equal(r1.numpy(), r2.numpy()) and np.array_equal(v1.numpy(), v2.numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOOD))
def test_gpu_canonical_csr_matches_reference(tmp_path, name):
    from paper_1207_6365_b200.mmio import load_matrix_market

    got = load_matrix_market(_write(tmp_path, name, GOOD[name]))
    ref = _golden_csr(name)
    assert got.shape == ref.shape
    assert np.array_equal(got.indptr, ref.indptr) and np.array_equal(got.indices, ref.indices)
    assert np.array_equal(got.data, ref.data)


@pytest.mark.gpu
def test_gpu_ingest_large_and_sketch(tmp_path):
    """300k entries with duplicates and zeros: GPU canonical CSR == scipy's,
    and the device CSR feeds S.A directly (== applying the scipy matrix)."""
    import torch

    from paper_1207_6365_b200 import SparseEmbedding
    from paper_1207_6365_b200.mmio import as_torch_csr, load_matrix_market_device, read_coo

    rng = np.random.default_rng(4)
    n, m, k = 20_000, 300, 300_000
    r = rng.integers(1, n + 1, k)
    c = rng.integers(1, m + 1, k)
    v = np.where(rng.random(k) < 0.01, 0.0, rng.standard_normal(k))
    p = tmp_path / "big.mtx"
    p.write_text(f"%%MatrixMarket matrix coordinate real general\n{n} {m} {k}\n" +
                 "".join(f"{a} {b} {float(x)!r}\n" for a, b, x in zip(r, c, v)))
    shape, ip, ix, vv = load_matrix_market_device(str(p))
    _, r0, c0, v0 = read_coo(str(p))
    ref = sp.csr_array(sp.coo_array((v0.numpy(), (r0.numpy(), c0.numpy())), shape=shape))
    ref.sum_duplicates()
    ref.eliminate_zeros()
    assert np.array_equal(ip.cpu().numpy(), ref.indptr) and np.array_equal(ix.cpu().numpy(), ref.indices)
    # duplicates: pairs sum identically in any order; larger runs to rounding
    assert np.allclose(vv.cpu().numpy(), ref.data, rtol=1e-14, atol=1e-14)
    op = SparseEmbedding(n, 512, 9)
    sa_dev = op.apply(as_torch_csr(shape, ip, ix, vv))
    sa_ref = op.apply(sp.csr_array((vv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=shape))
    assert np.array_equal(sa_dev.cpu().numpy(), sa_ref)


@pytest.mark.parametrize("name", sorted(NONFINITE))
def test_nonfinite_files_parse_on_host(tmp_path, name):
    """NaN / inf values are valid tokens for the parser (the reference's
    float()); the rejection comes from the canonicalisation (next test)."""
    from paper_1207_6365_b200.mmio import read_coo

    shape, r, c, v = read_coo(_write(tmp_path, name, NONFINITE[name]))
    assert not np.all(np.isfinite(v.numpy()))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(NONFINITE))
def test_gpu_nonfinite_rejected_like_reference(tmp_path, name):
    """as_csr's finiteness check (io.py:103, _validation.py:39-40): the same
    ValueError text as the reference, also when inf and -inf duplicates sum
    to NaN (nonfinite_cancel)."""
    from paper_1207_6365_b200.mmio import MatrixMarketError, load_matrix_market

    want = json.load(open(os.path.join(GOLDEN, "mm_errors.json")))[name]
    p = _write(tmp_path, name, NONFINITE[name])
    with pytest.raises(ValueError) as e:
        load_matrix_market(p)
    assert not isinstance(e.value, MatrixMarketError)
    assert str(e.value) == want.replace("{path}", p)
