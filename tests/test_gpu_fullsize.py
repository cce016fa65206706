"""Whole-matrix oracle parity at BASELINE's full sizes (configs 3, 4, 5 and
the leverage contraction K5 at config 4's shape).

The inputs are generated on the GPU by bench.py's seeded generators (the
exact matrices the benchmark times), copied to the host once, and the C
oracle (oracle/skt_oracle.c, thread-parallel form: buckets or rows split
over the host cores, every output element summed by one thread in the
reference's order -- bit-identical to the scalar restatement) recomputes the
WHOLE result:

* S.A: ``np.array_equal`` against the GPU's fp64 output (the reference's dtype;
  sketch.py:153-165 -- sequential fp64 per (bucket, column), rows ascending),
  and the fp32 output equals the oracle rounded once to fp32.
* config 5 fast mode (unordered atomics): <= 1e-12 normwise with an fp64
  accumulator, <= 1e-5 with the fp32 output the benchmark writes.
* K5 (leverage.py:90-91 -- rows = A @ probe, squared row norms, fp64): fp32
  input on the tensor cores <= 1e-5 relative per score; fp64 input (as_csr's
  upcast, the path the reference API takes) <= 1e-12 relative per score.
"""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import oracle as O
from paper_1207_6365_b200 import SparseEmbedding
from paper_1207_6365_b200.solvers import lev_rownorms

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DEV = torch.device("cuda", 0)


def _normwise(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def _csr_host(ip, ix, vv, shape):
    return sp.csr_array((vv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=shape)


def test_config3_whole_sa_bit_exact():
    from bench import CONFIGS, gen_dense_shard

    c = CONFIGS["c3"]
    n, d, m = c["n"], c["d"], c["m"]
    A = gen_dense_shard(torch, c, 0, n, DEV)
    op = SparseEmbedding(n, m, c["seed"], device=DEV)
    sa64 = op.apply(A).cpu().numpy()
    sa32 = op.apply(A, out_dtype=torch.float32).cpu().numpy()
    h, s = O.hash_signs(n, m, c["seed"])
    assert np.array_equal(op.h.cpu().numpy().view(np.uint32), h)
    a_host = A.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    ref = O.apply_dense(h, s, m, a_host, threads=0)
    assert np.array_equal(sa64, ref)
    assert np.array_equal(sa32, ref.astype(np.float32))


@pytest.fixture(scope="module")
def config4():
    from bench import CONFIGS, gen_csr_shard

    c = CONFIGS["c4"]
    ip, ix, vv = gen_csr_shard(torch, c, 0, c["n"], DEV)
    return c, (ip, ix, vv), _csr_host(ip, ix, vv, (c["n"], c["d"]))


def test_config4_whole_sa_bit_exact(config4):
    c, (ip, ix, vv), a = config4
    n, d, m = c["n"], c["d"], c["m"]
    op = SparseEmbedding(n, m, c["seed"], device=DEV)
    sa64 = op._apply_csr_device(ip, ix, vv, d, torch.float64, canonical=True).cpu().numpy()
    sa32 = op._apply_csr_device(ip, ix, vv, d, torch.float32, canonical=True).cpu().numpy()
    # the public API on the same matrix (canonical scipy CSR, fp64 result)
    api = op.apply(a)
    h, s = O.hash_signs(n, m, c["seed"])
    ref = O.apply_csr(h, s, m, a, threads=0)
    assert np.array_equal(sa64, ref)
    assert np.array_equal(api, ref)
    assert np.array_equal(sa32, ref.astype(np.float32))


def test_config4_leverage_contraction_full_size(config4):
    """K5 over config 4's 4.19 M rows, k = 32 (leverage.py:87-91)."""
    c, (ip, ix, vv), a = config4
    rng = np.random.default_rng(17)
    # a probe of the pipeline's shape and scale: N (d x d upper-triangular
    # inverse) times G^T / sqrt(k)
    r = np.triu(rng.standard_normal((c["d"], c["d"]))) + 8 * np.eye(c["d"])
    probe = np.linalg.inv(r) @ (rng.standard_normal((32, c["d"])).T / np.sqrt(32))
    ref = O.lev_rownorms_csr(a, probe, threads=0)
    assert np.all(ref > 0)
    got32 = lev_rownorms(torch.sparse_csr_tensor(ip, ix, vv, size=a.shape), probe).cpu().numpy()
    assert np.max(np.abs(got32 - ref) / ref) <= 1e-5
    a64 = sp.csr_array(a, dtype=np.float64)  # as_csr's upcast (_validation.py:33)
    ref64 = O.lev_rownorms_csr(a64, probe, threads=0)
    assert np.array_equal(ref64, ref)  # the oracle upcasts fp32 values exactly
    vv64 = vv.double()
    got64 = lev_rownorms(torch.sparse_csr_tensor(ip, ix, vv64, size=a.shape), probe).cpu().numpy()
    assert np.max(np.abs(got64 - ref) / ref) <= 1e-12


def test_config5_whole_sa_exact_and_fast():
    from bench import CONFIGS, gen_csr_shard

    c = CONFIGS["c5"]
    n, d, m = c["n"], c["d"], c["m"]
    ip, ix, vv = gen_csr_shard(torch, c, 0, n, DEV)
    op = SparseEmbedding(n, m, c["seed"], device=DEV)
    exact = op._apply_csr_device(ip, ix, vv, d, torch.float64, canonical=True).cpu().numpy()
    exact32 = op._apply_csr_device(ip, ix, vv, d, torch.float32, canonical=True).cpu().numpy()
    fast64 = op._apply_csr_device(ip, ix, vv, d, torch.float64, canonical=True, deterministic=False).cpu().numpy()
    fast32 = op._apply_csr_device(ip, ix, vv, d, torch.float32, canonical=True, deterministic=False).cpu().numpy()
    a = _csr_host(ip, ix, vv, (n, d))
    del ip, ix, vv
    torch.cuda.empty_cache()
    h, s = O.hash_signs(n, m, c["seed"])
    ref = O.apply_csr(h, s, m, a, threads=0)
    assert np.array_equal(exact, ref)
    assert np.array_equal(exact32, ref.astype(np.float32))
    assert _normwise(fast64, ref) <= 1e-12
    assert _normwise(fast32.astype(np.float64), ref) <= 1e-5
