"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The golden fixtures under tests/golden/ were produced by running the
unmodified reference (tests/golden/make_golden.py); these tests need no GPU.
"""

import hashlib
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import oracle as O
from tests import synth

from .conftest import GOLDEN


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def test_seedseq_and_pcg64_state():
    for row in json.load(open(os.path.join(GOLDEN, "seeds.json"))):
        assert O.seedseq_generate(row["seed"], row["key"], 4).tolist() == row["gen4"]
        st = O.pcg64_seed(row["seed"], row["key"])
        assert (int(st[0]) << 64 | int(st[1])) == int(row["state"])
        assert (int(st[2]) << 64 | int(st[3])) == int(row["inc"])
        assert [str(int(x)) for x in O.pcg64_raw(st, 8)] == row["raw8"]


def test_hash_signs_bit_exact():
    z = load("hash_cases.npz")
    meta = json.load(open(os.path.join(GOLDEN, "hash_cases.json")))
    for k, (n, t, seed) in enumerate(meta):
        h, s = O.hash_signs(n, t, seed)
        assert np.array_equal(h, z[f"h{k}"]), (n, t, seed)
        assert np.array_equal(s, z[f"s{k}"]), (n, t, seed)


def test_plan_is_reference_mat():
    z = load("hash_cases.npz")
    meta = json.load(open(os.path.join(GOLDEN, "hash_cases.json")))
    for k, (n, t, seed) in enumerate(meta):
        if t > 10**6:
            continue
        h = z[f"h{k}"]
        indptr, rows = O.plan(h, t)
        ref = sp.csr_array((np.ones(n), (h.astype(np.int64), np.arange(n))), shape=(t, n))
        assert np.array_equal(indptr, ref.indptr)
        assert np.array_equal(rows, ref.indices)


def _cases():
    meta = json.load(open(os.path.join(GOLDEN, "apply_cases.json")))
    return [m for m in meta if m["kind"] != "right"]


@pytest.mark.parametrize("case", _cases(), ids=lambda m: m["name"])
def test_apply_bit_exact(case):
    z = load("apply_cases.npz")
    name, n, t, seed = case["name"], case["n"], case["t"], case["seed"]
    h, s = O.hash_signs(n, t, seed)
    if case["kind"] == "csr":
        a = sp.csr_array((z[f"{name}_data"], z[f"{name}_indices"], z[f"{name}_indptr"]),
                         shape=tuple(z[f"{name}_shape"]))
        got = O.apply_csr(h, s, t, a)
        np_got = O.np_apply_csr(h, s, t, a)
        assert np.array_equal(np_got, z[f"{name}_sa"])
    else:
        a = z[f"{name}_a"]
        got = O.apply_dense(h, s, t, a)
        mat = O.np_sketch_matrix(h, s, t, n)
        assert np.array_equal(O.np_apply_dense(mat, a), z[f"{name}_sa"])
    assert np.array_equal(got, z[f"{name}_sa"]), name


def test_config1_digests():
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["config1"]
    a, b, seed = synth.config1()
    assert sha(a) == cfg["sha_a"]
    h, s = O.hash_signs(cfg["n"], cfg["t"], seed)
    assert sha(h) == cfg["sha_h"] and sha(s) == cfg["sha_s"]
    assert sha(O.apply_dense(h, s, cfg["t"], a)) == cfg["sha_sa"]
    assert sha(O.apply_dense(h, s, cfg["t"], b)) == cfg["sha_sb"]


def test_config2_digests():
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["config2"]
    a, b, seed = synth.config2()
    assert sha(a.indices) == cfg["sha_indices"] and sha(a.data) == cfg["sha_data"]
    h, s = O.hash_signs(cfg["n"], cfg["t"], seed)
    assert sha(h) == cfg["sha_h"] and sha(s) == cfg["sha_s"]
    assert sha(O.apply_csr(h, s, cfg["t"], a)) == cfg["sha_sa"]


def test_lev_contraction():
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["lev"]
    z = load("lev_case.npz")
    a, m, k, seed = synth.lev_case()
    got = O.lev_rownorms_csr(a, z["probe"])
    rel = np.abs(got - z["scores"]) / np.maximum(np.abs(z["scores"]), 1e-300)
    assert rel.max() <= 1e-12
    assert np.allclose(O.np_lev_rownorms(a, z["probe"]), z["scores"], rtol=1e-13, atol=0)


def test_threaded_oracle_equals_scalar_oracle():
    """The thread-parallel forms used for full-size parity (configs 3-5) split
    buckets / rows across threads, never one element's sum: bit-identical to
    the scalar restatement, including t = 1 and t > n."""
    import scipy.sparse as sp

    rng = np.random.default_rng(1)
    for n, t, d in [(100_000, 4_000, 20), (50_000, 1, 7), (3_000, 5_000, 3)]:
        h, s = O.hash_signs(n, t, 5)
        a = rng.standard_normal((n, d)).astype(np.float32)
        assert np.array_equal(O.apply_dense(h, s, t, a), O.apply_dense(h, s, t, a, threads=0))
        c = sp.csr_array(sp.random_array((n, d), density=0.3, rng=rng, format="csr"))
        assert np.array_equal(O.apply_csr(h, s, t, c), O.apply_csr(h, s, t, c, threads=5))
        p = rng.standard_normal((d, 8))
        assert np.array_equal(O.lev_rownorms_csr(c, p), O.lev_rownorms_csr(c, p, threads=3))
