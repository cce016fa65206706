"""Generate the golden fixtures from the REFERENCE itself (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified reference package ``sketchnla`` from /root/reference and
records its outputs on seeded inputs.  The GPU box has no /root/reference, so
the tests read only the committed outputs:

* ``hash_cases.npz``  -- bucket/sign vectors exactly as sketch.py:147-148 draw
  them (``_rng(seed, 0, 0).integers(0, t, size=n)`` / ``_rng(seed, 0, 1).choice``),
  incl. t = 1, powers of two, the config t values and the Lemire-rejection
  stress values t = 3*2^30, 2^31+1, and t = 2^32.
* ``apply_cases.npz`` -- small S.A cases through SparseEmbedding.apply (dense
  f64/f32, d = 1, CSR f64/f32, empty buckets, zero matrix, t > n) and
  apply_right, plus the inputs.
* ``configs.json``    -- full-size digests for BASELINE configs 1 and 2 (the
  inputs are regenerated bit-identically from their numpy seeds on the box):
  sha256 of h (uint32 LE), s (int8), SA (fp64 C-order) and the sketch-and-solve
  x / residual, plus a leverage-score pipeline case.
* ``seeds.json``      -- SeedSequence.generate_state / PCG64 state vectors.

numpy / scipy versions are recorded; the digests assume the same versions on
the box (the same image).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np
import scipy
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import sketchnla  # noqa: E402  (the reference, from PYTHONPATH)
from sketchnla import sketch as RS  # noqa: E402
from sketchnla.leverage import _basis_change  # noqa: E402
from sketchnla.linalg import DEFAULT_TOL, pivoted_qr_rank  # noqa: E402
from sketchnla.regress import sketch_solve_ls  # noqa: E402

from tests.synth import config1, config2, lev_case, lowrank_case  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hash_cases():
    cases = [
        (100, 1, 3),
        (5000, 2, 7),
        (20000, 4000, 1),
        (20000, 25000, 2),
        (20000, 65536, 3),
        (20000, 16384, 4),
        (20000, 400, 5),
        (20000, 7, 6),
        (20000, 3 * 2**30, 8),
        (20000, 2**31 + 1, 9),
        (20000, 2**32, 10),
        (4097, 12345, 2**40 + 17),
        (1, 5, 0),
    ]
    out = {}
    meta = []
    for k, (n, t, seed) in enumerate(cases):
        h = RS._rng(seed, 0, 0).integers(0, t, size=n)
        s = RS._rng(seed, 0, 1).choice(np.array([-1.0, 1.0]), size=n)
        out[f"h{k}"] = h.astype(np.uint32)
        out[f"s{k}"] = s.astype(np.int8)
        meta.append([n, t, seed])
    out["meta"] = np.asarray(meta, dtype=object)
    np.savez_compressed(os.path.join(HERE, "hash_cases.npz"), **{k: v for k, v in out.items() if k != "meta"},
                        meta=np.asarray(meta, dtype=np.float64))
    with open(os.path.join(HERE, "hash_cases.json"), "w") as f:
        json.dump(meta, f)


def apply_cases():
    g = np.random.default_rng(20240817)
    out = {}
    meta = []

    def add(name, n, t, seed, a):
        op = RS.SparseEmbedding(n, t, seed)
        sa = op.apply(a)
        if sp.issparse(a):
            a = sp.csr_array(a)
            out[f"{name}_indptr"] = a.indptr
            out[f"{name}_indices"] = a.indices
            out[f"{name}_data"] = a.data
            out[f"{name}_shape"] = np.asarray(a.shape)
            kind = "csr"
        else:
            out[f"{name}_a"] = a
            kind = "dense"
        out[f"{name}_sa"] = sa
        meta.append({"name": name, "n": n, "t": t, "seed": seed, "kind": kind})

    add("dense_f64", 300, 40, 1, g.standard_normal((300, 7)))
    add("dense_f32", 300, 40, 2, g.standard_normal((300, 33)).astype(np.float32))
    add("dense_d1", 500, 64, 3, g.standard_normal(500))
    add("dense_wide", 200, 16, 4, g.standard_normal((200, 300)))
    add("dense_tn", 5, 7, 3, g.standard_normal((5, 3)))  # t > n: empty buckets
    add("dense_zero", 50, 8, 0, np.zeros((50, 4)))
    add("dense_t1", 64, 1, 11, g.standard_normal((64, 5)))
    add("dense_rej", 1000, 3 * 2**20 + 1, 12, g.standard_normal((1000, 3)))
    m = sp.random_array((400, 30), density=0.2, rng=g, format="csr")
    add("csr_f64", 400, 37, 5, m)
    m32 = sp.csr_array(sp.random_array((1000, 64), density=0.25, rng=g, format="csr"), dtype=np.float32)
    add("csr_f32", 1000, 128, 6, m32)
    dup = sp.csr_array((np.array([1.0, 2.0, 3.0, 4.0, 5.0]), np.array([1, 1, 0, 2, 2]), np.array([0, 2, 3, 5])),
                       shape=(3, 4))
    add("csr_dup", 3, 2, 7, dup)
    add("csr_empty_rows", 200, 20, 8, sp.random_array((200, 10), density=0.02, rng=g, format="csr"))

    # apply_right (column sketch), dense and CSR
    op = RS.SparseEmbedding(60, 9, 13)
    ad = g.standard_normal((25, 60))
    out["right_dense_a"] = ad
    out["right_dense_y"] = RS.apply_right(ad, op)
    ac = sp.random_array((25, 60), density=0.3, rng=g, format="csr")
    ac = sp.csr_array(ac)
    out["right_csr_indptr"], out["right_csr_indices"], out["right_csr_data"] = ac.indptr, ac.indices, ac.data
    out["right_csr_y"] = RS.apply_right(ac, op)
    meta.append({"name": "right", "n": 60, "t": 9, "seed": 13, "kind": "right"})

    np.savez_compressed(os.path.join(HERE, "apply_cases.npz"), **out)
    with open(os.path.join(HERE, "apply_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)


def configs():
    res = {"numpy": np.__version__, "scipy": scipy.__version__, "sketchnla": sketchnla.__version__}
    # ---- config 1: dense fp64 100k x 20, m = 4000, sketch-and-solve
    a, b, seed = config1()
    op = RS.make_sparse_embedding(a.shape[0], 4000, seed)
    sa = op.apply(a)
    sb = op.apply(b)
    sol = sketch_solve_ls(a, b, eps=0.5, seed=seed, operator=op)
    res["config1"] = {
        "n": a.shape[0], "d": a.shape[1], "t": 4000, "seed": seed,
        "sha_a": sha(a), "sha_b": sha(b), "sha_h": sha(op.bucket.astype(np.uint32)), "sha_s": sha(op.sign.astype(np.int8)),
        "sha_sa": sha(sa), "sha_sb": sha(sb), "sha_x": sha(sol.x),
        "x": sol.x.ravel().tolist(), "residual_norm": sol.residual_norm,
        "sa_fro": float(np.linalg.norm(sa)),
    }
    # ---- config 2: CSR fp64 1e6 x 50, 5 nnz/row, m = 25000
    a, b, seed = config2()
    op = RS.make_sparse_embedding(a.shape[0], 25000, seed)
    sa = op.apply(a)
    sb = op.apply(b)
    sol = sketch_solve_ls(a, b, eps=0.5, seed=seed, operator=op)
    res["config2"] = {
        "n": a.shape[0], "d": a.shape[1], "t": 25000, "seed": seed,
        "sha_indices": sha(a.indices), "sha_data": sha(a.data), "sha_b": sha(b),
        "sha_h": sha(op.bucket.astype(np.uint32)), "sha_s": sha(op.sign.astype(np.int8)),
        "sha_sa": sha(sa), "sha_sb": sha(sb), "sha_x": sha(sol.x),
        "x": sol.x.ravel().tolist(), "residual_norm": sol.residual_norm,
    }
    # ---- leverage contraction pipeline (config-4 shape, scaled down), fp64 CSR
    a, m, k, seed = lev_case()
    sub = np.random.SeedSequence(seed, spawn_key=(100,)).generate_state(3)
    s = RS.make_sparse_embedding(a.shape[0], m, int(sub[0]))
    sa = s.apply(a)
    n_mat, rank = _basis_change(sa, DEFAULT_TOL)
    g = RS.make_gaussian_jl(k, rank, int(sub[2]))
    probe = n_mat @ g.entries.T
    rows = np.asarray(a @ probe)
    scores = np.einsum("ij,ij->i", rows, rows)
    np.savez_compressed(os.path.join(HERE, "lev_case.npz"), probe=probe, scores=scores, sa=sa)
    res["lev"] = {"n": a.shape[0], "d": a.shape[1], "m": m, "k": k, "seed": seed, "rank": rank,
                  "sha_sa": sha(sa), "sha_probe": sha(probe)}
    # ---- approx_leverage_scores end to end (sparse embedding + SRHT + JL probe + median)
    from sketchnla.leverage import approx_leverage_scores

    g5 = np.random.default_rng(55)
    dense = g5.standard_normal((5000, 6)) * (g5.random((5000, 6)) < 0.5)
    lv = approx_leverage_scores(sp.csr_array(dense), eps=0.5, repetitions=3, seed=9)
    np.savez_compressed(os.path.join(HERE, "approx_lev.npz"), a=dense, scores=lv.scores)
    res["approx_lev"] = {"eps": 0.5, "repetitions": 3, "seed": 9, "rank": lv.rank}
    # ---- low_rank_approx with explicit sparse-embedding sketches (config-5 shape, scaled)
    from sketchnla.lowrank import low_rank_approx

    a, k, seed, t_r, t_s = lowrank_case()
    r_op = RS.make_sparse_embedding(a.shape[1], t_r, 11)
    s_op = RS.make_sparse_embedding(a.shape[0], t_s, 12)
    lr = low_rank_approx(a, k, 0.5, seed=seed, r_op=r_op, s_op=s_op)
    np.savez_compressed(os.path.join(HERE, "lowrank_case.npz"), l=lr.factors.l, d=lr.factors.d,
                        w=lr.factors.w)
    res["lowrank"] = {"k": k, "seed": seed, "t_r": t_r, "t_s": t_s, "err": lr.err, "cond_su": lr.cond_su,
                      "r_op_seed": 11, "s_op_seed": 12, "eps": 0.5}
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(res, f, indent=1)


def srht_cases():
    """SrhtOperator(n, t, seed).apply on seeded inputs (sketch.py:241-297): the
    reference's own SRHT, for the GPU transform's bit-exact check."""
    g = np.random.default_rng(777)
    out, meta = {}, []
    for k, (n, d, t, seed) in enumerate([(1, 3, 1, 0), (5, 2, 4, 1), (1000, 7, 300, 2), (4097, 33, 700, 3),
                                          (20_000, 6, 2_000, 4)]):
        a = g.standard_normal((n, d))
        out[f"a{k}"] = a
        out[f"y{k}"] = RS.SrhtOperator(n, t, seed).apply(a)
        meta.append([n, d, t, seed])
    out["meta"] = np.asarray(meta, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "srht_cases.npz"), **out)


def gse_cases():
    """GeneralizedSparseEmbedding (sketch.py:176-238): its hashes and S.A on
    dense (fp64, fp32, 1-D) and CSR (canonical and with duplicate columns)."""
    g = np.random.default_rng(4242)
    out, meta = {}, []
    for k, (n, r, eps, delta, seed) in enumerate([(3000, 4, 0.5, 0.1, 7), (5000, 3, 0.4, 0.2, 11), (17, 2, 0.5, 0.5, 1)]):
        op = RS.GeneralizedSparseEmbedding(n, r, eps, delta, seed)
        out[f"outer{k}"] = op.outer_bucket.astype(np.uint32)
        out[f"inner{k}"] = op.inner_bucket.astype(np.uint32)
        out[f"sign{k}"] = op.inner_sign.astype(np.int8)
        a64 = g.standard_normal((n, 5))
        a32 = g.standard_normal((n, 7)).astype(np.float32)
        a1 = g.standard_normal(n)
        ac = sp.csr_array(sp.random_array((n, 40), density=0.1, rng=g, format="csr"))
        dup = sp.csr_array((np.array([1.5, -2.0, 0.25, 3.0]), np.array([3, 3, 0, 3]), np.array([0, 2, 4] + [4] * (n - 2))),
                           shape=(n, 5))
        out[f"a64_{k}"], out[f"a32_{k}"], out[f"a1_{k}"] = a64, a32, a1
        out[f"ac_indptr{k}"], out[f"ac_indices{k}"], out[f"ac_data{k}"] = ac.indptr, ac.indices, ac.data
        out[f"sa64_{k}"], out[f"sa32_{k}"], out[f"sa1_{k}"] = op.apply(a64), op.apply(a32), op.apply(a1)
        out[f"sac_{k}"], out[f"sadup_{k}"] = op.apply(ac), op.apply(dup)
        meta.append([n, r, eps, delta, seed, op.q, op.k_blocks, op.v, op.output_dim])
    out["meta"] = np.asarray(meta, dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "gse_cases.npz"), **out)


def mm_cases():
    """load_matrix_market (io.py:37-104) on the texts of tests/golden/mm_cases.py:
    canonical CSR arrays, and the error message for each malformed file."""
    import tempfile

    from sketchnla.io import load_matrix_market

    from tests.golden.mm_cases import BAD, GOOD, NONFINITE

    out, errors = {}, {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in GOOD.items():
            p = os.path.join(tmp, f"{name}.mtx")
            with open(p, "w") as f:
                f.write(text)
            m = load_matrix_market(p)
            out[f"{name}_indptr"], out[f"{name}_indices"], out[f"{name}_data"] = m.indptr, m.indices, m.data
            out[f"{name}_shape"] = np.asarray(m.shape)
        for name, text in {**BAD, **NONFINITE}.items():
            p = os.path.join(tmp, f"{name}.mtx")
            with open(p, "w") as f:
                f.write(text)
            try:
                load_matrix_market(p)
                errors[name] = None
            except ValueError as e:
                errors[name] = str(e).replace(p, "{path}")
    np.savez_compressed(os.path.join(HERE, "mm_cases.npz"), **out)
    with open(os.path.join(HERE, "mm_errors.json"), "w") as f:
        json.dump(errors, f, indent=1)


def seeds():
    rows = []
    for seed, key in [(0, ()), (1, (0, 0)), (1, (0, 1)), (5, (3,)), (2**40 + 17, (0, 0)),
                      (2**70 + 3, (100, 2)), (123456789, (7, 1)), (4294967295, (0, 1))]:
        ss = np.random.SeedSequence(seed, spawn_key=key)
        st = np.random.PCG64(ss).state["state"]
        raw = np.random.PCG64(np.random.SeedSequence(seed, spawn_key=key)).random_raw(8)
        rows.append({"seed": seed, "key": list(key), "gen4": ss.generate_state(4).tolist(),
                     "state": str(st["state"]), "inc": str(st["inc"]), "raw8": [str(int(x)) for x in raw]})
    with open(os.path.join(HERE, "seeds.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    assert "reference" in os.path.dirname(sketchnla.__file__), sketchnla.__file__
    if sys.argv[1:] == ["mm"]:  # regenerate only the Matrix Market fixtures
        mm_cases()
        sys.exit(0)
    seeds()
    srht_cases()
    gse_cases()
    mm_cases()
    hash_cases()
    apply_cases()
    configs()
    print("golden fixtures written to", HERE)
