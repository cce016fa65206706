"""Golden vectors for the preconditioned iterations and the rank-k Gram
residual, from the REFERENCE itself (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_precond.py

Records, for tests/synth.py's precond_cases(), the reference's
``precondition`` (regress.py:159-189: r_inv, rank, sketch_dim) and its
``richardson_solve`` / ``cgnr_solve`` (regress.py:226-285: x, iterations,
residual history, residual); for gram_cases() the factors (L, d, W) and
``lowrank._residual_norm`` (lowrank.py:100-108, the Gram-identity branch);
for nnls_cases() ``nonneg_regression`` (regress.py:330-370: x, residual,
sketch_dim); for lowrank_default_case() ``low_rank_approx`` with the default
"srht_compose" strategy (lowrank.py:111-222: factors, err, cond_su, t_r, t_s).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import sketchnla  # noqa: E402  (the reference, from PYTHONPATH)
from sketchnla import lowrank as RL  # noqa: E402
from sketchnla import regress as RR  # noqa: E402

from tests.synth import gram_cases, lowrank_default_case, nnls_cases, precond_cases  # noqa: E402


def main():
    assert "reference" in os.path.dirname(sketchnla.__file__), sketchnla.__file__
    out = {}
    for name, (a, b, eps0, seed) in precond_cases().items():
        pre = RR.precondition(a, eps0, seed=seed)
        out[f"{name}/r_inv"] = pre.r_inv
        out[f"{name}/rank"] = np.int64(pre.rank)
        out[f"{name}/sketch_dim"] = np.int64(pre.sketch_dim)
        for method, fn in (("richardson", RR.richardson_solve), ("cgnr", RR.cgnr_solve)):
            sol = fn(a, pre, b, 1e-6, max_iter=60)
            out[f"{name}/{method}/x"] = sol.x
            out[f"{name}/{method}/iterations"] = np.int64(sol.iterations)
            out[f"{name}/{method}/history"] = np.asarray(sol.residual_history)
            out[f"{name}/{method}/residual"] = np.float64(sol.residual_norm)
    rng = np.random.default_rng(44)
    for name, a in gram_cases().items():
        n, m = a.shape
        k = 5
        l, _ = np.linalg.qr(rng.standard_normal((n, k)))
        w, _ = np.linalg.qr(rng.standard_normal((m, k)))
        d = np.sort(rng.random(k) * 50.0)[::-1].copy()
        out[f"gram_{name}/l"] = l
        out[f"gram_{name}/w"] = w
        out[f"gram_{name}/d"] = d
        out[f"gram_{name}/value"] = np.float64(RL._residual_norm(a, l, d, w))
    for name, (a, b, eps, seed) in nnls_cases().items():
        sol = RR.nonneg_regression(a, b, eps, seed=seed)
        out[f"nnls_{name}/x"] = sol.x
        out[f"nnls_{name}/residual"] = np.float64(sol.residual_norm)
        out[f"nnls_{name}/sketch_dim"] = np.int64(sol.sketch_dim)
    res = RL.low_rank_approx(lowrank_default_case(), 5, 0.5, seed=11)
    for key in ("l", "d", "w"):
        out[f"lowrank_default/{key}"] = getattr(res.factors, key)
    out["lowrank_default/err"] = np.float64(res.err)
    out["lowrank_default/cond_su"] = np.float64(res.cond_su)
    out["lowrank_default/t_r"] = np.int64(res.t_r)
    out["lowrank_default/t_s"] = np.int64(res.t_s)
    srht = sketchnla.sketch.SrhtOperator(1000, 300, 2)
    out["srht_views/sign"] = srht.sign
    out["srht_views/rows"] = srht.sampled_rows
    out["versions"] = np.array([np.__version__, __import__("scipy").__version__])
    np.savez_compressed(os.path.join(HERE, "precond_cases.npz"), **out)
    print({k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items() if "iterations" in k or "rank" in k})


if __name__ == "__main__":
    main()
