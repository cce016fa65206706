"""Rebind the reference package onto the GPU operator.

The reference resolves ``SparseEmbedding`` as a module global at call time in
make_sparse_embedding (sketch.py:400), sparse_embedding_or_identity
(sketch.py:426) and from_descriptor (sketch.py:465), so replacing that one
attribute sends every caller -- sketch_solve_ls (regress.py:106), precondition
(regress.py:174), nonneg_regression (regress.py:351), approx_leverage_scores
(leverage.py:74), low_rank_approx (lowrank.py:156,159,181), verify.py -- through
the B200 kernels.  ``apply_right`` is also rebound (sketch.py:445-448 and the
name imported by lowrank.py:29) so the column sketch is transpose-free, and
``SrhtOperator`` (resolved at call time by srht_or_identity, sketch.py:433) so
the SRHT stages of precondition, nonneg_regression, approx_leverage_scores and
the srht_compose low-rank strategy run on the GPU too.
"""

from __future__ import annotations

import importlib

from . import generalized as _gen
from . import sketch as _gpu
from . import solvers as _sol

_saved: dict = {}


def install() -> None:
    ref = importlib.import_module("sketchnla.sketch")
    low = importlib.import_module("sketchnla.lowrank")
    lp = importlib.import_module("sketchnla.lp")
    if not _saved:
        _saved["SparseEmbedding"] = ref.SparseEmbedding
        _saved["apply_right"] = ref.apply_right
        _saved["low.apply_right"] = low.apply_right
        _saved["GeneralizedSparseEmbedding"] = ref.GeneralizedSparseEmbedding
        _saved["lp.GeneralizedSparseEmbedding"] = lp.GeneralizedSparseEmbedding
        _saved["SrhtOperator"] = ref.SrhtOperator
    ref.SparseEmbedding = _gpu.SparseEmbedding
    ref.apply_right = _gpu.apply_right
    low.apply_right = _gpu.apply_right
    ref.GeneralizedSparseEmbedding = _gen.GeneralizedSparseEmbedding
    lp.GeneralizedSparseEmbedding = _gen.GeneralizedSparseEmbedding
    ref.SrhtOperator = _sol.SrhtOperator


def uninstall() -> None:
    if not _saved:
        return
    ref = importlib.import_module("sketchnla.sketch")
    low = importlib.import_module("sketchnla.lowrank")
    lp = importlib.import_module("sketchnla.lp")
    ref.SparseEmbedding = _saved["SparseEmbedding"]
    ref.apply_right = _saved["apply_right"]
    low.apply_right = _saved["low.apply_right"]
    ref.GeneralizedSparseEmbedding = _saved["GeneralizedSparseEmbedding"]
    lp.GeneralizedSparseEmbedding = _saved["lp.GeneralizedSparseEmbedding"]
    ref.SrhtOperator = _saved["SrhtOperator"]
    _saved.clear()
