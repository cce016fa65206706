"""paper_1207_6365_b200 -- B200-native CountSketch (sparse embedding) hot path
of Clarkson-Woodruff input-sparsity-time sketching (arXiv 1207.6365).

A drop-in for the reference package's SparseEmbedding / sketch-apply path
(/root/reference/pkg/src/sketchnla/sketch.py:138-173) backed by hand-written
sm_100a CUDA kernels behind the C ABI in include/sketch_b200.h.
"""

from ._lib import SketchError, launch_count
from .sketch import (
    ComposedSketch,
    IdentityOperator,
    SparseEmbedding,
    apply_left,
    apply_right,
    compose,
    default_sparse_dim,
    derived_seed,
    from_descriptor,
    make_sparse_embedding,
    sparse_embedding_or_identity,
    to_descriptor,
)
from .generalized import GeneralizedSparseEmbedding, generalized_dims, make_generalized_sparse_embedding
from .precond import Preconditioner, SolverError, cgnr_solve, precondition, richardson_solve
from .solvers import SrhtOperator, lawson_hanson_nnls, nonneg_regression, srht_or_identity
from .shim import install, uninstall

__version__ = "0.1.0"
