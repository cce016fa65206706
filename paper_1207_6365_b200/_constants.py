"""Sketch-size constants, restated from the reference's calibrated values
(/root/reference/pkg/src/sketchnla/_constants.py:9-39).  Only the ones the
CountSketch path and its callers read are kept; default_sparse_dim
(sketch.py:56-66) depends on SPARSE_DIM_C / SPARSE_DIM_FLOOR."""

SPARSE_DIM_C = 1.0
SPARSE_DIM_FLOOR = 4

# SRHT rows t = C (sqrt r + sqrt log n)^2 log(r + 1) / eps^2 (sketch.py:83-94)
SRHT_DIM_C = 1.5

# leverage.py:100-107 and :87 (JL probe width)
LEVERAGE_F_C = 40.0
LEVERAGE_JL_C = 16.0

# generalized sparse embedding dims (sketch.py:69-80, _constants.py:13-19)
GEN_K_C = 1.0
GEN_V_C = 1.0
GEN_Q_C = 1.0
