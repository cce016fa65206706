import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1207_6365_b200 import SparseEmbedding
from tests import synth
a, b, seed = synth.config1()
for n, t, arr in [(100000, 4000, b), (3000, 211, np.random.default_rng(0).standard_normal((3000, 1))), (100000, 4000, a[:, :1].copy()), (100000, 4000, a[:, :2].copy())]:
    op = SparseEmbedding(n, t, seed)
    h, s = O.hash_signs(n, t, seed)
    g = op.apply(arr); r = O.apply_dense(h, s, t, arr)
    bad = np.nonzero(g != r)
    print(n, t, arr.shape, 'mismatch', len(bad[0]), 'maxabs', np.abs(g - r).max(), bad[0][:5], (g - r)[bad][:3])
