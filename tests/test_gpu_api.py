"""The drop-in boundary on the GPU: descriptor round trips land on this
package's GPU classes (reference from_descriptor, sketch.py:460-478), and
input layouts the reference accepts (broadcast / strided views) are read
correctly."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
import paper_1207_6365_b200 as skb
from paper_1207_6365_b200 import sketch as S

pytestmark = pytest.mark.gpu


def test_from_descriptor_returns_gpu_classes_for_every_owned_family():
    ops = [
        skb.SparseEmbedding(1000, 64, 3),
        skb.GeneralizedSparseEmbedding(1000, 4, 0.5, 0.25, 7),
        skb.SrhtOperator(1000, 40, 5),
        skb.SrhtOperator(300, 300, 5, all_rows=True),
        S.IdentityOperator(17),
    ]
    ops.append(S.compose(skb.SrhtOperator(64, 16, 2), skb.SparseEmbedding(1000, 64, 3)))
    rng = np.random.default_rng(0)
    for op in ops:
        back = S.from_descriptor(op.descriptor())
        assert type(back) is type(op), (type(back), type(op))
        assert back.descriptor() == op.descriptor()
        a = rng.standard_normal((op.input_dim, 3))
        assert np.array_equal(np.asarray(back.apply(a)), np.asarray(op.apply(a)))
    comp = S.from_descriptor(ops[-1].descriptor())
    assert type(comp.outer) is skb.SrhtOperator and type(comp.inner) is skb.SparseEmbedding


def test_broadcast_and_strided_views():
    """x[None].expand(n, d) has row stride 0: materialised before K3 reads it
    (an n*d read of a d-element allocation would run out of bounds)."""
    n, d, t = 5000, 128, 300
    op = skb.SparseEmbedding(n, t, 4)
    h, s = O.hash_signs(n, t, 4)
    x = torch.randn(d, dtype=torch.float32, device="cuda")
    got = op.apply(x[None].expand(n, d))
    ref = O.apply_dense(h, s, t, np.broadcast_to(x.cpu().numpy()[None], (n, d)))
    assert np.array_equal(got.cpu().numpy(), ref)
    # a column slice (row stride > d) and a transposed view (column stride != 1)
    big = torch.randn(n, 2 * d, dtype=torch.float64, device="cuda")
    assert np.array_equal(op.apply(big[:, 5:5 + d]).cpu().numpy(),
                          O.apply_dense(h, s, t, big[:, 5:5 + d].cpu().numpy()))
    tt = torch.randn(d, n, dtype=torch.float64, device="cuda").T
    assert np.array_equal(op.apply(tt).cpu().numpy(), O.apply_dense(h, s, t, tt.cpu().numpy()))
