"""Row-window CSR kernels (opt-in): csrc/csr_window.cuh (SKT_CSR_WINDOW=1, rows
routed through an L2 slot ring) and csrc/csr_cta.cuh (SKT_CSR_WINDOW=cta, window
gather with SM-owned buckets).  S.A bit-identical to the oracle's restatement of sketch.py:155-164 and to the
default per-bucket kernel, over window tails, empty rows, rows longer than a
slot (read straight from A), int64 indptr, d not a multiple of 64 and both
output dtypes."""

import numpy as np
import pytest
import scipy.sparse as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _csr(n, d, dens, longfrac, rng):
    m = sp.random_array((n, d), density=dens, rng=rng, format="csr", dtype=np.float32)
    if longfrac:
        lil = m.tolil()
        for r in np.flatnonzero(rng.random(n) < longfrac)[:500]:
            lil[r, :] = rng.standard_normal(d).astype(np.float32)
        m = sp.csr_array(lil.tocsr())
    m.sort_indices()
    return m


@pytest.mark.parametrize(
    "n,d,t,dens,longfrac,i64",
    [
        (1000, 64, 50, 0.25, 0.0, False),
        (20_000, 64, 777, 0.25, 0.02, False),
        (60_001, 50, 4000, 0.2, 0.02, True),
        (50_000, 128, 3000, 0.1, 0.01, False),
        (30_000, 7, 100, 0.9, 0.0, False),
        (35, 64, 3, 0.3, 0.1, False),
    ],
)
@pytest.mark.parametrize("mode", ["1", "cta"])
def test_window_kernel_bit_identical(monkeypatch, mode, n, d, t, dens, longfrac, i64):
    from oracle import oracle as O
    from paper_1207_6365_b200 import SparseEmbedding

    monkeypatch.setenv("SKT_CSR_WINDOW", mode)
    rng = np.random.default_rng(n + d)
    m = _csr(n, d, dens, longfrac, rng)
    dev = torch.device("cuda:0")
    ip = torch.from_numpy(m.indptr.astype(np.int64 if i64 else np.int32)).to(dev)
    ix = torch.from_numpy(m.indices.astype(np.int32)).to(dev)
    vv = torch.from_numpy(m.data).to(dev)
    op = SparseEmbedding(n, t, 11, device=dev)
    plan = op.cta_plan(d) if mode == "cta" else op.window_plan(d)
    assert plan is not None and op._window_mode(ip, ix, vv) == mode
    h, s = O.hash_signs(n, t, 11)
    ref = O.apply_csr(h, s, t, m)
    got64 = op._apply_csr_device(ip, ix, vv, d, torch.float64, True).cpu().numpy()
    assert np.array_equal(got64, ref)
    got32 = op._apply_csr_device(ip, ix, vv, d, torch.float32, True).cpu().numpy()
    assert np.array_equal(got32, ref.astype(np.float32))
    # the default kernel (explicit shift bypasses the window path)
    tile = op._apply_csr_device(ip, ix, vv, d, torch.float64, True, shift=0).cpu().numpy()
    assert np.array_equal(tile, got64)


@pytest.mark.parametrize("mode", ["1", "cta"])
def test_window_kernel_multi_window_and_empty_rows(monkeypatch, mode):
    """More rows than one window (W = 148 x 1024 on B200) with a ragged tail,
    empty rows and an all-empty leading block."""
    from oracle import oracle as O
    from paper_1207_6365_b200 import SparseEmbedding

    monkeypatch.setenv("SKT_CSR_WINDOW", mode)
    rng = np.random.default_rng(3)
    n, d, t = 151_552 * 2 + 17, 64, 16_384
    m = _csr(n, d, 0.25, 0.01, rng).tolil()
    m[:300, :] = 0
    m = sp.csr_array(m.tocsr())
    m.eliminate_zeros()
    m.sort_indices()
    dev = torch.device("cuda:0")
    ip, ix, vv = (torch.from_numpy(x).to(dev) for x in (m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data))
    op = SparseEmbedding(n, t, 5, device=dev)
    assert (op.cta_plan(d) if mode == "cta" else op.window_plan(d)) is not None
    h, s = O.hash_signs(n, t, 5)
    got = op._apply_csr_device(ip, ix, vv, d, torch.float64, True).cpu().numpy()
    assert np.array_equal(got, O.apply_csr(h, s, t, m))


def test_window_plan_matches_stable_sort():
    """pos / wpi = the rows of every window stably sorted by bucket."""
    from paper_1207_6365_b200 import SparseEmbedding

    n, t = 400_000, 1000
    op = SparseEmbedding(n, t, 2, device=torch.device("cuda:0"))
    plan = op.window_plan(64)
    assert plan is not None
    w, pos, wpi = plan
    pos = pos.cpu().numpy().view(np.uint32)
    wpi = wpi.cpu().numpy()
    h = op.bucket
    for win in range(wpi.shape[0]):
        r0, r1 = win * w, min(n, (win + 1) * w)
        order = np.argsort(h[r0:r1], kind="stable")
        want = np.empty(r1 - r0, dtype=np.int64)
        want[order] = np.arange(r1 - r0)
        assert np.array_equal(pos[r0:r1] & 0x7FFFFFFF, want)
        assert np.array_equal((pos[r0:r1] >> 31).astype(np.float64), (op.sign[r0:r1] < 0).astype(np.float64))
        counts = np.bincount(h[r0:r1], minlength=t)
        assert np.array_equal(wpi[win], np.concatenate([[0], np.cumsum(counts)]))


def test_cta_plan_rows_are_the_inverse_of_pos():
    """wrows (csr_cta) lists every window's rows in the order pos ranks them."""
    from paper_1207_6365_b200 import SparseEmbedding

    n, t = 300_000, 700
    op = SparseEmbedding(n, t, 4, device=torch.device("cuda:0"))
    plan = op.cta_plan(64)
    assert plan is not None
    w, wrows, wpi = plan
    wrows = wrows.cpu().numpy().view(np.uint32)
    h = op.bucket
    for win in range(wpi.shape[0]):
        r0, r1 = win * w, min(n, (win + 1) * w)
        order = np.argsort(h[r0:r1], kind="stable") + r0
        assert np.array_equal(wrows[r0:r1] & 0x7FFFFFFF, order)
        assert np.array_equal(wrows[r0:r1] >> 31, (op.sign[order] < 0).astype(np.uint32))


def test_cta_kernel_few_buckets_many_rounds(monkeypatch):
    """t smaller than the SM count: one bucket per CTA, windows cut into several
    rounds of the slot ring; and a wide d that only this kernel takes."""
    from oracle import oracle as O
    from paper_1207_6365_b200 import SparseEmbedding

    monkeypatch.setenv("SKT_CSR_WINDOW", "cta")
    rng = np.random.default_rng(9)
    dev = torch.device("cuda:0")
    for n, d, t in [(200_000, 64, 20), (100_000, 200, 2000)]:
        m = _csr(n, d, 0.1, 0.01, rng)
        ip, ix, vv = (torch.from_numpy(x).to(dev) for x in (m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data))
        op = SparseEmbedding(n, t, 8, device=dev)
        assert op.cta_plan(d) is not None
        h, s = O.hash_signs(n, t, 8)
        got = op._apply_csr_device(ip, ix, vv, d, torch.float64, True).cpu().numpy()
        assert np.array_equal(got, O.apply_csr(h, s, t, m))
