"""A/B of the row-window CSR kernel (csr_window.cuh) against csr_tile on the GPU.

Checks that the window kernel's SA is bit-identical to the per-bucket tile
kernel's (itself pinned to the reference by the parity tests) on a set of
small shapes (tails, empty rows, long rows, int64 indptr, d not a multiple of
64) and on a BASELINE config, then times both with CUDA events.

    python tools/csr_window_ab.py --config c4 [--small-only]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def small_cases(torch, SparseEmbedding, dev):
    import numpy as np
    import scipy.sparse as sp

    rng = np.random.default_rng(5)
    ok = True
    for (n, d, t, dens, longfrac, i64) in [
        (1000, 64, 50, 0.25, 0.0, False),
        (50_000, 64, 777, 0.25, 0.01, False),
        (200_001, 50, 4000, 0.2, 0.02, True),
        (300_000, 128, 3000, 0.1, 0.01, False),
        (151_552 * 2 + 17, 64, 16_384, 0.25, 0.01, False),
        (40_000, 7, 100, 0.9, 0.0, False),
        (120_000, 200, 2000, 0.05, 0.005, False),
    ]:
        m = sp.random_array((n, d), density=dens, rng=rng, format="csr", dtype=np.float32)
        if longfrac:
            dense_rows = np.flatnonzero(rng.random(n) < longfrac)
            lil = m.tolil()
            for r in dense_rows[:2000]:
                lil[r, :] = rng.standard_normal(d).astype(np.float32)
            m = sp.csr_array(lil.tocsr())
        m.sort_indices()
        ip = torch.from_numpy(m.indptr.astype(np.int64 if i64 else np.int32)).to(dev)
        ix = torch.from_numpy(m.indices.astype(np.int32)).to(dev)
        vv = torch.from_numpy(m.data.astype(np.float32)).to(dev)
        op = SparseEmbedding(n, t, 3, device=dev)
        for odt in (torch.float64, torch.float32):
            ref = op._apply_csr_device(ip, ix, vv, d, odt, True, shift=0)
            assert op._window_eligible(ip, ix, vv, d, vv.numel())
            plan = op.cta_plan(d) if os.environ["SKT_CSR_WINDOW"] == "cta" else op.window_plan(d)
            if plan is None:
                print(f"n={n} d={d} t={t}: window kernel not applicable", flush=True)
                continue
            got = op._apply_csr_device(ip, ix, vv, d, odt, True)
            torch.cuda.synchronize()
            view = torch.int64 if odt == torch.float64 else torch.int32
            same = bool(torch.equal(got.view(view), ref.view(view)))
            ok &= same
            print(f"n={n} d={d} t={t} nnz={vv.numel()} i64={i64} out={odt}: bit-identical {same}", flush=True)
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--small-only", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    ap.add_argument("--kernel", default="1", choices=["1", "cta"], help="1: csr_window, cta: csr_cta")
    args = ap.parse_args()
    import torch

    import bench
    from paper_1207_6365_b200 import SparseEmbedding

    dev = torch.device("cuda:0")
    os.environ["SKT_CSR_WINDOW"] = args.kernel  # the kernels are opt-in
    if not args.skip_small:
        ok = small_cases(torch, SparseEmbedding, dev)
        print("small cases:", "OK" if ok else "MISMATCH", flush=True)
    if args.small_only:
        return
    cfg = bench.CONFIGS[args.config]
    ip, ix, vv = bench.gen_csr_shard(torch, cfg, 0, cfg["n"], dev)
    op = SparseEmbedding(cfg["n"], cfg["m"], cfg["seed"], device=dev)
    odt = torch.float32
    alg = vv.numel() * (vv.element_size() + 4) + ip.numel() * ip.element_size() + cfg["m"] * cfg["d"] * 4
    ref = op._apply_csr_device(ip, ix, vv, cfg["d"], odt, True, shift=0)
    got = op._apply_csr_device(ip, ix, vv, cfg["d"], odt, True)
    torch.cuda.synchronize()
    print("kernel", args.kernel, "bit-identical to csr_tile:", bool(torch.equal(got.view(torch.int32), ref.view(torch.int32))), flush=True)
    for name, kw in (("csr_tile", dict(shift=0)), ("csr_window", dict())):
        out = torch.empty_like(ref)
        times = []
        for _ in range(args.iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op._apply_csr_device(ip, ix, vv, cfg["d"], odt, True, out=out, **kw)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        times.sort()
        ms = times[len(times) // 2]
        print(f"{args.config} {name}: median {ms:.4f} ms, min {times[0]:.4f} ms "
              f"({alg / ms / 1e6:.0f} GB/s algorithmic)", flush=True)


if __name__ == "__main__":
    main()
