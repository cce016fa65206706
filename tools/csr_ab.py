"""A/B of the CSR S.A kernel families on a BASELINE config (GPU).

For each plan shift (0 = per-bucket plan -> csr_tile; k > 0 = bucket-group
plan -> csr_sweep for rows of 8+ nonzeros, csr_group for short rows) builds the
plan, checks the SA is bit-identical to shift 0's (itself pinned to the
reference by tests/test_gpu_csr.py) and times the kernel with CUDA events
(median of --iters launches; inputs larger than L2, or an L2-flushing write
before every launch when they fit).

    python tools/csr_ab.py --config c4 --shifts 0 1 2 3
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--shifts", type=int, nargs="+", default=[0, 1, 2, 3])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="f32", choices=["f32", "f64"])
    args = ap.parse_args()
    import torch

    import bench
    from paper_1207_6365_b200 import SparseEmbedding

    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda:0")
    ip, ix, vv = bench.gen_csr_shard(torch, cfg, 0, cfg["n"], dev)
    op = SparseEmbedding(cfg["n"], cfg["m"], cfg["seed"], device=dev)
    odt = torch.float32 if args.out == "f32" else torch.float64
    alg = vv.numel() * (vv.element_size() + 4) + ip.numel() * ip.element_size() + cfg["m"] * cfg["d"] * (4 if args.out == "f32" else 8)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if alg < 4 * (126 << 20) else None
    ref = None
    for shift in args.shifts:
        op.grouped_plan(shift)
        out = op._apply_csr_device(ip, ix, vv, cfg["d"], odt, True, shift=shift)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out.view(torch.int32 if odt == torch.float32 else torch.int64),
                                ref.view(torch.int32 if odt == torch.float32 else torch.int64)))
        times = []
        for _ in range(args.iters):
            if flush is not None:
                flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op._apply_csr_device(ip, ix, vv, cfg["d"], odt, True, out=out, shift=shift)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        times.sort()
        ms = times[len(times) // 2]
        print(f"{args.config} shift={shift} R={os.environ.get('SKT_SWEEP_R', '-')}: {ms:.4f} ms "
              f"({alg / ms / 1e6:.0f} GB/s algorithmic), bit-identical to shift 0: {same}", flush=True)


if __name__ == "__main__":
    main()
