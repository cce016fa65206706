#!/usr/bin/env python3
"""Benchmark of the CountSketch S.A hot path (BASELINE.json metric:
"CountSketch S.A nonzeros/sec and % of HBM roofline at 1/2/4/8 B200").

Default workload = BASELINE config 3 (the config the metric's 1/2/4/8-GPU
clause is quoted on): dense fp32 A, n = 16,777,216 x d = 128 (8.6 GB), rows
N(0,1) scaled by lognormal(0,1), CountSketch m = 65,536; S.A only, rows
sharded across the N ranks, partial m x d SA all-reduced with NCCL (strong
scaling: total n fixed).  A step = one S.A over the rank's shard (+ the
all-reduce when N > 1), inputs resident in HBM.  Each SA entry is accumulated
in fp64 in ascending row order (bit-identical to the reference) and written
as fp32.  Synthetic data (no dataset is named); inputs (8.6 GB) exceed the
126 MB L2, so no flush is needed between steps.

Run:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
      torchrun --nproc-per-node N bench.py --gpus N ...
Other configs for profiling: --config c1|c2|c4 (not the headline line).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
L2_FLUSH_BELOW = 4 * 126 * 2**20  # inputs below 4x the 126 MB L2 get an L2 flush per step
sys.path.insert(0, ROOT)

METRIC = "CountSketch S·A nonzeros/sec and % of HBM roofline at 1/2/4/8 B200"
CONFIGS = {
    "c1": dict(kind="dense", n=100_000, d=20, m=4_000, dtype="f64", seed=1,
               workload="config1: dense fp64 100000x20 N(0,1), m=4000"),
    "c2": dict(kind="csr", n=1_000_000, d=50, m=25_000, dtype="f64", per_row=5, seed=1,
               workload="config2: CSR fp64 1000000x50, 5 nnz/row, m=25000"),
    "c3": dict(kind="dense", n=16_777_216, d=128, m=65_536, dtype="f32", seed=1, lognormal=True,
               workload="config3: dense fp32 16777216x128 (rows N(0,1)*lognormal(0,1)), m=65536, S.A row-sharded + all-reduce"),
    "c4": dict(kind="csr", n=4_194_304, d=64, m=16_384, dtype="f32", per_row=16, dense_frac=0.01, seed=1,
               workload="config4: CSR fp32 4194304x64, 16 nnz/row + 1% dense rows N(0,100), m=16384"),
    "c5": dict(kind="csr", n=262_144, d=262_144, m=400, dtype="f32", per_row=262, lowrank=10, seed=1,
               shard="bucket",
               workload="config5: CSR fp32 262144x262144, 262 nnz/row (0.1%), values (U V^T)_ij + 0.01 N, "
                        "rank 10; m=400 row sketch"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampler thread: SM clock + throttle reasons during the timed region."""

    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "hw_power_brake_slowdown": 0x80}
    OTHER = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
             "sync_boost": 0x10, "display_clock_setting": 0x100}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("nvml unavailable:", e)
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in {**self.BAD, **self.OTHER}.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons - {"gpu_idle"}),
                "samples": len(self.samples)}

    def rejected(self):
        if self.reasons & set(self.BAD):
            return True
        s = self.summary()
        return bool(s["sm_mhz"] and s["sm_max_mhz"] and s["sm_mhz"] < 0.5 * s["sm_max_mhz"]
                    and "sw_power_cap" not in self.reasons)


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def gather_ceiling_ms(cfg_name: str):
    """The config's CSR access pattern run without arithmetic (random row
    order, indptr pair + index / value segments per row; tools/gather_bench.cu,
    profiles/r01_gather_ceiling.json), or None."""
    p = os.path.join(ROOT, "profiles", "r01_gather_ceiling.json")
    try:
        with open(p) as f:
            return float(json.load(f)["csr_pattern_ms"][cfg_name])
    except Exception:
        return None


def dominant_kernel(cfg, lev: bool, args, sa_dt) -> str:
    """Name of the kernel the line's roofline describes (the library picks it by
    shape)."""
    if lev:
        if args.lev_f64:
            return "lev_dmma_kernel (fp64 tensor cores, DMMA.8x8x4)"
        return "lev_tc3_kernel (tcgen05 kind::f16, scaled 2xFP16)"
    if cfg["kind"] == "dense":
        esz = 4 if cfg["dtype"] == "f32" else 8
        rb = cfg["d"] * esz
        if 512 <= rb <= 2048 and rb % 16 == 0 and os.environ.get("SKT_DENSE_G4", "1") != "0":
            return "dense_g4_kernel (TMA tile::gather4 into an mbarrier smem ring)"
        return "apply_dense_kernel (register gather)"
    if args.fast:
        return "csr_atomic_kernel (fast mode: unordered RED.ADD)"
    if cfg["d"] > 25_000:
        return "csr_fine_scatter + csr_fine_accum (deterministic wide-d: entries ordered by 1024-column block, then a warp per (bucket, block) adds in row order)"
    if cfg.get("per_row", 16) <= 8:
        return "csr_group_kernel (grouped sweep)"
    if cfg["dtype"] == "f32" and cfg["d"] <= 64 and os.environ.get("SKT_CSR_KERNEL") not in ("tile", "lane"):
        return "csr_quad_kernel (densify tiles, 128-bit loads, row pointers kept in L2)"
    return "csr_tile_kernel (densify tiles)"


def traffic_for(cfg_name: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg_name)
    except Exception:
        return None


# ---------------------------------------------------------------- data
def gen_dense_shard(torch, cfg, r0, r1, device):
    """Rows [r0, r1) of the synthetic A; generated in fixed 2^20-row blocks with
    per-block seeds, so any sharding yields the same global matrix."""
    blk = 1 << 20
    dt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    out = torch.empty((r1 - r0, cfg["d"]), dtype=dt, device=device)
    g = torch.Generator(device=device)
    for b0 in range((r0 // blk) * blk, r1, blk):
        b1 = min(b0 + blk, cfg["n"])
        g.manual_seed(1_000_003 * (b0 // blk) + 17)
        x = torch.randn((b1 - b0, cfg["d"]), generator=g, device=device, dtype=torch.float32)
        if cfg.get("lognormal"):
            x *= torch.exp(torch.randn((b1 - b0, 1), generator=g, device=device, dtype=torch.float32))
        lo, hi = max(b0, r0), min(b1, r1)
        out[lo - r0 : hi - r0] = x[lo - b0 : hi - b0].to(dt)
    return out


def gen_lowrank_csr_shard(torch, cfg, r0, r1, device):
    """Config 5: rows [r0, r1) of a square CSR with `per_row` distinct columns
    per row (one uniform column in each of `per_row` equal column strata, so
    they are distinct and sorted), values (U V^T)_ij + 0.01 N(0,1) with
    U, V ~ N(0,1)^{n x k}; generated in row chunks with per-chunk seeds."""
    n, d, per, k = cfg["n"], cfg["d"], cfg["per_row"], cfg["lowrank"]
    dt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(99)
    V = torch.randn((d, k), generator=g, device=device)
    stride = d // per
    m = r1 - r0
    indices = torch.empty(m * per, dtype=torch.int32, device=device)
    vals = torch.empty(m * per, dtype=dt, device=device)
    chunk = 1 << 14
    for c0 in range(r0 - r0 % chunk, r1, chunk):
        c1 = min(c0 + chunk, n)
        g.manual_seed(5_000_011 + c0 // chunk)
        U = torch.randn((c1 - c0, k), generator=g, device=device)
        cols = (torch.arange(per, device=device) * stride)[None, :] + torch.randint(
            0, stride, (c1 - c0, per), generator=g, device=device)
        v = (U[:, None, :] * V[cols]).sum(-1) + 0.01 * torch.randn((c1 - c0, per), generator=g, device=device)
        lo, hi = max(c0, r0), min(c1, r1)
        indices[(lo - r0) * per:(hi - r0) * per] = cols[lo - c0:hi - c0].reshape(-1).to(torch.int32)
        vals[(lo - r0) * per:(hi - r0) * per] = v[lo - c0:hi - c0].reshape(-1).to(dt)
    indptr = torch.arange(0, (m + 1) * per, per, device=device, dtype=torch.int64)
    if m * per < 2**31:
        indptr = indptr.to(torch.int32)
    return indptr, indices, vals


def gen_csr_shard(torch, cfg, r0, r1, device):
    """CSR rows [r0, r1): `per_row` distinct uniform columns per row, N(0,1)
    values; a `dense_frac` of rows fully dense with N(0, 100) values (c4)."""
    if cfg.get("lowrank"):
        return gen_lowrank_csr_shard(torch, cfg, r0, r1, device)
    d, per = cfg["d"], cfg["per_row"]
    dt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(7_000_003 + r0)
    m = r1 - r0
    dense_rows = torch.zeros(m, dtype=torch.bool, device=device)
    if cfg.get("dense_frac"):
        dense_rows = torch.rand(m, generator=g, device=device) < cfg["dense_frac"]
    keys = torch.rand((m, d), generator=g, device=device)
    sel = torch.zeros((m, d), dtype=torch.bool, device=device)
    top = torch.topk(keys, per, dim=1).indices
    sel.scatter_(1, top, True)
    sel |= dense_rows[:, None]
    counts = sel.sum(1)
    indptr = torch.zeros(m + 1, dtype=torch.int64, device=device)
    indptr[1:] = torch.cumsum(counts, 0)
    indices = sel.nonzero()[:, 1].to(torch.int32)
    nnz = int(indptr[-1])
    row_of = torch.repeat_interleave(torch.arange(m, device=device), counts)
    scale = torch.where(dense_rows[row_of], 10.0, 1.0)
    vals = (torch.randn(nnz, generator=g, device=device) * scale).to(dt)
    if nnz < 2**31:
        indptr = indptr.to(torch.int32)
    return indptr, indices, vals


# ---------------------------------------------------------------- arms
def reference_arm(args, cfg):
    """The reference's CPU implementation of the path on this host: the oracle
    port of sketch.py:153-165 with the reference's own primitives (dense:
    as_dense's fp64 upcast + finiteness scan, then scipy's CSR @ dense =
    csr_matvecs; CSR: repeat + bincount), single-threaded like the reference
    (numpy / scipy C loops).  The input is the SAME matrix our arm times
    (bench.py's seeded generators, generated on cuda:0 and copied to the host).
    Configs 1, 2, 4, 5: each step is the whole apply.  Config 3 (about 34 s per
    whole apply on one core): each step applies S to one 2^20-row block of the
    full 16.7 M-row matrix, S's columns for those rows (the full operator's
    buckets and signs, the same m x d output), cycling over the 16 blocks so
    16 steps cover the whole workload once."""
    import numpy as np
    import torch

    from oracle import oracle as O

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    n, d, m = cfg["n"], cfg["d"], cfg["m"]
    gen_dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    t_prep = time.perf_counter()
    h, s = O.hash_signs(n, m, cfg["seed"])
    if cfg["kind"] == "dense":
        blk = n if n <= (1 << 20) else (1 << 20)
        a = np.empty((n, d), dtype=np.float32 if cfg["dtype"] == "f32" else np.float64)
        for r0 in range(0, n, blk):
            a[r0:r0 + blk] = gen_dense_shard(torch, cfg, r0, min(n, r0 + blk), gen_dev).cpu().numpy()
        blocks = [(r0, min(n, r0 + blk)) for r0 in range(0, n, blk)]
        mats = [O.np_sketch_matrix(h[r0:r1], s[r0:r1], m, r1 - r0) for r0, r1 in blocks]
        nnz_per = [(r1 - r0) * d for r0, r1 in blocks]

        def step(j):
            r0, r1 = blocks[j % len(blocks)]
            O.np_apply_dense(mats[j % len(blocks)], a[r0:r1])
            return nnz_per[j % len(blocks)]
        sample = (f"whole apply of config 1" if len(blocks) == 1 else
                  f"each step one {blk}-row block of the full {n}-row matrix with the full operator's "
                  f"columns (same m x d output), cycling over the {len(blocks)} blocks")
    else:
        import scipy.sparse as sp

        ip, ix, vv = gen_csr_shard(torch, cfg, 0, n, gen_dev)
        a = sp.csr_array((vv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=(n, d))
        del ip, ix, vv

        def step(j):
            O.np_apply_csr(h, s, m, a)
            return a.nnz
        sample = "whole apply (the full matrix every step)"
    prep_s = time.perf_counter() - t_prep
    for j in range(args.warmup):
        step(j)
    t0 = time.perf_counter()
    nnz = 0
    for j in range(args.steps):
        nnz += step(args.warmup + j)
    dt = time.perf_counter() - t0
    value = nnz / dt
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (the same seeded matrix as our arm)",
        "config": {"workload": cfg["workload"], "n": n, "d": d, "m": m, "input_dtype": cfg["dtype"]},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": 1, "kind": "port",
                         "sample": sample + "; reference primitives (sketch.py:153-165, _validation.py:16-27), "
                                   "single-threaded like the reference", "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "prep_s": round(prep_s, 1),
    }
    return line


def cpu_baseline_sample(cfg_name, cfg, a_dev_sample, torch):
    """Oracle port (reference primitives) timed on this host over a bounded
    sample (~10-30 s of CPU work)."""
    import numpy as np

    from oracle import oracle as O

    a = a_dev_sample.cpu().numpy()
    rows = a.shape[0]
    h, s = O.hash_signs(rows, cfg["m"], cfg["seed"])
    mat = O.np_sketch_matrix(h, s, cfg["m"], rows)
    best = float("inf")
    t_end = time.perf_counter() + 12.0
    reps = 0
    while reps < 2 or (time.perf_counter() < t_end and reps < 20):
        t0 = time.perf_counter()
        O.np_apply_dense(mat, a)
        best = min(best, time.perf_counter() - t0)
        reps += 1
    return {"value": a.size / best, "unit": "nnz/s", "cores": 1, "kind": "port",
            "sample": f"rows [0, {rows}) of the workload x {cfg['d']} cols, best of {reps} "
                      "(scipy CSR @ dense after fp64 upcast, the reference's sketch.py:165 path)"}


def cpu_baseline_csr(cfg, ip, ix, vv):
    """Oracle port of sketch.py:155-164 (repeat + bincount) on the whole CSR
    matrix of the workload, best of up to 5 within ~12 s, one core."""
    import numpy as np
    import scipy.sparse as sp

    from oracle import oracle as O

    n, d, m = cfg["n"], cfg["d"], cfg["m"]
    a = sp.csr_array((vv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=(n, d))
    h, s = O.hash_signs(n, m, cfg["seed"])
    best, reps, t_end = float("inf"), 0, time.perf_counter() + 12.0
    while reps < 1 or (time.perf_counter() < t_end and reps < 5):
        t0 = time.perf_counter()
        O.np_apply_csr(h, s, m, a)
        best = min(best, time.perf_counter() - t0)
        reps += 1
    return {"value": a.nnz / best, "unit": "nnz/s", "cores": 1, "kind": "port",
            "sample": f"the whole matrix ({a.nnz} nnz), best of {reps} (repeat + bincount, "
                      "the reference's sketch.py:155-164 path)"}


def lowrank_report(args, cfg):
    """Config 5's second half: low_rank_approx(k=10) with the m=400 row sketch
    (s_op) and a sparse-embedding column sketch (r_op, t_r from
    sketch_dims_lowrank(10, 0.5)) on the GPU, host SVDs of the sketches, and the
    Frobenius error ratio err / Delta_10.  Delta_10 comes from randomized
    subspace iteration on the GPU -- a SUBSTITUTE oracle: the reference's
    best_rank_k_error densifies A (550 GB here)."""
    import scipy.sparse as sp
    import torch

    from paper_1207_6365_b200 import SparseEmbedding
    from paper_1207_6365_b200.lowrank import best_rank_k_error_gpu, low_rank_approx, sketch_dims_lowrank

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, d = cfg["n"], cfg["d"]
    ip, ix, vv = gen_csr_shard(torch, cfg, 0, n, dev)
    a = sp.csr_array((vv.double().cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=(n, d))
    k, eps = cfg["lowrank"], 0.5
    t_r = sketch_dims_lowrank(k, eps)[0]
    t0 = time.perf_counter()
    r_op = SparseEmbedding(d, t_r, 2, device=dev)
    s_op = SparseEmbedding(n, cfg["m"], cfg["seed"], device=dev)
    res = low_rank_approx(a, k, eps, seed=3, r_op=r_op, s_op=s_op)
    t1 = time.perf_counter()
    delta = best_rank_k_error_gpu(a, k)
    t2 = time.perf_counter()
    return {
        "metric": "config5 low-rank: Frobenius error ratio err / Delta_10 (lower is better)",
        "value": res.err / delta, "unit": "ratio", "higher_is_better": False,
        "err": res.err, "delta_10": delta, "delta_source": "randomized subspace iteration on GPU (substitute)",
        "t_r": t_r, "t_s": res.t_s, "cond_su": res.cond_su, "low_rank_approx_s": round(t1 - t0, 3),
        "delta_s": round(t2 - t1, 3), "config": {"workload": cfg["workload"], "k": k, "eps": eps},
    }


def our_arm(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1207_6365_b200 import SparseEmbedding, launch_count

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or (args.fused and "RANK" in os.environ):
        # communicator lines on stderr (NCCL_DEBUG=INFO) so a scaling run shows
        # every rank's device, transport (NVLink / NVLS) and ring layout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH")
        dist.init_process_group("nccl", device_id=dev)
    n, d, m = cfg["n"], cfg["d"], cfg["m"]
    # config 5 at N > 1: bucket ownership -- every rank holds the
    # whole input and computes only its SA rows [b0, b1); no collective
    bucket_mode = world > 1 and cfg.get("shard") == "bucket" and args.kernel == "sa"
    r0, r1 = (0, n) if bucket_mode else (rank * n // world, (rank + 1) * n // world)
    b0, b1 = (rank * m // world, (rank + 1) * m // world) if bucket_mode else (0, m)
    sa_dt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    fast = bool(args.fast)  # unordered atomics (not bit-exact); default: the deterministic kernels

    # ---- inputs resident in HBM
    if cfg["kind"] == "dense":
        A = gen_dense_shard(torch, cfg, r0, r1, dev)
        nnz_local = A.numel()
        in_bytes = A.numel() * A.element_size()
    else:
        ip, ix, vv = gen_csr_shard(torch, cfg, r0, r1, dev)
        if args.kernel == "lev" and args.lev_f64:
            vv = vv.double()  # as_csr's upcast: the dtype the reference API hands K5 (_validation.py:30-41)
        nnz_local = vv.numel()
        in_bytes = vv.numel() * (vv.element_size() + 4) + ip.numel() * ip.element_size()
    torch.cuda.synchronize()

    # ---- operator build (K1 + K2), timed separately (mirrors __init__)
    tb0, tb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tb0.record()
    op = SparseEmbedding(n, m, cfg["seed"], device=dev, row_range=(r0, r1))
    tb1.record()
    torch.cuda.synchronize()
    build_ms = tb0.elapsed_time(tb1)
    if bucket_mode:  # this rank's work: the rows hashed into its buckets
        gptr, grows, _ = op.grouped_plan(0)
        p0, p1 = int(gptr[b0]), int(gptr[b1])
        mine = (grows[p0:p1] & 0x7FFFFFFF).long()
        lens = (ip[1:] - ip[:-1]).long()
        nnz_local = int(lens[mine].sum())
        in_bytes = nnz_local * (vv.element_size() + 4) + (p1 - p0) * 2 * ip.element_size()

    SA = torch.empty((m, d), dtype=sa_dt, device=dev)
    stream = torch.cuda.current_stream(dev)
    fin_flags = torch.zeros((args.steps + args.warmup + 2) * max(1, args.chunks), dtype=torch.int32, device=dev)
    fin_i = [0]

    lev = None
    if args.kernel == "lev":
        # K5: leverage contraction rows = A @ (R^-1 G), squared row norms (config 4 pipeline)
        from paper_1207_6365_b200.solvers import basis_change, gaussian_jl_entries

        sa64 = op._apply_csr_device(ip, ix, vv, d, torch.float64, canonical=True).cpu().numpy()
        n_mat, qr_rank = basis_change(sa64)
        probe = torch.from_numpy(n_mat @ gaussian_jl_entries(32, qr_rank, 7).T).to(dev)
        scores = torch.empty(nnz_local and (r1 - r0), dtype=torch.float64, device=dev)
        lev = (probe, scores)

    def apply_once():
        if lev is not None:
            from paper_1207_6365_b200 import _lib
            from paper_1207_6365_b200.sketch import _ITYPE, _TORCH_TO_SKT, _ptr, _stream_ptr

            _lib.check(_lib.lib().skt_lev_rownorms_csr(
                r1 - r0, d, _ptr(ip), _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype], _ptr(vv),
                _TORCH_TO_SKT[vv.dtype], _ptr(lev[0]), lev[0].shape[1], _ptr(lev[1]), _lib.SKT_F64,
                _stream_ptr(dev)))
        elif cfg["kind"] == "dense":
            # the API's work: the fused finiteness scan included (as_dense,
            # _validation.py:25-26); the flag is read once after the timed loop
            fin_i[0] += 1
            op._apply_dense_device(A, sa_dt, out=SA, flag=fin_flags[fin_i[0] % fin_flags.numel()])
        else:
            op._apply_csr_device(ip, ix, vv, d, sa_dt, canonical=True, out=SA,
                                 deterministic=not fast,
                                 buckets=(b0, b1) if bucket_mode else None)

    # N > 1, dense: pipelined exchange -- SA is computed in contiguous bucket
    # ranges and each range is all-reduced (async, NCCL stream) while the next
    # range is computed (distributed.ShardedSparseEmbedding.apply(chunks=K)).
    fused = None
    if args.fused and cfg["kind"] == "dense" and lev is None and dist.is_initialized():
        from paper_1207_6365_b200.distributed import FusedShardedSparseEmbedding

        fused = FusedShardedSparseEmbedding(n, m, cfg["seed"], device=dev)
    pipelined = world > 1 and cfg["kind"] == "dense" and lev is None and args.chunks > 1 and fused is None
    ranges = [(k * m // args.chunks, (k + 1) * m // args.chunks) for k in range(args.chunks)]

    def step(kev=None):
        if kev is not None:
            kev[0].record(stream)
        if fused is not None:
            fused.apply(A, sa_dt)
            if kev is not None:
                kev[1].record(stream)
            return
        if pipelined:
            works = []
            for c0, c1 in ranges:
                fin_i[0] += 1
                op._apply_dense_device(A, sa_dt, out=SA, buckets=(c0, c1),
                                       flag=fin_flags[fin_i[0] % fin_flags.numel()])
                works.append(dist.all_reduce(SA[c0:c1], async_op=True))
            if kev is not None:
                kev[1].record(stream)
            for w in works:
                w.wait()
            return
        apply_once()
        if kev is not None:
            kev[1].record(stream)
        if world > 1 and lev is None and not bucket_mode:
            dist.all_reduce(SA)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # inputs that fit in L2 (configs 1, 2): L2 is flushed before every step by
    # writing a 512 MB buffer, and the steps are timed individually (events
    # around each step only) so the flush is not counted
    flush_l2 = in_bytes < L2_FLUSH_BELOW
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush_l2 else None

    def timed_region():
        kevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        sevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        lc0 = launch_count()
        with ClockSampler(local) as clk:
            e0.record(stream)
            for i in range(args.steps):
                if flush_l2:
                    flush_buf.fill_(i & 0xFF)
                    sevs[i][0].record(stream)
                step(kevs[i])
                if flush_l2:
                    sevs[i][1].record(stream)
            e1.record(stream)
            torch.cuda.synchronize()
        launches = launch_count() - lc0
        if world > 1:
            dist.barrier()
        total_ms = sum(a.elapsed_time(b) for a, b in sevs) if flush_l2 else e0.elapsed_time(e1)
        kern_ms = sum(a.elapsed_time(b) for a, b in kevs) / args.steps
        return total_ms, kern_ms, launches, clk

    total_ms, kern_ms, launches, clk = timed_region()
    if int(fin_flags.max()) != 0:
        raise ValueError("matrix contains non-finite entries")
    remeasured = False
    if clk.rejected():
        log("clock check failed", clk.summary(), "- re-measuring once")
        total_ms, kern_ms, launches, clk = timed_region()
        remeasured = True

    # max over ranks
    t = torch.tensor([total_ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_ms_max = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    nnz_total = (n * d) if cfg["kind"] == "dense" else None
    if nnz_total is None:
        tt = torch.tensor([nnz_local], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt)
        nnz_total = int(tt.item())
    value = nnz_total / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel (this rank's apply launch)
    alg_bytes = in_bytes + ((b1 - b0) * d * SA.element_size() if lev is None else (r1 - r0) * 8)
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    peak, peak_src = peak_hbm()
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic_for(args.config if lev is None else args.config + "_lev"),
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs copy bandwidth)",
                "kernel_ms": round(kern_ms, 4), "alg_bytes_per_launch": alg_bytes,
                "frac_of_8TBps_nominal": round(achieved / 8000.0, 4),
                "kernel": dominant_kernel(cfg, lev is not None, args, sa_dt)}
    gc = gather_ceiling_ms(args.config) if (cfg["kind"] == "csr" and lev is None and world == 1) else None
    if gc is not None:
        # CSR S.A reads every row's (indptr pair, index segment, value segment)
        # in bucket order = random rows, which B200 serves at a request rate
        # well below streaming HBM: the kernel's ceiling is that access pattern
        roofline["gather_ceiling"] = {
            "ms": gc, "frac": round(gc / kern_ms, 4),
            "source": "the bucket-ordered access pattern with 32-bit loads and without arithmetic, L2 flushed "
                      "(tools/gather_bench.cu, profiles/r01_gather_ceiling.json); csr_quad's 128-bit loads "
                      "pass it (frac > 1)"}

    # ---- end to end through the public API, host buffers
    e2e, e2e_numpy = None, None
    if not args.no_e2e and cfg["kind"] == "dense" and lev is None:
        host = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
        host.copy_(A)
        torch.cuda.synchronize()
        e_steps = max(1, min(args.steps, args.e2e_steps))
        for _ in range(2):  # warm-up: device block and two page-locked result blocks cached
            res = op.apply(host, out_dtype=sa_dt)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            res = op.apply(host, out_dtype=sa_dt)  # H2D + kernel + finiteness check + D2H
            if world > 1:
                rt = res.to(dev)
                dist.all_reduce(rt)
                res = rt.cpu()
        e2e_s = torch.tensor([(time.perf_counter() - t0) / e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": nnz_total / float(e2e_s), "unit": "nnz/s",
               "h2d_bytes_per_step": host.numel() * host.element_size(),
               "d2h_bytes_per_step": res.numel() * res.element_size(),
               "steps": e_steps, "ms_per_step": 1e3 * float(e2e_s),
               "api": "SparseEmbedding.apply(pinned host tensor)"}
        if world == 1:
            # the reference's calling convention: a pageable numpy ndarray in,
            # a new fp64 numpy SA out (sketch.py:153-165)
            arr = np.array(host.numpy())  # a pageable copy (host is page-locked)
            del host
            op.apply(arr)
            t0 = time.perf_counter()
            for _ in range(e_steps):
                res = op.apply(arr)
            dt = (time.perf_counter() - t0) / e_steps
            e2e_numpy = {"value": nnz_total / dt, "unit": "nnz/s", "h2d_bytes_per_step": arr.nbytes,
                         "d2h_bytes_per_step": res.nbytes, "steps": e_steps, "ms_per_step": 1e3 * dt,
                         "api": "SparseEmbedding.apply(numpy ndarray, pageable) -> numpy fp64"}
            del arr
        else:
            del host
    elif not args.no_e2e and cfg["kind"] == "csr" and lev is None and world == 1:
        # scipy CSR in (the reference's convention; canonical, as as_csr leaves
        # it), numpy fp64 SA out; every step copies indptr / indices / data
        import scipy.sparse as sp

        a_sp = sp.csr_array((vv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=(n, d))
        det = not fast
        e_steps = max(1, min(args.steps, args.e2e_steps))
        res = op.apply(a_sp, deterministic=det)
        t0 = time.perf_counter()
        for _ in range(e_steps):
            res = op.apply(a_sp, deterministic=det)
        dt = (time.perf_counter() - t0) / e_steps
        e2e = {"value": nnz_total / dt, "unit": "nnz/s",
               "h2d_bytes_per_step": a_sp.data.nbytes + a_sp.indices.nbytes + a_sp.indptr.nbytes,
               "d2h_bytes_per_step": res.nbytes, "steps": e_steps, "ms_per_step": 1e3 * dt,
               "api": "SparseEmbedding.apply(scipy.sparse.csr_array, pageable) -> numpy fp64"}
        del a_sp

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and lev is None:
        if cfg["kind"] == "dense":
            rows = min(r1 - r0, 1 << 21)
            cpu = cpu_baseline_sample(args.config, cfg, A[:rows], torch)
        else:
            cpu = cpu_baseline_csr(cfg, ip, ix, vv)

    line = {
        "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded torch generator, BASELINE shapes/distributions)",
        "config": {"workload": cfg["workload"], "n": n, "d": d, "m": m, "input_dtype": cfg["dtype"],
                   "sa_dtype": "f32" if sa_dt == torch.float32 else "f64",
                   "accumulate": "fp64, ascending row order (bit-identical to the reference)",
                   "l2": ("L2 flushed before every step (512 MB write, outside the per-step events)" if flush_l2
                          else "inputs larger than L2 (no flush needed)"),
                   "parallelism": (f"bucket-ownership x{world}: rank owns SA rows [{b0}, {b1}), whole input on "
                                   "every rank, no collective") if bucket_mode else
                                  (f"row-shard x{world} + exchange fused into K3 (push to owner slots over "
                                   "symmetric memory, slot sums, all-gather)") if fused is not None else
                                  f"row-shard x{world}" + (
                       (f" + NCCL all-reduce of m x d partials, pipelined over {args.chunks} bucket ranges"
                        if pipelined else " + NCCL all-reduce of m x d partials") if world > 1 else "")},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_numpy": e2e_numpy, "gpu_launches": launches,
        "clocks": clk.summary(), "remeasured": remeasured,
        "build_ms": round(build_ms, 3), "kernel_ms_max_over_ranks": round(kern_ms_max, 4),
    }
    if dist.is_initialized():
        dist.destroy_process_group()
    return line if rank == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--kernel", default="sa", choices=["sa", "lev", "lowrank"],
                    help="sa: the S.A hot path (headline); lev: K5 leverage contraction (config c4); "
                         "lowrank: config 5 low-rank error ratio")
    ap.add_argument("--lev-f64", action="store_true",
                    help="--kernel lev: fp64 CSR values (the reference API's dtype) -> the fp64 tensor-core kernel")
    ap.add_argument("--fast", action="store_true",
                    help="CSR: unordered-atomics fast mode (equal to the reference up to rounding, not bit-exact)")
    ap.add_argument("--exact", action="store_true", help="accepted for compatibility (exact is the default)")
    ap.add_argument("--fused", action="store_true",
                    help="dense, under torchrun: exchange fused into K3 (partial rows pushed to owner ranks over "
                         "NVLink symmetric memory, owner slot sums, all-gather) instead of the NCCL all-reduce")
    ap.add_argument("--chunks", type=int, default=4,
                    help="N > 1: bucket ranges whose all-reduce overlaps the next range's compute")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # W >= 3 warm-up steps
    cfg = CONFIGS[args.config]
    # stdout carries exactly ONE JSON line: anything native libraries print to
    # fd 1 during the run (NCCL prints its version / INFO lines there when
    # NCCL_DEBUG is set in the environment) goes to stderr instead
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    if args.kernel == "lowrank":
        line = lowrank_report(args, cfg)
    else:
        line = reference_arm(args, cfg) if args.impl == "reference" else our_arm(args, cfg)
    sys.stdout.flush()
    if line is not None:
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    os.close(json_fd)


if __name__ == "__main__":
    main()
