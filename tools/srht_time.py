"""Time skt_srht_apply on config 4's t1 x d sketch (363,409 x 64 fp64 -> 20,000 rows)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1207_6365_b200.solvers import srht_apply
from oracle import oracle as O
a = torch.randn(363_409, 64, dtype=torch.float64, device="cuda")
for _ in range(3): srht_apply(a, 20_000, 1)
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): srht_apply(a, 20_000, 1)
e1.record(); torch.cuda.synchronize()
gpu_ms = e0.elapsed_time(e1) / 10
ah = a.cpu().numpy(); t0 = time.perf_counter(); O.srht_apply(ah, 20_000, 1); cpu_ms = 1e3 * (time.perf_counter() - t0)
print(f"srht 363409x64 -> 20000: GPU {gpu_ms:.3f} ms per call (incl. host RNG for sign/rows + H2D of them), "
      f"reference-path numpy {cpu_ms:.1f} ms")
