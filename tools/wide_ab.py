"""A/B of the wide-CSR paths (SKT_CSR_WIDE = unset: fine blocks | partition |
colblock) on config 5: small oracle cases, sha256 of the full-size SA, timing."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1207_6365_b200 import SparseEmbedding
from tests.test_gpu_wide import _check, _random_csr
mode = os.environ.get("SKT_CSR_WIDE", "fine")
for n, d, t, per, dt in [(3000, 70001, 37, 60, np.float32), (5000, 30000, 2, 20, np.float32),
                         (2000, 40000, 5, 300, np.float64), (20000, 262144, 7, 262, np.float32)]:
    rng = np.random.default_rng(n + d)
    a = _random_csr(rng, n, d, per, dt)
    _check(SparseEmbedding(n, t, 3), a, t, 3, d)
print("small cases ok, wide path", mode, flush=True)
cfg = bench.CONFIGS["c5"]
dev = torch.device("cuda:0")
ip, ix, vv = bench.gen_csr_shard(torch, cfg, 0, cfg["n"], dev)
op = SparseEmbedding(cfg["n"], cfg["m"], cfg["seed"], device=dev)
out = op._apply_csr_device(ip, ix, vv, cfg["d"], torch.float32, True)
torch.cuda.synchronize()
print("sha", hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16], flush=True)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); op._apply_csr_device(ip, ix, vv, cfg["d"], torch.float32, True, out=out); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts.sort(); print("c5 exact (%s): median %.4f ms min %.4f ms" % (mode, ts[len(ts) // 2], ts[0]), flush=True)
