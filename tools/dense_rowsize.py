"""K3 at different row sizes: TMA gather4 vs the register gather (A/B through
SKT_DENSE_G4 in child processes).  ~8.6 GB of input per shape, median of 10.
    python tools/dense_rowsize.py"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, torch
sys.path.insert(0, %r)
from paper_1207_6365_b200 import SparseEmbedding
d, dt = int(sys.argv[1]), getattr(torch, sys.argv[2])
esz = torch.tensor([], dtype=dt).element_size()
n = (8 << 30) // (d * esz)
a = torch.randn(n, d, device="cuda").to(dt)
op = SparseEmbedding(n, max(1, n // 256), 1, device=torch.device("cuda:0"))
for _ in range(3):
    op._apply_dense_device(a, torch.float32, check_finite=False)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); op._apply_dense_device(a, torch.float32, check_finite=False); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[5]
print(f"d={d} {sys.argv[2]} row={d*esz} B: {ms:.3f} ms {a.numel()*esz/ms/1e6:.0f} GB/s")
""" % ROOT

for d, dt in [(32, "float32"), (64, "float32"), (128, "float32"), (256, "float32"), (384, "float32"),
              (512, "float32"), (32, "float64"), (64, "float64"), (128, "float64"), (256, "float64")]:
    for g4 in ("1", "0"):
        env = dict(os.environ, SKT_DENSE_G4=g4)
        out = subprocess.run([sys.executable, "-c", CHILD, str(d), dt], env=env, capture_output=True, text=True)
        print(f"g4={g4}", (out.stdout or out.stderr).strip().splitlines()[-1], flush=True)
