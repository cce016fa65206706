"""Where does the end-to-end time of SparseEmbedding.apply(pinned host tensor) go?
(config 3 shape; run on the GPU box)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1207_6365_b200 import SparseEmbedding
n, d, m = 16_777_216, 128, 65_536
op = SparseEmbedding(n, m, 3, device=torch.device("cuda", 0))
h = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
h.normal_()
torch.cuda.synchronize()
res = op.apply(h, out_dtype=torch.float32)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = op.apply(h, out_dtype=torch.float32)
    t1 = time.perf_counter()
    print(f"apply(host) total {1e3*(t1-t0):.1f} ms")
# phases
torch.cuda.synchronize(); t0 = time.perf_counter()
da = h.to("cuda", non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
out = op._apply_dense_device(da, torch.float32, True); torch.cuda.synchronize(); t2 = time.perf_counter()
r = out.cpu(); t3 = time.perf_counter()
print(f"h2d {1e3*(t1-t0):.1f} ms, kernel+check {1e3*(t2-t1):.1f} ms, d2h {1e3*(t3-t2):.1f} ms")
del da
torch.cuda.synchronize(); t0 = time.perf_counter()
da = torch.empty((n, d), dtype=torch.float32, device="cuda"); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"alloc {1e3*(t1-t0):.2f} ms")
