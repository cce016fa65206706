"""K5 on fp64 CSR (the reference API's dtype: as_csr converts to fp64), config
4's shape, CUDA-core fp64 path: median of 10 launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1207_6365_b200 import _lib  # noqa: E402
from paper_1207_6365_b200.sketch import _ITYPE, _TORCH_TO_SKT, _ptr, _stream_ptr  # noqa: E402

cfg = bench.CONFIGS["c4"]
dev = torch.device("cuda:0")
ip, ix, vv = bench.gen_csr_shard(torch, cfg, 0, cfg["n"], dev)
vv = vv.double()
probe = torch.randn(cfg["d"], 32, dtype=torch.float64, device=dev)
scores = torch.empty(cfg["n"], dtype=torch.float64, device=dev)
L = _lib.lib()


def run():
    _lib.check(L.skt_lev_rownorms_csr(cfg["n"], cfg["d"], _ptr(ip), _ITYPE[ip.dtype], _ptr(ix), _ITYPE[ix.dtype],
                                      _ptr(vv), _TORCH_TO_SKT[vv.dtype], _ptr(probe), 32, _ptr(scores), _lib.SKT_F64,
                                      _stream_ptr(dev)))


for _ in range(3):
    run()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
ref = ((torch.sparse_csr_tensor(ip.long(), ix.long(), vv, size=(cfg["n"], cfg["d"])) @ probe) ** 2).sum(1)
print(f"fp64 K5 config-4 shape: {ts[5]:.3f} ms, max rel err vs torch {float(((scores - ref).abs() / ref.clamp_min(1e-300)).max()):.2e}")
