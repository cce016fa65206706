"""Config 4 kernel time with an L2 set-aside for persisting (evict_last) lines:
cudaLimitPersistingL2CacheSize = 0 / 32 MB / 64 MB."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1207_6365_b200 import SparseEmbedding
rt = ctypes.CDLL("libcudart.so.12")
cfg = bench.CONFIGS["c4"]
dev = torch.device("cuda:0")
ip, ix, vv = bench.gen_csr_shard(torch, cfg, 0, cfg["n"], dev)
op = SparseEmbedding(cfg["n"], cfg["m"], cfg["seed"], device=dev)
out = op._apply_csr_device(ip, ix, vv, cfg["d"], torch.float32, True)
mx = ctypes.c_int()
rt.cudaDeviceGetAttribute(ctypes.byref(mx), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
print("max persisting L2 bytes", mx.value, flush=True)
for mb in (None, 32, 64, 0):
    if mb is not None:
        print("set", mb, "MB ->", rt.cudaDeviceSetLimit(6, ctypes.c_size_t(min(mb << 20, mx.value))))
    v = ctypes.c_size_t()
    rt.cudaDeviceGetLimit(ctypes.byref(v), 6)
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); op._apply_csr_device(ip, ix, vv, cfg["d"], torch.float32, True, out=out); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    print("persisting L2", v.value >> 20, "MB: median %.4f ms min %.4f" % (ts[len(ts) // 2], ts[0]), flush=True)
