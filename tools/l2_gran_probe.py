"""Config 4 kernel time under cudaLimitMaxL2FetchGranularity = 32 / 64 / 128."""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for gran in (0, 32, 64, 128):
    if gran:
        print("set", gran, rt.cudaDeviceSetLimit(5, ctypes.c_size_t(gran)))
    v = ctypes.c_size_t()
    rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
    ts = []
    for _ in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); op._apply_csr_device(ip, ix, vv, cfg["d"], torch.float32, True, out=out); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    print("granularity", v.value, "median %.4f ms min %.4f" % (ts[len(ts) // 2], ts[0]), flush=True)
