"""Read-bandwidth ceiling probes (tools only): plain LDG.128 streaming with U
loads in flight, and 1D bulk-copy (cp.async.bulk, TMA) streaming into a smem
ring.  8 GiB fp32 buffer (>> L2).  Prints JSON."""
import ctypes, json, os, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmembench.so"))
n = 1 << 31  # floats = 8 GiB
A = torch.empty(n, device="cuda", dtype=torch.float32).normal_()
out = torch.zeros(1, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
res = {}
for u in (4, 8, 16):
    for blocks in (148 * 4, 148 * 8, 148 * 16):
        ms = t(lambda: L.mb_read(ctypes.c_void_p(A.data_ptr()), ctypes.c_int64(n // 4), u, blocks, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
        res[f"ldg_u{u}_b{blocks}"] = round(n * 4 / ms / 1e6, 1)
for chunk_kb in (128, 32):
    for u in (4, 8):
        cf4 = chunk_kb * 1024 // 16
        ms = t(lambda: L.mb_stream(ctypes.c_void_p(A.data_ptr()), ctypes.c_int64(n // 4), ctypes.c_int64(cf4), u, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
        res[f"stream_{chunk_kb}k_u{u}"] = round(n * 4 / ms / 1e6, 1)
for blocks in (148, 148 * 2, 148 * 3):
    ms = t(lambda: L.mb_bulk(ctypes.c_void_p(A.data_ptr()), ctypes.c_int64(n * 4), blocks, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
    res[f"bulk_b{blocks}"] = round(n * 4 / ms / 1e6, 1)
print(json.dumps(res))
