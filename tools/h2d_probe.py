import torch, time
n = 8_589_934_592 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for chunks in (1, 8, 32):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        step = n // chunks
        for i in range(chunks):
            d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"chunks={chunks}: {dt*1e3:.1f} ms  {n*4/dt/1e9:.1f} GB/s")
# two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
half = n // 2
with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"2 streams: {dt*1e3:.1f} ms {n*4/dt/1e9:.1f} GB/s")
