"""Does L2 residency speed up the bucket-ordered CSR kernel (csr_tile)?
Config-4-shaped CSR at 1/8, 1/4, 1/2 and full size; each S.A timed with the
inputs L2-warm (no flush) and after a 512 MB L2 flush."""
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS, gen_csr_shard  # noqa: E402
from paper_1207_6365_b200 import SparseEmbedding  # noqa: E402

dev = torch.device("cuda", 0)
c = dict(CONFIGS["c4"])
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for frac in (8, 4, 2, 1):
    n = c["n"] // frac
    cc = dict(c, n=n)
    ip, ix, vv = gen_csr_shard(torch, cc, 0, n, dev)
    op = SparseEmbedding(n, c["m"] // frac, 1, device=dev)
    out = torch.empty((c["m"] // frac, c["d"]), dtype=torch.float32, device=dev)
    mb = (vv.numel() * 8 + ip.numel() * 4) / 1e6
    for mode in ("warm", "flushed"):
        ts = []
        for i in range(12):
            if mode == "flushed":
                flush.fill_(i & 0xFF)
            else:
                op._apply_csr_device(ip, ix, vv, c["d"], torch.float32, canonical=True, out=out)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op._apply_csr_device(ip, ix, vv, c["d"], torch.float32, canonical=True, out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts[2:])[len(ts[2:]) // 2]
        print(f"n={n:8d} A={mb:7.1f} MB {mode:8s}: {ms:.4f} ms  ({ms * frac:.4f} ms scaled to full size)", flush=True)
