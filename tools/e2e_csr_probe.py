"""Where the time of SparseEmbedding.apply(scipy CSR) goes (config 4)."""
import sys
import time

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, ".")
from bench import CONFIGS, gen_csr_shard  # noqa: E402
from paper_1207_6365_b200 import SparseEmbedding  # noqa: E402
from paper_1207_6365_b200.sketch import _host, csr_is_canonical_device  # noqa: E402

dev = torch.device("cuda", 0)
c = CONFIGS["c4"]
ip, ix, vv = gen_csr_shard(torch, c, 0, c["n"], dev)
a = sp.csr_array((vv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=(c["n"], c["d"]))
op = SparseEmbedding(c["n"], c["m"], 1, device=dev)
op.apply(a)


def t(label, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label:40s} {1e3 * min(ts):8.2f} ms", flush=True)
    return r


t("apply(scipy CSR) total", lambda: op.apply(a))
t("H2D indptr (pageable)", lambda: torch.from_numpy(a.indptr).to(dev))
t("H2D indices (pageable)", lambda: torch.from_numpy(a.indices).to(dev))
t("H2D data (pageable)", lambda: torch.from_numpy(a.data).to(dev))
pin = [torch.from_numpy(x).pin_memory() for x in (a.indptr, a.indices, a.data)]
from paper_1207_6365_b200.sketch import _to_device  # noqa: E402
t("H2D 3 arrays (staged ring)", lambda: [_to_device(x, dev) for x in (a.indptr, a.indices, a.data)])
t("H2D 3 arrays (pinned)", lambda: [p.to(dev, non_blocking=True) for p in pin])
t("device canonical check", lambda: csr_is_canonical_device(ip, ix, c["n"]))
res = t("kernel (fp64 out)", lambda: op._apply_csr_device(ip, ix, vv, c["d"], torch.float64, True))
t("D2H SA fp64 (_host)", lambda: _host(res))
t("D2H SA fp64 .cpu()", lambda: res.cpu())
