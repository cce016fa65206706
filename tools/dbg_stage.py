import sys, numpy as np, scipy.sparse as sp, torch
sys.path.insert(0, ".")
from bench import CONFIGS, gen_csr_shard
from paper_1207_6365_b200 import SparseEmbedding
from paper_1207_6365_b200.sketch import _to_device, csr_is_canonical_device
from oracle import oracle as O
c = CONFIGS["c4"]; dev = torch.device("cuda", 0)
ip, ix, vv = gen_csr_shard(torch, c, 0, c["n"], dev)
a = sp.csr_array((vv.cpu().numpy(), ix.cpu().numpy(), ip.cpu().numpy()), shape=(c["n"], c["d"]))
a_s = a[slice(0, 400_000)]
print("dtypes", a_s.indptr.dtype, a_s.indices.dtype, a_s.data.dtype, a_s.indptr[0], a_s.nnz)
for rep in range(3):
    for name, x in (("indptr", a_s.indptr), ("indices", a_s.indices), ("data", a_s.data)):
        t = _to_device(x, dev)
        torch.cuda.synchronize()
        ok = np.array_equal(t.cpu().numpy(), x)
        if not ok:
            bad = np.nonzero(t.cpu().numpy() != x)[0]
            print(rep, name, "MISMATCH", len(bad), bad[:5], bad[-5:], x.nbytes)
        else:
            print(rep, name, "ok", x.nbytes)
op_s = SparseEmbedding(400_000, c["m"], c["seed"], device=dev)
h_s, s_s = O.hash_signs(400_000, c["m"], c["seed"])
ref = O.np_apply_csr(h_s, s_s, c["m"], a_s)
ipd, ixd, vvd = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (a_s.indptr, a_s.indices, a_s.data))
print("canon", csr_is_canonical_device(ipd, ixd, 400_000), a_s.has_canonical_format)
got = op_s._apply_csr_device(ipd, ixd, vvd, 64, torch.float64, True).cpu().numpy()
print("device path equal", np.array_equal(got, ref))
got2 = op_s.apply(a_s)
print("apply equal", np.array_equal(got2, ref))
