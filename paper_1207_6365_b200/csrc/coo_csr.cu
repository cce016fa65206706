// coo_csr.cu -- device canonicalisation of a COO matrix into CSR, the second
// half of Matrix Market ingest (reference io.py:101-102: coo_array -> as_csr,
// _validation.py:30-41: duplicates summed, explicit zeros dropped, rows with
// sorted column indices).  Entries are ordered by (row, col) with two stable
// passes of the plan builder K2 (by column, then by row: ties keep file
// order), duplicate runs are summed in file order, entries whose sum is 0 are
// dropped, and indptr comes from an integer row histogram + the device scan;
// a non-finite kept sum raises the caller's flag (as_csr's finiteness check).
// Deterministic (integer atomics only).
#include "common.cuh"
#include "scan.cuh"

namespace skt {
namespace {

__global__ void coo_keys_kernel(const int64_t *__restrict__ key, const uint32_t *__restrict__ perm, int64_t count,
                                uint32_t *__restrict__ out, int8_t *__restrict__ zero) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    out[e] = (uint32_t)key[perm ? (int64_t)perm[e] : e];
    if (zero) zero[e] = 0;
  }
}

__global__ void coo_order_kernel(const uint32_t *__restrict__ p1, const uint32_t *__restrict__ p2, int64_t count,
                                 const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                                 uint32_t *__restrict__ ord, uint32_t *__restrict__ rs, uint32_t *__restrict__ cs) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = p1[p2[e] & 0x7fffffffu] & 0x7fffffffu;
    ord[e] = o;
    rs[e] = (uint32_t)rows[o];
    cs[e] = (uint32_t)cols[o];
  }
}

// run heads: sum the run in file order; keep = head && sum != 0
__global__ void coo_runs_kernel(const uint32_t *__restrict__ ord, const uint32_t *__restrict__ rs,
                                const uint32_t *__restrict__ cs, const double *__restrict__ vals, int64_t count,
                                double *__restrict__ sums, uint32_t *__restrict__ keep,
                                uint32_t *__restrict__ rowcnt, int32_t *__restrict__ nonfinite) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const bool head = e == 0 || rs[e] != rs[e - 1] || cs[e] != cs[e - 1];
    uint32_t k = 0;
    if (head) {
      double s = vals[ord[e]];
      for (int64_t f = e + 1; f < count && rs[f] == rs[e] && cs[f] == cs[e]; ++f) s += vals[ord[f]];
      sums[e] = s;
      k = s != 0.0;  // NaN and inf sums are kept, as eliminate_zeros keeps them
      if (k) atomicAdd(rowcnt + rs[e], 1u);
      // as_csr's finiteness check on the canonical data (_validation.py:39-40)
      if (nonfinite && !isfinite(s)) atomicOr(nonfinite, 1);
    }
    keep[e] = k;
  }
}

__global__ void coo_emit_kernel(const uint32_t *__restrict__ keep_scan, const uint32_t *__restrict__ cs,
                                const double *__restrict__ sums, const uint32_t *__restrict__ keep_flag, int64_t count,
                                int32_t *__restrict__ indices, double *__restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    if (keep_flag[e]) {
      const uint32_t p = keep_scan[e];
      indices[p] = (int32_t)cs[e];
      out[p] = sums[e];
    }
  }
}

__global__ void coo_indptr_kernel(const uint32_t *__restrict__ scan, int64_t n1, int64_t *__restrict__ indptr,
                                  const uint32_t *__restrict__ total, int64_t *__restrict__ nnz) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n1; e += (int64_t)gridDim.x * blockDim.x)
    indptr[e] = (int64_t)scan[e];
  if (blockIdx.x == 0 && threadIdx.x == 0) *nnz = (int64_t)*total;
}

inline unsigned gridn(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 16));
}

struct CooWs {
  uint32_t *keys, *p1, *p2, *ord, *rs, *cs, *keep, *keep_scan, *rowcnt, *part;
  int8_t *zero;
  double *sums;
  int64_t *pind;
  unsigned char *plan_ws;
  size_t plan_bytes, total;
};

// carve the workspace (sizes only when base == nullptr)
inline CooWs carve(unsigned char *base, int64_t count, int64_t n_rows, int64_t n_cols, size_t plan_bytes) {
  CooWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char *p = base ? base + off : nullptr;
    off += (bytes + 255) & ~(size_t)255;
    return p;
  };
  const int64_t c = std::max<int64_t>(count, 1);
  w.keys = (uint32_t *)take(c * 4);
  w.p1 = (uint32_t *)take(c * 4);
  w.p2 = (uint32_t *)take(c * 4);
  w.ord = (uint32_t *)take(c * 4);
  w.rs = (uint32_t *)take(c * 4);
  w.cs = (uint32_t *)take(c * 4);
  w.keep = (uint32_t *)take(c * 4);
  w.keep_scan = (uint32_t *)take(c * 4);
  w.zero = (int8_t *)take(c);
  w.sums = (double *)take(c * 8);
  w.rowcnt = (uint32_t *)take((n_rows + 1) * 4);
  w.part = (uint32_t *)take((size_t)scan_partials_len(std::max<int64_t>(c, n_rows + 1)) * 4);
  w.pind = (int64_t *)take((std::max(n_rows, n_cols) + 2) * 8);
  w.plan_ws = take(plan_bytes);
  w.plan_bytes = plan_bytes;
  w.total = off;
  return w;
}

inline size_t plan_need(int64_t count, int64_t n_rows, int64_t n_cols) {
  size_t a = 0, b = 0;
  skt_plan_workspace(std::max<int64_t>(count, 1), (uint64_t)std::max<int64_t>(n_cols, 1), 0, &a);
  skt_plan_workspace(std::max<int64_t>(count, 1), (uint64_t)std::max<int64_t>(n_rows, 1), 0, &b);
  return std::max(a, b);
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_coo_to_csr_workspace(int64_t count, int64_t n_rows, int64_t n_cols, size_t *bytes) {
  if (count < 0 || n_rows < 0 || n_cols < 0 || !bytes) return fail(SKT_EINVAL, "skt_coo_to_csr_workspace", "bad arguments");
  *bytes = carve(nullptr, count, n_rows, n_cols, plan_need(count, n_rows, n_cols)).total;
  return SKT_OK;
}

extern "C" skt_status skt_coo_to_csr(const int64_t *rows, const int64_t *cols, const double *vals, int64_t count,
                                     int64_t n_rows, int64_t n_cols, int64_t *indptr, int32_t *indices,
                                     double *out_vals, int64_t *nnz, int32_t *nonfinite, void *ws, size_t ws_bytes,
                                     void *stream_) {
  static const char *fn = "skt_coo_to_csr";
  if (count < 0 || n_rows < 0 || n_cols < 0 || count >= (1LL << 31) || n_rows >= (1LL << 32) ||
      n_cols >= (1LL << 31) || !indptr || !nnz || (count > 0 && (!rows || !cols || !vals || !indices || !out_vals)))
    return fail(SKT_EINVAL, fn, "bad arguments");
  cudaStream_t st = as_stream(stream_);
  const size_t pn = plan_need(count, n_rows, n_cols);
  CooWs w = carve((unsigned char *)ws, count, n_rows, n_cols, pn);
  if (!ws || ws_bytes < w.total) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  SKT_CUDA_TRY(cudaMemsetAsync(w.rowcnt, 0, (n_rows + 1) * 4, st), fn);
  if (nonfinite) SKT_CUDA_TRY(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), st), fn);
  if (count > 0 && n_rows > 0 && n_cols > 0) {
    // (1) stable sort by column, (2) stable sort by row -> (row, col) order, ties in file order
    SKT_LAUNCH(coo_keys_kernel, gridn(count), 256, 0, st, cols, (const uint32_t *)nullptr, count, w.keys, w.zero);
    skt_status s = skt_plan_build(w.keys, w.zero, count, (uint64_t)n_cols, 0, w.pind, w.p1, nullptr, w.plan_ws,
                                  w.plan_bytes, st);
    if (s != SKT_OK) return s;
    SKT_LAUNCH(coo_keys_kernel, gridn(count), 256, 0, st, rows, w.p1, count, w.keys, (int8_t *)nullptr);
    s = skt_plan_build(w.keys, w.zero, count, (uint64_t)n_rows, 0, w.pind, w.p2, nullptr, w.plan_ws, w.plan_bytes, st);
    if (s != SKT_OK) return s;
    SKT_LAUNCH(coo_order_kernel, gridn(count), 256, 0, st, w.p1, w.p2, count, rows, cols, w.ord, w.rs, w.cs);
    SKT_LAUNCH(coo_runs_kernel, gridn(count), 256, 0, st, w.ord, w.rs, w.cs, vals, count, w.sums, w.keep, w.rowcnt,
               nonfinite);
    SKT_CUDA_TRY(cudaMemcpyAsync(w.keep_scan, w.keep, count * 4, cudaMemcpyDeviceToDevice, st), fn);
    s = exclusive_scan_u32(w.keep_scan, count, w.part, st, fn);
    if (s != SKT_OK) return s;
    SKT_LAUNCH(coo_emit_kernel, gridn(count), 256, 0, st, w.keep_scan, w.cs, w.sums, w.keep, count, indices, out_vals);
  }
  const skt_status s2 = exclusive_scan_u32(w.rowcnt, n_rows + 1, w.part, st, fn);
  if (s2 != SKT_OK) return s2;
  const int64_t nbr = (n_rows + 1 + kScanTile - 1) / kScanTile;
  SKT_LAUNCH(coo_indptr_kernel, gridn(n_rows + 1), 256, 0, st, w.rowcnt, n_rows + 1, indptr, w.part + nbr, nnz);
  return check_launch(fn);
}

// ---- canonical-format check on the device --------------------------------
// *flag = 1 if some row's column indices are not strictly increasing
// (duplicates or unsorted: not as_csr's canonical form, _validation.py:30-41)
// -- replaces scipy's O(nnz) host scan (has_canonical_format) before choosing
// the S.A kernel.  The flag is zeroed first.  Warp per 32 entries: entry p is
// checked against entry p - 1 unless p starts its row.
template <typename IP, typename IX>
__global__ void csr_sorted_kernel(int64_t n, const IP *__restrict__ aip, const IX *__restrict__ aix,
                                  int32_t *__restrict__ flag) {
  const int64_t nnz = (int64_t)aip[n];
  const int64_t base = (int64_t)aip[0];
  bool bad = false;
  for (int64_t p = base + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!(__ldg(aix + p) > __ldg(aix + p - 1))) {
      // a row start between p - 1 and p makes the pair unrelated
      int64_t lo = 0, hi = n;  // last row r with aip[r] <= p
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)aip[mid] <= p) lo = mid; else hi = mid;
      }
      if ((int64_t)aip[lo] != p) bad = true;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

extern "C" skt_status skt_csr_check_sorted(int64_t n, const void *a_indptr, skt_itype indptr_type,
                                           const void *a_indices, skt_itype index_type, int32_t *flag,
                                           void *stream_) {
  static const char *fn = "skt_csr_check_sorted";
  if (n < 0 || !a_indptr || !flag || (indptr_type != SKT_I32 && indptr_type != SKT_I64) ||
      (index_type != SKT_I32 && index_type != SKT_I64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  cudaStream_t st = as_stream(stream_);
  SKT_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int32_t), st), fn);
  if (n == 0) return SKT_OK;
  const unsigned blocks = (unsigned)kNumSMs * 8;
  if (indptr_type == SKT_I32) {
    if (index_type == SKT_I32)
      SKT_LAUNCH((csr_sorted_kernel<int32_t, int32_t>), blocks, 256, 0, st, n, (const int32_t *)a_indptr, (const int32_t *)a_indices, flag);
    else
      SKT_LAUNCH((csr_sorted_kernel<int32_t, int64_t>), blocks, 256, 0, st, n, (const int32_t *)a_indptr, (const int64_t *)a_indices, flag);
  } else {
    if (index_type == SKT_I32)
      SKT_LAUNCH((csr_sorted_kernel<int64_t, int32_t>), blocks, 256, 0, st, n, (const int64_t *)a_indptr, (const int32_t *)a_indices, flag);
    else
      SKT_LAUNCH((csr_sorted_kernel<int64_t, int64_t>), blocks, 256, 0, st, n, (const int64_t *)a_indptr, (const int64_t *)a_indices, flag);
  }
  return check_launch(fn);
}
