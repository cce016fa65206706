// apply_csr_wide.cu -- K4 for CSR A too wide for on-chip accumulators of
// whole SA rows: the column-sweep kernel (csr_colsweep.cuh) behind
// skt_apply_csr_wide (sketch.py:155-164, BASELINE config 5).
#include <cstdlib>

#include "common.cuh"
#include "csr_colblock.cuh"
#include "csr_colsweep.cuh"

namespace skt {
namespace {

// ---- column sweep (csr_colsweep.cuh): geometry and launch ------------------
struct ColsweepGeom {
  int nblk;
  int64_t blk_cols;
};
inline int num_sms() {
  static const int n = [] {
    int dev = 0, v = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}
// column blocks per bucket: about 4 waves of 2 CTAs per SM, whole super-steps
inline ColsweepGeom colsweep_geom(uint64_t t, int64_t d) {
  const int64_t steps = std::max<int64_t>(1, (d + kCsStep - 1) / kCsStep);
  const int64_t slots = 2LL * num_sms();
  int64_t nblk = std::min<int64_t>(steps, std::max<int64_t>(1, (4 * slots + (int64_t)t - 1) / (int64_t)t));
  const int64_t per = (steps + nblk - 1) / nblk;
  nblk = (steps + per - 1) / per;
  return ColsweepGeom{(int)nblk, per * kCsStep};
}

// SKT_CSR_WIDE=colsweep selects the column-sweep kernel (A/B)
inline bool use_colsweep() {
  static const bool on = [] {
    const char *e = getenv("SKT_CSR_WIDE");
    return e && e[0] == 'c' && e[3] == 's';
  }();
  return on;
}
inline int colblock_nblk(int64_t d) { return (int)std::max<int64_t>(1, (d + kCbCols - 1) / kCbCols); }

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch_colblock(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                           const void *aix, const void *av, int64_t d, void *sa, int64_t ldsa, int32_t *bnd,
                           cudaStream_t stream) {
  static const char *fn = "skt_apply_csr_wide";
  const int nblk = colblock_nblk(d);
  if (nblk > 1 && n > 0) {
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 16);
    SKT_LAUNCH((csr_colblock_bounds_kernel<IP, IX>), (unsigned)blocks, 256, 0, stream, n, nblk, (const IP *)aip,
               (const IX *)aix, bnd);
    SKT_CUDA_TRY(cudaGetLastError(), fn);
  }
  auto k = csr_colblock_kernel<IP, IX, TV, TOut>;
  const int smem = (int)sizeof(CbSmem);
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), fn);
  SKT_LAUNCH(k, (unsigned)(t * nblk), kCbThreads, smem, stream, pindptr, prow, nblk, d, (const IP *)aip,
             (const IX *)aix, (const TV *)av, bnd, (TOut *)sa, ldsa);
  return check_launch(fn);
}

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch_colsweep(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                           const void *aix, const void *av, int64_t d, void *sa, int64_t ldsa, int32_t *cursor,
                           cudaStream_t stream) {
  static const char *fn = "skt_apply_csr_wide";
  if (!use_colsweep()) return launch_colblock<IP, IX, TV, TOut>(pindptr, prow, t, n, aip, aix, av, d, sa, ldsa, cursor, stream);
  const ColsweepGeom g = colsweep_geom(t, d);
  const int64_t items = (int64_t)n * g.nblk;
  if (items > 0) {
    SKT_LAUNCH((csr_colsweep_init_kernel<IP, IX>), (unsigned)((items + 255) / 256), 256, 0, stream, prow, n,
               g.nblk, g.blk_cols, (const IP *)aip, (const IX *)aix, cursor);
    SKT_CUDA_TRY(cudaGetLastError(), fn);
  }
  auto k = csr_colsweep_kernel<IP, IX, TV, TOut>;
  const int smem = (int)sizeof(CsSmem);
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), fn);
  SKT_LAUNCH(k, (unsigned)(t * g.nblk), kCsThreads, smem, stream, pindptr, prow, n, t, g.nblk, g.blk_cols, d,
             (const IP *)aip, (const IX *)aix, (const TV *)av, cursor, (TOut *)sa, ldsa);
  return check_launch(fn);
}

template <typename IP, typename IX>
skt_status colsweep_by_vals(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                            const void *aix, const void *av, skt_dtype vt, int64_t d, void *sa, skt_dtype ot,
                            int64_t ldsa, int32_t *cursor, cudaStream_t s) {
  if (vt == SKT_F32)
    return ot == SKT_F64 ? launch_colsweep<IP, IX, float, double>(pindptr, prow, t, n, aip, aix, av, d, sa, ldsa, cursor, s)
                         : launch_colsweep<IP, IX, float, float>(pindptr, prow, t, n, aip, aix, av, d, sa, ldsa, cursor, s);
  return ot == SKT_F64 ? launch_colsweep<IP, IX, double, double>(pindptr, prow, t, n, aip, aix, av, d, sa, ldsa, cursor, s)
                       : launch_colsweep<IP, IX, double, float>(pindptr, prow, t, n, aip, aix, av, d, sa, ldsa, cursor, s);
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_apply_csr_wide_workspace(int64_t n, uint64_t t, int64_t d, size_t *bytes) {
  if (!bytes || n < 0 || t < 1 || d < 0) return fail(SKT_EINVAL, "skt_apply_csr_wide_workspace", "bad arguments");
  const size_t sweep = (size_t)std::max<int64_t>(1, n) * (size_t)colsweep_geom(t, d).nblk * sizeof(int32_t);
  const size_t block = (size_t)std::max<int64_t>(1, n) * (size_t)std::max(1, colblock_nblk(d) - 1) * sizeof(int32_t);
  *bytes = std::max(sweep, block);
  return SKT_OK;
}

extern "C" skt_status skt_apply_csr_wide(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                                         const void *a_indptr, skt_itype indptr_type, const void *a_indices,
                                         skt_itype index_type, const void *a_vals, skt_dtype val_dtype,
                                         int64_t nnz, int64_t d, void *sa, skt_dtype sa_dtype, int64_t ldsa,
                                         void *ws, size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_apply_csr_wide";
  if (!indptr || t < 1 || t > (1ull << 32) || n < 0 || d < 0 || ldsa < d || !a_indptr || nnz < 0 ||
      (indptr_type != SKT_I32 && indptr_type != SKT_I64) || (index_type != SKT_I32 && index_type != SKT_I64) ||
      (val_dtype != SKT_F32 && val_dtype != SKT_F64) || (sa_dtype != SKT_F32 && sa_dtype != SKT_F64) ||
      d >= (1LL << 31))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (d == 0) return SKT_OK;
  if (!sa || (n > 0 && !rows)) return fail(SKT_EINVAL, fn, "NULL buffer");
  size_t need = 0;
  skt_apply_csr_wide_workspace(n, t, d, &need);
  if (!ws || ws_bytes < need) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  cudaStream_t s = as_stream(stream_);
  int32_t *cur = (int32_t *)ws;
  if (indptr_type == SKT_I32)
    return index_type == SKT_I32
               ? colsweep_by_vals<int32_t, int32_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, d, sa, sa_dtype, ldsa, cur, s)
               : colsweep_by_vals<int32_t, int64_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, d, sa, sa_dtype, ldsa, cur, s);
  return index_type == SKT_I32
             ? colsweep_by_vals<int64_t, int32_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, d, sa, sa_dtype, ldsa, cur, s)
             : colsweep_by_vals<int64_t, int64_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, d, sa, sa_dtype, ldsa, cur, s);
}
