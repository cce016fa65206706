// apply_right.cu -- column sketch Y = A . S^T (reference apply_right,
// sketch.py:445-448: (S.apply(A.T)).T, which materialises the transpose and
// then scatters).  Here the work is row-local and transpose-free: one warp
// owns one row i of A, keeps Y[i, :] as t fp64 accumulators in shared memory
// and walks the row's entries in ascending column order, adding
// s(j) * A[i, j] into bucket h(j).  Per output (i, b) that is ascending j --
// the reference's order -- so fp64 results are bit-identical.  Lanes of one
// 32-column chunk that hash to the same bucket are serialised in lane (=
// column) order with __match_any_sync.
#include "common.cuh"

namespace skt {
namespace {

constexpr int kMaxWarps = 8;

__device__ __forceinline__ bool nonfinite(float x) {
  return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}
__device__ __forceinline__ bool nonfinite(double x) {
  return ((uint32_t)(__double_as_longlong(x) >> 32) & 0x7ff00000u) == 0x7ff00000u;
}

__device__ __forceinline__ void ordered_add(double *acc, int b, double v, bool has) {
  const uint32_t lt_mask = (1u << (threadIdx.x & 31)) - 1u;
  const uint32_t peers = __match_any_sync(0xffffffffu, has ? b : -1);
  const int rank = __popc(peers & lt_mask);
  const int rounds = __reduce_max_sync(0xffffffffu, has ? rank + 1 : 0);
  if (rounds == 1) {
    if (has) acc[b] += v;
  } else {
    for (int rr = 0; rr < rounds; ++rr) {
      if (has && rank == rr) acc[b] += v;
      __syncwarp();
    }
  }
  __syncwarp();
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kMaxWarps * 32) right_dense_kernel(
    const uint32_t *__restrict__ h, const int8_t *__restrict__ s, uint64_t t, int64_t n_rows,
    int64_t ncols, const TIn *__restrict__ a, int64_t lda, TOut *__restrict__ y, int64_t ldy,
    int32_t *__restrict__ flag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (i >= n_rows) return;
  const size_t slice = ((size_t)t * 8 + 15) & ~(size_t)15;
  double *acc = (double *)(smem_raw + w * slice);
  for (int64_t b = lane; b < (int64_t)t; b += 32) acc[b] = 0.0;
  __syncwarp();
  bool bad = false;
  const TIn *arow = a + i * lda;
  for (int64_t j0 = 0; j0 < ncols; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool has = j < ncols;
    const TIn x = has ? arow[j] : (TIn)0;
    bad |= nonfinite(x);
    const int b = has ? (int)__ldg(h + j) : 0;
    const double v = (has && __ldg(s + j) < 0) ? -(double)x : (double)x;
    ordered_add(acc, b, v, has);
  }
  TOut *o = y + i * ldy;
  for (int64_t b = lane; b < (int64_t)t; b += 32) o[b] = (TOut)acc[b];
  if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

template <typename IP, typename IX, typename TV, typename TOut>
__global__ void __launch_bounds__(kMaxWarps * 32) right_csr_kernel(
    const uint32_t *__restrict__ h, const int8_t *__restrict__ s, uint64_t t, int64_t n_rows,
    const IP *__restrict__ aip, const IX *__restrict__ aix, const TV *__restrict__ av,
    TOut *__restrict__ y, int64_t ldy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (i >= n_rows) return;
  const size_t slice = ((size_t)t * 8 + 15) & ~(size_t)15;
  double *acc = (double *)(smem_raw + w * slice);
  for (int64_t b = lane; b < (int64_t)t; b += 32) acc[b] = 0.0;
  __syncwarp();
  const int64_t rs = (int64_t)aip[i], re = (int64_t)aip[i + 1];
  for (int64_t p0 = rs; p0 < re; p0 += 32) {
    const int64_t p = p0 + lane;
    const bool has = p < re;
    const int64_t j = has ? (int64_t)aix[p] : 0;
    const double x = has ? (double)av[p] : 0.0;
    const int b = has ? (int)__ldg(h + j) : 0;
    const double v = (has && __ldg(s + j) < 0) ? -x : x;
    ordered_add(acc, b, v, has);
  }
  TOut *o = y + i * ldy;
  for (int64_t b = lane; b < (int64_t)t; b += 32) o[b] = (TOut)acc[b];
}

struct Cfg {
  int warps;
  size_t smem;
};
inline skt_status config(uint64_t t, const char *fn, Cfg *c) {
  const size_t slice = ((size_t)t * 8 + 15) & ~(size_t)15;
  const size_t kSmemMax = 200 * 1024;
  c->warps = (int)std::min<size_t>(kMaxWarps, kSmemMax / slice);
  if (c->warps < 1) return fail(SKT_ENOTSUP, fn, "t too large for the shared-memory accumulator");
  c->smem = slice * c->warps;
  return SKT_OK;
}

template <typename TIn, typename TOut>
skt_status launch_dense(const uint32_t *h, const int8_t *s, uint64_t t, int64_t n_rows,
                        int64_t ncols, const void *a, int64_t lda, void *y, int64_t ldy,
                        int32_t *flag, cudaStream_t stream) {
  static const char *fn = "skt_apply_right_dense";
  Cfg c;
  skt_status st = config(t, fn, &c);
  if (st != SKT_OK) return st;
  auto k = right_dense_kernel<TIn, TOut>;
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem), fn);
  const int64_t blocks = (n_rows + c.warps - 1) / c.warps;
  SKT_LAUNCH(k, (unsigned)blocks, c.warps * 32, c.smem, stream, h, s, t, n_rows, ncols,
             (const TIn *)a, lda, (TOut *)y, ldy, flag);
  return check_launch(fn);
}

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch_csr(const uint32_t *h, const int8_t *s, uint64_t t, int64_t n_rows,
                      const void *aip, const void *aix, const void *av, void *y, int64_t ldy,
                      cudaStream_t stream) {
  static const char *fn = "skt_apply_right_csr";
  Cfg c;
  skt_status st = config(t, fn, &c);
  if (st != SKT_OK) return st;
  auto k = right_csr_kernel<IP, IX, TV, TOut>;
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem), fn);
  const int64_t blocks = (n_rows + c.warps - 1) / c.warps;
  SKT_LAUNCH(k, (unsigned)blocks, c.warps * 32, c.smem, stream, h, s, t, n_rows, (const IP *)aip,
             (const IX *)aix, (const TV *)av, (TOut *)y, ldy);
  return check_launch(fn);
}

template <typename IP, typename IX>
skt_status csr_vals(const uint32_t *h, const int8_t *s, uint64_t t, int64_t n_rows, const void *aip,
                    const void *aix, const void *av, skt_dtype vt, void *y, skt_dtype yt,
                    int64_t ldy, cudaStream_t st) {
  if (vt == SKT_F32)
    return yt == SKT_F64 ? launch_csr<IP, IX, float, double>(h, s, t, n_rows, aip, aix, av, y, ldy, st)
                         : launch_csr<IP, IX, float, float>(h, s, t, n_rows, aip, aix, av, y, ldy, st);
  return yt == SKT_F64 ? launch_csr<IP, IX, double, double>(h, s, t, n_rows, aip, aix, av, y, ldy, st)
                       : launch_csr<IP, IX, double, float>(h, s, t, n_rows, aip, aix, av, y, ldy, st);
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_apply_right_dense(const uint32_t *h, const int8_t *s, uint64_t t,
                                            int64_t n_rows, int64_t ncols, const void *a,
                                            skt_dtype a_dtype, int64_t lda, void *y,
                                            skt_dtype y_dtype, int64_t ldy,
                                            int32_t *nonfinite_flag, void *stream_) {
  static const char *fn = "skt_apply_right_dense";
  if (t < 1 || t > (1ull << 31) || n_rows < 0 || ncols < 0 || lda < ncols || ldy < (int64_t)t ||
      (a_dtype != SKT_F32 && a_dtype != SKT_F64) || (y_dtype != SKT_F32 && y_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  cudaStream_t stream = as_stream(stream_);
  if (nonfinite_flag) SKT_CUDA_TRY(cudaMemsetAsync(nonfinite_flag, 0, sizeof(int32_t), stream), fn);
  if (n_rows == 0) return SKT_OK;
  if (!y || (ncols > 0 && (!a || !h || !s))) return fail(SKT_EINVAL, fn, "NULL buffer");
  if (a_dtype == SKT_F32)
    return y_dtype == SKT_F64 ? launch_dense<float, double>(h, s, t, n_rows, ncols, a, lda, y, ldy, nonfinite_flag, stream)
                              : launch_dense<float, float>(h, s, t, n_rows, ncols, a, lda, y, ldy, nonfinite_flag, stream);
  return y_dtype == SKT_F64 ? launch_dense<double, double>(h, s, t, n_rows, ncols, a, lda, y, ldy, nonfinite_flag, stream)
                            : launch_dense<double, float>(h, s, t, n_rows, ncols, a, lda, y, ldy, nonfinite_flag, stream);
}

extern "C" skt_status skt_apply_right_csr(const uint32_t *h, const int8_t *s, uint64_t t,
                                          int64_t n_rows, int64_t ncols, const void *a_indptr,
                                          skt_itype indptr_type, const void *a_indices,
                                          skt_itype index_type, const void *a_vals,
                                          skt_dtype val_dtype, void *y, skt_dtype y_dtype,
                                          int64_t ldy, void *stream_) {
  static const char *fn = "skt_apply_right_csr";
  if (t < 1 || t > (1ull << 31) || n_rows < 0 || ncols < 0 || ldy < (int64_t)t || !a_indptr ||
      (indptr_type != SKT_I32 && indptr_type != SKT_I64) ||
      (index_type != SKT_I32 && index_type != SKT_I64) ||
      (val_dtype != SKT_F32 && val_dtype != SKT_F64) || (y_dtype != SKT_F32 && y_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (n_rows == 0) return SKT_OK;
  if (!y || (ncols > 0 && (!h || !s))) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
  if (indptr_type == SKT_I32)
    return index_type == SKT_I32
               ? csr_vals<int32_t, int32_t>(h, s, t, n_rows, a_indptr, a_indices, a_vals, val_dtype, y, y_dtype, ldy, st)
               : csr_vals<int32_t, int64_t>(h, s, t, n_rows, a_indptr, a_indices, a_vals, val_dtype, y, y_dtype, ldy, st);
  return index_type == SKT_I32
             ? csr_vals<int64_t, int32_t>(h, s, t, n_rows, a_indptr, a_indices, a_vals, val_dtype, y, y_dtype, ldy, st)
             : csr_vals<int64_t, int64_t>(h, s, t, n_rows, a_indptr, a_indices, a_vals, val_dtype, y, y_dtype, ldy, st);
}
