// residual.cu -- the residual pass of the sketch-and-solve callers
// (regress.py:81-82 `_residual_fro`: ||A X - B||_F on the original data),
// fused: one read of A, the n x k product never leaves registers.
//
// Rows are handled by groups of g lanes (g = the power of two covering d, at
// most 32; 32/g rows per warp step): lane l of a group takes columns / stored
// entries l, l+g, ... of its row and forms the k dot products with X (staged
// in shared memory as fp64) by fp64 FMA, the group reduces them with a fixed
// shuffle butterfly, subtracts B and accumulates the squares.  Warp sums ->
// block sums (fixed order) -> one partial per block in the workspace -> a
// single-block fixed-order reduction writes sum_ij (AX - B)_ij^2 to *out_sq.
// The grid size is fixed, so the result is deterministic run to run; against
// the reference (BLAS gemv/SpMV + norm) it agrees to fp64 rounding.
#include <type_traits>

#include "common.cuh"

namespace skt {
namespace {

constexpr int kResThreads = 256;
constexpr int kResBlocks = kNumSMs * 8;
constexpr size_t kResXSmemMax = 48 * 1024;

__device__ __forceinline__ double group_sum(double v, int g) {
  for (int o = g >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide fixed-order sum of one double per thread; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

template <typename TB>
__device__ __forceinline__ double bval(const TB *b, int64_t i, int64_t ldb, int c) {
  return (double)b[i * ldb + c];
}

template <typename TA, typename TB>
__global__ void __launch_bounds__(kResThreads) resid_dense_kernel(int64_t n, int d, const TA *__restrict__ a,
                                                                  int64_t lda, const double *__restrict__ x,
                                                                  int k, bool x_smem, const TB *__restrict__ b,
                                                                  int64_t ldb, int g, double *__restrict__ part) {
  extern __shared__ double sx[];
  __shared__ double red[kResThreads / 32];
  if (x_smem) {
    for (int i = threadIdx.x; i < d * k; i += blockDim.x) sx[i] = x[i];
    __syncthreads();
  }
  const double *X = x_smem ? sx : x;
  const int lane = threadIdx.x & 31, gl = lane & (g - 1), grp = lane / g, per = 32 / g;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t r0 = warp * per; r0 < n; r0 += nwarps * per) {
    const int64_t i = r0 + grp;
    const bool live = i < n;
    for (int c = 0; c < k; ++c) {
      double dot = 0.0;
      if (live)
        for (int j = gl; j < d; j += g) dot = fma((double)a[i * lda + j], X[(int64_t)j * k + c], dot);
      dot = group_sum(dot, g);
      if (live && gl == 0) {
        const double r = dot - bval(b, i, ldb, c);
        acc = fma(r, r, acc);
      }
    }
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

template <typename IP, typename IX, typename TV, typename TB>
__global__ void __launch_bounds__(kResThreads) resid_csr_kernel(int64_t n, int d, const IP *__restrict__ aip,
                                                                const IX *__restrict__ aix,
                                                                const TV *__restrict__ av,
                                                                const double *__restrict__ x, int k, bool x_smem,
                                                                const TB *__restrict__ b, int64_t ldb, int g,
                                                                double *__restrict__ part) {
  extern __shared__ double sx[];
  __shared__ double red[kResThreads / 32];
  if (x_smem) {
    for (int i = threadIdx.x; i < d * k; i += blockDim.x) sx[i] = x[i];
    __syncthreads();
  }
  const double *X = x_smem ? sx : x;
  const int lane = threadIdx.x & 31, gl = lane & (g - 1), grp = lane / g, per = 32 / g;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t r0 = warp * per; r0 < n; r0 += nwarps * per) {
    const int64_t i = r0 + grp;
    const bool live = i < n;
    int64_t rs = 0, re = 0;
    if (live) {
      rs = (int64_t)aip[i];
      re = (int64_t)aip[i + 1];
    }
    for (int c = 0; c < k; ++c) {
      double dot = 0.0;
      for (int64_t p = rs + gl; p < re; p += g) dot = fma((double)__ldg(av + p), X[(int64_t)__ldg(aix + p) * k + c], dot);
      dot = group_sum(dot, g);
      if (live && gl == 0) {
        const double r = dot - bval(b, i, ldb, c);
        acc = fma(r, r, acc);
      }
    }
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kResThreads) resid_final_kernel(const double *__restrict__ part, int np,
                                                                  double *__restrict__ out) {
  __shared__ double red[kResThreads / 32];
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += part[i];
  const double s = block_sum(v, red);
  if (threadIdx.x == 0) out[0] = s;
}

inline int lanes_for(int64_t width) {
  int g = 1;
  while (g < 32 && g < width) g <<= 1;
  return g;
}

inline int64_t res_blocks(int64_t n, int g) {
  const int64_t rows_per_block = (int64_t)(kResThreads / 32) * (32 / g);
  return std::max<int64_t>(1, std::min<int64_t>(kResBlocks, (n + rows_per_block - 1) / rows_per_block));
}

template <typename TA, typename TB>
skt_status dense_launch(int64_t n, int64_t d, const void *a, int64_t lda, const double *x, int64_t k,
                        const void *b, int64_t ldb, double *out, double *part, cudaStream_t st) {
  static const char *fn = "skt_residual_dense";
  const int g = lanes_for(d);
  const int64_t blocks = res_blocks(n, g);
  const size_t xb = (size_t)d * k * sizeof(double);
  const bool xs = xb <= kResXSmemMax;
  SKT_LAUNCH((resid_dense_kernel<TA, TB>), (unsigned)blocks, kResThreads, xs ? xb : 0, st, n, (int)d,
             (const TA *)a, lda, x, (int)k, xs, (const TB *)b, ldb, g, part);
  SKT_LAUNCH(resid_final_kernel, 1, kResThreads, 0, st, part, (int)blocks, out);
  return check_launch(fn);
}

template <typename IP, typename IX, typename TV, typename TB>
skt_status csr_launch(int64_t n, int64_t d, const void *aip, const void *aix, const void *av,
                      const double *x, int64_t k, const void *b, int64_t ldb, double *out, double *part,
                      cudaStream_t st) {
  static const char *fn = "skt_residual_csr";
  const int g = 16;  // lanes per row: rows of a few to a few dozen stored entries
  const int64_t blocks = res_blocks(n, g);
  const size_t xb = (size_t)d * k * sizeof(double);
  const bool xs = xb <= kResXSmemMax;
  SKT_LAUNCH((resid_csr_kernel<IP, IX, TV, TB>), (unsigned)blocks, kResThreads, xs ? xb : 0, st, n, (int)d,
             (const IP *)aip, (const IX *)aix, (const TV *)av, x, (int)k, xs, (const TB *)b, ldb, g, part);
  SKT_LAUNCH(resid_final_kernel, 1, kResThreads, 0, st, part, (int)blocks, out);
  return check_launch(fn);
}

template <typename IP, typename IX, typename TV>
skt_status csr_by_b(int64_t n, int64_t d, const void *aip, const void *aix, const void *av, const double *x,
                    int64_t k, const void *b, skt_dtype bt, int64_t ldb, double *out, double *part,
                    cudaStream_t st) {
  return bt == SKT_F32 ? csr_launch<IP, IX, TV, float>(n, d, aip, aix, av, x, k, b, ldb, out, part, st)
                       : csr_launch<IP, IX, TV, double>(n, d, aip, aix, av, x, k, b, ldb, out, part, st);
}

template <typename IP, typename IX>
skt_status csr_by_v(int64_t n, int64_t d, const void *aip, const void *aix, const void *av, skt_dtype vt,
                    const double *x, int64_t k, const void *b, skt_dtype bt, int64_t ldb, double *out,
                    double *part, cudaStream_t st) {
  return vt == SKT_F32 ? csr_by_b<IP, IX, float>(n, d, aip, aix, av, x, k, b, bt, ldb, out, part, st)
                       : csr_by_b<IP, IX, double>(n, d, aip, aix, av, x, k, b, bt, ldb, out, part, st);
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_residual_workspace(size_t *bytes) {
  if (!bytes) return fail(SKT_EINVAL, "skt_residual_workspace", "NULL output");
  *bytes = (size_t)kResBlocks * sizeof(double);
  return SKT_OK;
}

extern "C" skt_status skt_residual_dense(int64_t n, int64_t d, const void *a, skt_dtype a_dtype, int64_t lda,
                                         const double *x, int64_t k, const void *b, skt_dtype b_dtype,
                                         int64_t ldb, double *out_sq, void *ws, size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_residual_dense";
  if (n < 0 || d < 0 || k < 1 || lda < d || ldb < k || !out_sq || d >= (1LL << 31) || k >= (1 << 30) ||
      (a_dtype != SKT_F32 && a_dtype != SKT_F64) || (b_dtype != SKT_F32 && b_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (ws_bytes < (size_t)kResBlocks * sizeof(double) || !ws) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  if (n > 0 && (!b || (d > 0 && (!a || !x)))) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
  double *part = (double *)ws;
  if (a_dtype == SKT_F32)
    return b_dtype == SKT_F32 ? dense_launch<float, float>(n, d, a, lda, x, k, b, ldb, out_sq, part, st)
                              : dense_launch<float, double>(n, d, a, lda, x, k, b, ldb, out_sq, part, st);
  return b_dtype == SKT_F32 ? dense_launch<double, float>(n, d, a, lda, x, k, b, ldb, out_sq, part, st)
                            : dense_launch<double, double>(n, d, a, lda, x, k, b, ldb, out_sq, part, st);
}

extern "C" skt_status skt_residual_csr(int64_t n, int64_t d, const void *a_indptr, skt_itype indptr_type,
                                       const void *a_indices, skt_itype index_type, const void *a_vals,
                                       skt_dtype val_dtype, const double *x, int64_t k, const void *b,
                                       skt_dtype b_dtype, int64_t ldb, double *out_sq, void *ws,
                                       size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_residual_csr";
  if (n < 0 || d < 0 || k < 1 || ldb < k || !out_sq || d >= (1LL << 31) || k >= (1 << 30) ||
      (indptr_type != SKT_I32 && indptr_type != SKT_I64) || (index_type != SKT_I32 && index_type != SKT_I64) ||
      (val_dtype != SKT_F32 && val_dtype != SKT_F64) || (b_dtype != SKT_F32 && b_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (ws_bytes < (size_t)kResBlocks * sizeof(double) || !ws) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  if (n > 0 && (!a_indptr || !b || (d > 0 && !x))) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
  double *part = (double *)ws;
  if (indptr_type == SKT_I32)
    return index_type == SKT_I32
               ? csr_by_v<int32_t, int32_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, x, k, b, b_dtype, ldb, out_sq, part, st)
               : csr_by_v<int32_t, int64_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, x, k, b, b_dtype, ldb, out_sq, part, st);
  return index_type == SKT_I32
             ? csr_by_v<int64_t, int32_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, x, k, b, b_dtype, ldb, out_sq, part, st)
             : csr_by_v<int64_t, int64_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, x, k, b, b_dtype, ldb, out_sq, part, st);
}
