// lsq.cu -- passes over the original data that follow the sketch (SURVEY §8f
// rank 2): the products of the preconditioned iterations (regress.py:192-283,
// M = A R), the sparse product that forms M for CSR A, and the Gram-identity
// residual of the rank-k approximation (lowrank.py:100-108).
//
// Every pass reads its big operand once, keeps the per-row work in registers
// and reduces deterministically: warp shuffles in a fixed butterfly, warps of a
// block in index order, one partial per block in a caller workspace, then a
// single fixed-order reduction kernel -- the same bits run to run.  Against
// the reference's numpy / scipy products the values agree to fp64 rounding.
//
//  * skt_spmm_csr          Y = A X (n x k), A CSR, X d x k fp64 (M = A R)
//  * skt_lsq_residual_grad res2 = ||b - M y||^2 and g = M^T (b - M y)
//                          (Richardson: one pass per iteration; the residual
//                          of iterate y is the one _iterate records)
//  * skt_lsq_matvec_norm   q = M p, qq = ||q||^2 (CGNR's M p and denom)
//  * skt_lsq_update_grad   r <- r - alpha q, z = M^T r, res2 = ||M y - b||^2
//                          (CGNR's residual update, M^T r and _iterate's
//                          residual of the new iterate in one pass)
//  * skt_gram_cross_csr /_dense  cross = sum_i <A_i M, L_i>, fro2 = ||A||_F^2
//                          (M = W diag(d), one pass over A)
//
// M is row-major n x r (r <= 256, lda = ldm); a warp owns one row at a time,
// lane l holds M[i, l + 32 q] for q < Q.  One right-hand-side column per call
// (the callers loop over columns of b).
#include <type_traits>

#include "common.cuh"

namespace skt {
namespace {

constexpr int kLsqThreads = 256;
constexpr int kLsqWarps = kLsqThreads / 32;
constexpr int kLsqBlocks = kNumSMs * 4;
constexpr int kLsqMaxR = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order block reduction of `cnt` per-warp vectors red[w][j] -> part[j]
__device__ __forceinline__ void block_vec_reduce(const double *red, int cnt, double *part) {
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kLsqWarps; ++w) s += red[w * cnt + j];
    part[j] = s;
  }
}

// ---- Richardson: res2 = ||b - M y||^2, g = M^T (b - M y) -------------------
// workspace per block: [r values of g][res2]
template <int Q>
__global__ void __launch_bounds__(kLsqThreads) lsq_resgrad_kernel(int64_t n, int r, const double *__restrict__ m,
                                                                  int64_t ldm, const double *__restrict__ y,
                                                                  const double *__restrict__ b, int64_t ldb,
                                                                  double *__restrict__ part) {
  extern __shared__ double red[];  // [warps][r + 1]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double yl[Q], gl[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = lane + 32 * q;
    yl[q] = j < r ? y[j] : 0.0;
    gl[q] = 0.0;
  }
  double res = 0.0;
  const int64_t warp = ((int64_t)blockIdx.x * kLsqThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kLsqThreads) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    double ml[Q];
    double dot = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = lane + 32 * q;
      ml[q] = j < r ? __ldg(m + i * ldm + j) : 0.0;
      dot = fma(ml[q], yl[q], dot);
    }
    dot = warp_sum(dot);
    const double ri = __ldg(b + i * ldb) - dot;
    res = fma(ri, ri, res);
#pragma unroll
    for (int q = 0; q < Q; ++q) gl[q] = fma(ml[q], ri, gl[q]);
  }
  const int cnt = r + 1;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = lane + 32 * q;
    if (j < r) red[w * cnt + j] = gl[q];
  }
  if (lane == 0) red[w * cnt + r] = res;  // every lane holds the same res
  __syncthreads();
  block_vec_reduce(red, cnt, part + (size_t)blockIdx.x * cnt);
}

// ---- CGNR (a): q = M p, qq = ||q||^2 ---------------------------------------
template <int Q>
__global__ void __launch_bounds__(kLsqThreads) lsq_matvec_kernel(int64_t n, int r, const double *__restrict__ m,
                                                                 int64_t ldm, const double *__restrict__ p,
                                                                 double *__restrict__ qv, int64_t ldq,
                                                                 double *__restrict__ part) {
  __shared__ double red[kLsqWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double pl[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = lane + 32 * q;
    pl[q] = j < r ? p[j] : 0.0;
  }
  double acc = 0.0;
  const int64_t warp = ((int64_t)blockIdx.x * kLsqThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kLsqThreads) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    double dot = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = lane + 32 * q;
      if (j < r) dot = fma(__ldg(m + i * ldm + j), pl[q], dot);
    }
    dot = warp_sum(dot);
    if (lane == 0) qv[i * ldq] = dot;
    acc = fma(dot, dot, acc);
  }
  if (lane == 0) red[w] = acc;
  __syncthreads();
  block_vec_reduce(red, 1, part + blockIdx.x);
}

// ---- CGNR (b): r <- r - alpha q; z = M^T r; res2 = ||M y - b||^2 -------------
template <int Q>
__global__ void __launch_bounds__(kLsqThreads) lsq_update_kernel(int64_t n, int r, const double *__restrict__ m,
                                                                 int64_t ldm, const double *__restrict__ qv,
                                                                 int64_t ldq, double alpha, double *__restrict__ rv,
                                                                 int64_t ldr, const double *__restrict__ y,
                                                                 const double *__restrict__ b, int64_t ldb,
                                                                 double *__restrict__ part) {
  extern __shared__ double red[];  // [warps][r + 1]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double yl[Q], zl[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = lane + 32 * q;
    yl[q] = j < r ? y[j] : 0.0;
    zl[q] = 0.0;
  }
  double res = 0.0;
  const int64_t warp = ((int64_t)blockIdx.x * kLsqThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kLsqThreads) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    double ml[Q];
    double dot = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = lane + 32 * q;
      ml[q] = j < r ? __ldg(m + i * ldm + j) : 0.0;
      dot = fma(ml[q], yl[q], dot);
    }
    dot = warp_sum(dot);
    const double e = dot - __ldg(b + i * ldb);
    res = fma(e, e, res);
    // r_i - q_i * alpha, as numpy's r - mp * alpha (product rounded, then the
    // subtraction; no fused multiply-add)
    const double ri = __dsub_rn(rv[i * ldr], __dmul_rn(qv[i * ldq], alpha));
    __syncwarp();
    if (lane == 0) rv[i * ldr] = ri;
#pragma unroll
    for (int q = 0; q < Q; ++q) zl[q] = fma(ml[q], ri, zl[q]);
  }
  const int cnt = r + 1;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = lane + 32 * q;
    if (j < r) red[w * cnt + j] = zl[q];
  }
  if (lane == 0) red[w * cnt + r] = res;
  __syncthreads();
  block_vec_reduce(red, cnt, part + (size_t)blockIdx.x * cnt);
}

// fixed-order sum over blocks of the per-block vectors: out[j] = sum_b part[b][j]
__global__ void __launch_bounds__(kLsqThreads) lsq_final_kernel(const double *__restrict__ part, int nblocks,
                                                                int cnt, double *__restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int bk = 0; bk < nblocks; ++bk) s += part[(size_t)bk * cnt + j];
    out[j] = s;
  }
}

// ---- Y = A X for CSR A (M = A R for a sparse A) ----------------------------
// g lanes per row (g | 32), lane-partial dot products reduced by a butterfly
template <typename IP, typename IX, typename TV>
__global__ void __launch_bounds__(kLsqThreads) spmm_csr_kernel(int64_t n, const IP *__restrict__ aip,
                                                               const IX *__restrict__ aix,
                                                               const TV *__restrict__ av,
                                                               const double *__restrict__ x, int k, int g,
                                                               double *__restrict__ yv, int64_t ldy) {
  const int lane = threadIdx.x & 31, gl = lane & (g - 1), grp = lane / g, per = 32 / g;
  const int64_t warp = ((int64_t)blockIdx.x * kLsqThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kLsqThreads) >> 5;
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
      for (int64_t p = rs + gl; p < re; p += g) dot = fma((double)__ldg(av + p), x[(int64_t)__ldg(aix + p) * k + c], dot);
      for (int o = g >> 1; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (live && gl == 0) yv[i * ldy + c] = dot;
    }
  }
}

// ---- Y = A X for dense A (M = A R, regress.py:200) ---------------------------
// One output element per thread (block = 256 consecutive elements of the
// row-major n x k result); X is staged through shared memory in chunks of
// rows, A[i, c] is read from L1/L2 (lanes of a warp share few rows); the dot
// product runs over c in ascending order with fma, fp64.
constexpr int kGemmChunk = 4096;  // doubles of X per shared-memory chunk (32 KB)

template <typename TA>
__global__ void __launch_bounds__(256) gemm_dense_kernel(int64_t n, int64_t d, const TA *__restrict__ a, int64_t lda,
                                                         const double *__restrict__ x, int64_t k,
                                                         double *__restrict__ y, int64_t ldy) {
  __shared__ double xs[kGemmChunk];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = e < n * k;
  const int64_t i = live ? e / k : 0, j = live ? e - i * k : 0;
  const int64_t rows = std::max<int64_t>(1, kGemmChunk / k);
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < d; c0 += rows) {
    const int64_t c1 = std::min<int64_t>(d, c0 + rows);
    __syncthreads();
    for (int64_t q = threadIdx.x; q < (c1 - c0) * k; q += blockDim.x) xs[q] = x[c0 * k + q];
    __syncthreads();
    if (live) {
      const TA *ar = a + i * lda;
      for (int64_t c = c0; c < c1; ++c) acc = fma((double)__ldg(ar + c), xs[(c - c0) * k + j], acc);
    }
  }
  if (live) y[i * ldy + j] = acc;
}

// ---- Gram-identity residual: cross = sum_i <A_i M, L_i>, fro2 = sum a^2 ------
// warp per row; lane takes stored entries p = rs + lane (+32): <M[col_p], L_i>
// from L_i staged in shared memory (k <= 64)
constexpr int kGramMaxK = 64;

template <typename IP, typename IX, typename TV>
__global__ void __launch_bounds__(kLsqThreads) gram_csr_kernel(int64_t n, const IP *__restrict__ aip,
                                                               const IX *__restrict__ aix,
                                                               const TV *__restrict__ av,
                                                               const double *__restrict__ mw, int64_t ldm, int k,
                                                               const double *__restrict__ l, int64_t ldl,
                                                               double *__restrict__ part) {
  __shared__ double sl[kLsqWarps][kGramMaxK];
  __shared__ double red[kLsqWarps * 2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double cross = 0.0, fro = 0.0;
  const int64_t warp = ((int64_t)blockIdx.x * kLsqThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kLsqThreads) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    __syncwarp();
    for (int c = lane; c < k; c += 32) sl[w][c] = l[i * ldl + c];
    __syncwarp();
    const int64_t rs = (int64_t)aip[i], re = (int64_t)aip[i + 1];
    for (int64_t p = rs + lane; p < re; p += 32) {
      const double a = (double)__ldg(av + p);
      const double *mr = mw + (int64_t)__ldg(aix + p) * ldm;
      double dot = 0.0;
      for (int c = 0; c < k; ++c) dot = fma(__ldg(mr + c), sl[w][c], dot);
      cross = fma(a, dot, cross);
      fro = fma(a, a, fro);
    }
  }
  cross = warp_sum(cross);
  fro = warp_sum(fro);
  if (lane == 0) {
    red[w] = cross;
    red[kLsqWarps + w] = fro;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int i = 0; i < kLsqWarps; ++i) s += red[threadIdx.x * kLsqWarps + i];
    part[(size_t)blockIdx.x * 2 + threadIdx.x] = s;
  }
}

template <typename TA>
__global__ void __launch_bounds__(kLsqThreads) gram_dense_kernel(int64_t n, int64_t ncols, const TA *__restrict__ a,
                                                                 int64_t lda, const double *__restrict__ mw,
                                                                 int64_t ldm, int k, const double *__restrict__ l,
                                                                 int64_t ldl, double *__restrict__ part) {
  __shared__ double sl[kLsqWarps][kGramMaxK];
  __shared__ double red[kLsqWarps * 2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double cross = 0.0, fro = 0.0;
  const int64_t warp = ((int64_t)blockIdx.x * kLsqThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kLsqThreads) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    __syncwarp();
    for (int c = lane; c < k; c += 32) sl[w][c] = l[i * ldl + c];
    __syncwarp();
    for (int64_t j = lane; j < ncols; j += 32) {
      const double x = (double)__ldg(a + i * lda + j);
      const double *mr = mw + j * ldm;
      double dot = 0.0;
      for (int c = 0; c < k; ++c) dot = fma(__ldg(mr + c), sl[w][c], dot);
      cross = fma(x, dot, cross);
      fro = fma(x, x, fro);
    }
  }
  cross = warp_sum(cross);
  fro = warp_sum(fro);
  if (lane == 0) {
    red[w] = cross;
    red[kLsqWarps + w] = fro;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int i = 0; i < kLsqWarps; ++i) s += red[threadIdx.x * kLsqWarps + i];
    part[(size_t)blockIdx.x * 2 + threadIdx.x] = s;
  }
}

inline int64_t lsq_blocks(int64_t rows) {
  return std::max<int64_t>(1, std::min<int64_t>(kLsqBlocks, (rows + kLsqWarps - 1) / kLsqWarps));
}


#define SKT_Q_DISPATCH(r, KERNEL, ...)                                      \
  ((r) <= 32 ? KERNEL<1>(__VA_ARGS__)                                       \
             : (r) <= 64 ? KERNEL<2>(__VA_ARGS__)                           \
                         : (r) <= 128 ? KERNEL<4>(__VA_ARGS__) : KERNEL<8>(__VA_ARGS__))

template <int Q>
skt_status launch_resgrad(int64_t n, int r, const double *m, int64_t ldm, const double *y, const double *b,
                          int64_t ldb, double *g, double *res2, double *part, cudaStream_t st) {
  const int64_t blocks = lsq_blocks(n);
  const size_t smem = (size_t)kLsqWarps * (r + 1) * sizeof(double);
  SKT_LAUNCH(lsq_resgrad_kernel<Q>, (unsigned)blocks, kLsqThreads, smem, st, n, r, m, ldm, y, b, ldb, part);
  // out = [g (r), res2]: g's slot first, res2 after it -- written to g[0..r) and res2
  double *fin = part + (size_t)blocks * (r + 1);
  SKT_LAUNCH(lsq_final_kernel, 1, kLsqThreads, 0, st, part, (int)blocks, r + 1, fin);
  if (g && r > 0) SKT_CUDA_TRY(cudaMemcpyAsync(g, fin, (size_t)r * sizeof(double), cudaMemcpyDeviceToDevice, st), "skt_lsq_residual_grad");
  SKT_CUDA_TRY(cudaMemcpyAsync(res2, fin + r, sizeof(double), cudaMemcpyDeviceToDevice, st), "skt_lsq_residual_grad");
  return check_launch("skt_lsq_residual_grad");
}

template <int Q>
skt_status launch_matvec(int64_t n, int r, const double *m, int64_t ldm, const double *p, double *qv, int64_t ldq,
                         double *qq, double *part, cudaStream_t st) {
  const int64_t blocks = lsq_blocks(n);
  SKT_LAUNCH(lsq_matvec_kernel<Q>, (unsigned)blocks, kLsqThreads, 0, st, n, r, m, ldm, p, qv, ldq, part);
  SKT_LAUNCH(lsq_final_kernel, 1, kLsqThreads, 0, st, part, (int)blocks, 1, qq);
  return check_launch("skt_lsq_matvec_norm");
}

template <int Q>
skt_status launch_update(int64_t n, int r, const double *m, int64_t ldm, const double *qv, int64_t ldq, double alpha,
                         double *rv, int64_t ldr, const double *y, const double *b, int64_t ldb, double *z,
                         double *res2, double *part, cudaStream_t st) {
  const int64_t blocks = lsq_blocks(n);
  const size_t smem = (size_t)kLsqWarps * (r + 1) * sizeof(double);
  SKT_LAUNCH(lsq_update_kernel<Q>, (unsigned)blocks, kLsqThreads, smem, st, n, r, m, ldm, qv, ldq, alpha, rv, ldr, y,
             b, ldb, part);
  double *fin = part + (size_t)blocks * (r + 1);
  SKT_LAUNCH(lsq_final_kernel, 1, kLsqThreads, 0, st, part, (int)blocks, r + 1, fin);
  if (r > 0) SKT_CUDA_TRY(cudaMemcpyAsync(z, fin, (size_t)r * sizeof(double), cudaMemcpyDeviceToDevice, st), "skt_lsq_update_grad");
  SKT_CUDA_TRY(cudaMemcpyAsync(res2, fin + r, sizeof(double), cudaMemcpyDeviceToDevice, st), "skt_lsq_update_grad");
  return check_launch("skt_lsq_update_grad");
}

template <typename IP, typename IX, typename TV>
skt_status launch_spmm(int64_t n, const void *aip, const void *aix, const void *av, const double *x, int64_t k,
                       double *y, int64_t ldy, int64_t nnz, cudaStream_t st) {
  const int64_t mean = n > 0 ? nnz / n : 0;
  int g = 1;
  while (g < 32 && g < mean) g <<= 1;
  const int64_t rows_per_block = (int64_t)kLsqWarps * (32 / g);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)kNumSMs * 8, (n + rows_per_block - 1) / rows_per_block));
  SKT_LAUNCH((spmm_csr_kernel<IP, IX, TV>), (unsigned)blocks, kLsqThreads, 0, st, n, (const IP *)aip, (const IX *)aix,
             (const TV *)av, x, (int)k, g, y, ldy);
  return check_launch("skt_spmm_csr");
}

template <typename IP, typename IX, typename TV>
skt_status launch_gram_csr(int64_t n, const void *aip, const void *aix, const void *av, const double *mw, int64_t ldm,
                           int k, const double *l, int64_t ldl, double *out, double *part, cudaStream_t st) {
  const int64_t blocks = lsq_blocks(n);
  SKT_LAUNCH((gram_csr_kernel<IP, IX, TV>), (unsigned)blocks, kLsqThreads, 0, st, n, (const IP *)aip,
             (const IX *)aix, (const TV *)av, mw, ldm, k, l, ldl, part);
  SKT_LAUNCH(lsq_final_kernel, 1, kLsqThreads, 0, st, part, (int)blocks, 2, out);
  return check_launch("skt_gram_cross_csr");
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_lsq_workspace(int64_t r, size_t *bytes) {
  if (!bytes || r < 0 || r > kLsqMaxR) return fail(SKT_EINVAL, "skt_lsq_workspace", "bad arguments");
  *bytes = ((size_t)kLsqBlocks + 1) * (size_t)(r + 2) * sizeof(double);
  return SKT_OK;
}

#define SKT_LSQ_WS_CHECK(fn, r)                                                             \
  do {                                                                                      \
    size_t need = 0;                                                                        \
    if (skt_lsq_workspace((r), &need) != SKT_OK) return fail(SKT_EINVAL, fn, "r out of range (0..256)"); \
    if (!ws || ws_bytes < need) return fail(SKT_EWORKSPACE, fn, "workspace too small");    \
  } while (0)

extern "C" skt_status skt_lsq_residual_grad(int64_t n, int64_t r, const double *m, int64_t ldm, const double *y,
                                            const double *b, int64_t ldb, double *g, double *res2, void *ws,
                                            size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_lsq_residual_grad";
  if (n < 0 || r < 0 || ldm < r || ldb < 1 || !res2 || (n > 0 && (!b || (r > 0 && (!m || !y)))))
    return fail(SKT_EINVAL, fn, "bad arguments");
  SKT_LSQ_WS_CHECK(fn, r);
  cudaStream_t st = as_stream(stream_);
  return SKT_Q_DISPATCH(r, launch_resgrad, n, (int)r, m, ldm, y, b, ldb, g, res2, (double *)ws, st);
}

extern "C" skt_status skt_lsq_matvec_norm(int64_t n, int64_t r, const double *m, int64_t ldm, const double *p,
                                          double *q, int64_t ldq, double *qq, void *ws, size_t ws_bytes,
                                          void *stream_) {
  static const char *fn = "skt_lsq_matvec_norm";
  if (n < 0 || r < 0 || ldm < r || ldq < 1 || !qq || (n > 0 && (!q || (r > 0 && (!m || !p)))))
    return fail(SKT_EINVAL, fn, "bad arguments");
  SKT_LSQ_WS_CHECK(fn, r);
  cudaStream_t st = as_stream(stream_);
  return SKT_Q_DISPATCH(r, launch_matvec, n, (int)r, m, ldm, p, q, ldq, qq, (double *)ws, st);
}

extern "C" skt_status skt_lsq_update_grad(int64_t n, int64_t r, const double *m, int64_t ldm, const double *q,
                                          int64_t ldq, double alpha, double *rvec, int64_t ldr, const double *y,
                                          const double *b, int64_t ldb, double *z, double *res2, void *ws,
                                          size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_lsq_update_grad";
  if (n < 0 || r < 0 || ldm < r || ldq < 1 || ldr < 1 || ldb < 1 || !res2 || (r > 0 && !z) ||
      (n > 0 && (!q || !rvec || !b || (r > 0 && (!m || !y)))))
    return fail(SKT_EINVAL, fn, "bad arguments");
  SKT_LSQ_WS_CHECK(fn, r);
  cudaStream_t st = as_stream(stream_);
  return SKT_Q_DISPATCH(r, launch_update, n, (int)r, m, ldm, q, ldq, alpha, rvec, ldr, y, b, ldb, z, res2,
                        (double *)ws, st);
}

extern "C" skt_status skt_spmm_csr(int64_t n, int64_t d, const void *a_indptr, skt_itype indptr_type,
                                   const void *a_indices, skt_itype index_type, const void *a_vals,
                                   skt_dtype val_dtype, int64_t nnz, const double *x, int64_t k, double *y,
                                   int64_t ldy, void *stream_) {
  static const char *fn = "skt_spmm_csr";
  if (n < 0 || d < 0 || k < 0 || nnz < 0 || ldy < k || (indptr_type != SKT_I32 && indptr_type != SKT_I64) ||
      (index_type != SKT_I32 && index_type != SKT_I64) || (val_dtype != SKT_F32 && val_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (n == 0 || k == 0) return SKT_OK;
  if (!a_indptr || !y || (d > 0 && !x)) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
#define SKT_SPMM(IP, IX)                                                                              \
  (val_dtype == SKT_F32 ? launch_spmm<IP, IX, float>(n, a_indptr, a_indices, a_vals, x, k, y, ldy, nnz, st) \
                        : launch_spmm<IP, IX, double>(n, a_indptr, a_indices, a_vals, x, k, y, ldy, nnz, st))
  if (indptr_type == SKT_I32) return index_type == SKT_I32 ? SKT_SPMM(int32_t, int32_t) : SKT_SPMM(int32_t, int64_t);
  return index_type == SKT_I32 ? SKT_SPMM(int64_t, int32_t) : SKT_SPMM(int64_t, int64_t);
#undef SKT_SPMM
}

extern "C" skt_status skt_gram_cross_csr(int64_t n, int64_t ncols, const void *a_indptr, skt_itype indptr_type,
                                         const void *a_indices, skt_itype index_type, const void *a_vals,
                                         skt_dtype val_dtype, const double *mw, int64_t ldm, int64_t k,
                                         const double *l, int64_t ldl, double *out2, void *ws, size_t ws_bytes,
                                         void *stream_) {
  static const char *fn = "skt_gram_cross_csr";
  if (n < 0 || ncols < 0 || k < 0 || k > kGramMaxK || ldm < k || ldl < k || !out2 ||
      (indptr_type != SKT_I32 && indptr_type != SKT_I64) || (index_type != SKT_I32 && index_type != SKT_I64) ||
      (val_dtype != SKT_F32 && val_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (!ws || ws_bytes < (size_t)kLsqBlocks * 2 * sizeof(double)) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  if (n > 0 && (!a_indptr || (k > 0 && (!mw || !l)))) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
  double *part = (double *)ws;
  if (n == 0) return cudaMemsetAsync(out2, 0, 2 * sizeof(double), st) == cudaSuccess ? SKT_OK : fail(SKT_ECUDA, fn, "memset");
#define SKT_GRAM(IP, IX)                                                                                        \
  (val_dtype == SKT_F32 ? launch_gram_csr<IP, IX, float>(n, a_indptr, a_indices, a_vals, mw, ldm, (int)k, l, ldl, out2, part, st) \
                        : launch_gram_csr<IP, IX, double>(n, a_indptr, a_indices, a_vals, mw, ldm, (int)k, l, ldl, out2, part, st))
  if (indptr_type == SKT_I32) return index_type == SKT_I32 ? SKT_GRAM(int32_t, int32_t) : SKT_GRAM(int32_t, int64_t);
  return index_type == SKT_I32 ? SKT_GRAM(int64_t, int32_t) : SKT_GRAM(int64_t, int64_t);
#undef SKT_GRAM
}

extern "C" skt_status skt_gram_cross_dense(int64_t n, int64_t ncols, const void *a, skt_dtype a_dtype, int64_t lda,
                                           const double *mw, int64_t ldm, int64_t k, const double *l, int64_t ldl,
                                           double *out2, void *ws, size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_gram_cross_dense";
  if (n < 0 || ncols < 0 || k < 0 || k > kGramMaxK || lda < ncols || ldm < k || ldl < k || !out2 ||
      (a_dtype != SKT_F32 && a_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (!ws || ws_bytes < (size_t)kLsqBlocks * 2 * sizeof(double)) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  if (n > 0 && ((ncols > 0 && !a) || (k > 0 && (!mw || !l)))) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
  double *part = (double *)ws;
  if (n == 0) return cudaMemsetAsync(out2, 0, 2 * sizeof(double), st) == cudaSuccess ? SKT_OK : fail(SKT_ECUDA, fn, "memset");
  const int64_t blocks = lsq_blocks(n);
  if (a_dtype == SKT_F32)
    SKT_LAUNCH(gram_dense_kernel<float>, (unsigned)blocks, kLsqThreads, 0, st, n, ncols, (const float *)a, lda, mw,
               ldm, (int)k, l, ldl, part);
  else
    SKT_LAUNCH(gram_dense_kernel<double>, (unsigned)blocks, kLsqThreads, 0, st, n, ncols, (const double *)a, lda, mw,
               ldm, (int)k, l, ldl, part);
  SKT_LAUNCH(lsq_final_kernel, 1, kLsqThreads, 0, st, part, (int)blocks, 2, out2);
  return check_launch(fn);
}

extern "C" skt_status skt_gemm_dense(int64_t n, int64_t d, const void *a, skt_dtype a_dtype, int64_t lda,
                                     const double *x, int64_t k, double *y, int64_t ldy, void *stream_) {
  static const char *fn = "skt_gemm_dense";
  if (n < 0 || d < 0 || k < 0 || k > kGemmChunk || lda < d || ldy < k || (a_dtype != SKT_F32 && a_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (n == 0 || k == 0) return SKT_OK;
  if (!y || (d > 0 && (!a || !x))) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
  const int64_t blocks = (n * k + 255) / 256;
  if (a_dtype == SKT_F32)
    SKT_LAUNCH(gemm_dense_kernel<float>, (unsigned)blocks, 256, 0, st, n, d, (const float *)a, lda, x, k, y, ldy);
  else
    SKT_LAUNCH(gemm_dense_kernel<double>, (unsigned)blocks, 256, 0, st, n, d, (const double *)a, lda, x, k, y, ldy);
  return check_launch(fn);
}
