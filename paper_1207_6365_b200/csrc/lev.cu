// lev.cu -- K5: leverage-score contraction (reference leverage.py:87-91):
//   rows = A @ probe   (probe = N G^T, d x k)      scores_i = sum_c rows_ic^2
// fused: A is streamed once, the n x k product never touches HBM, only the n
// scores are written.
//
// This file holds the fp64 CUDA-core path (used for fp64 A, and as the
// exact-accumulation path for fp32 A): one warp per row, lane c owns probe
// column c (k > 32 loops over column chunks), the probe lives in shared memory
// as fp64, nonzeros are fetched 32 at a time and broadcast with shuffles, the
// next row's nonzeros are prefetched while the current row is contracted.
// Per (row, column) the products are accumulated in stored-nonzero order with
// fp64 FMA; the 32-lane square-sum uses a fixed butterfly (deterministic).
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "lev_tc.cuh"
#include "lev_tc2.cuh"
#include "lev_tc3.cuh"

namespace skt {
namespace {
// SKT_LEV_TC=0 keeps fp32 inputs on the fp64 CUDA-core path (A/B checks).
inline bool lev_tc_enabled() {
  static const bool on = [] {
    const char *e = getenv("SKT_LEV_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}
// SKT_LEV_TC3=0 keeps k % 32 == 0 shapes on the 3xTF32 kernel (lev_tc.cuh).
inline bool lev_tc3_enabled() {
  static const bool on = [] {
    const char *e = getenv("SKT_LEV_TC3");
    return !(e && e[0] == '0');
  }();
  return on;
}
// SKT_LEV_TC2=1 selects the staged, warp-specialised 2xFP16 kernel
// (lev_tc2.cuh; measured slower than lev_tc.cuh on config 4, kept for A/B).
inline bool lev_tc2_enabled() {
  static const bool on = [] {
    const char *e = getenv("SKT_LEV_TC2");
    return e && e[0] == '1';
  }();
  return on;
}
}  // namespace
}  // namespace skt

namespace skt {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr size_t kProbeSmemMax = 96 * 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <bool kSmemProbe>
__device__ __forceinline__ double probe_at(const double *sp, const double *gp, int64_t idx) {
  return kSmemProbe ? sp[idx] : __ldg(gp + idx);
}

template <typename IP, typename IX, typename TV, typename TS, bool kSmemProbe>
__global__ void __launch_bounds__(kThreads) lev_csr_kernel(
    int64_t n, int64_t d, const IP *__restrict__ aip, const IX *__restrict__ aix,
    const TV *__restrict__ av, const double *__restrict__ probe, int64_t k,
    TS *__restrict__ scores) {
  extern __shared__ __align__(16) double sprobe[];
  if (kSmemProbe) {
    for (int64_t i = threadIdx.x; i < d * k; i += blockDim.x) sprobe[i] = probe[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
  for (int64_t row = warp; row < n; row += nwarps) {
    const int64_t rs = (int64_t)aip[row], re = (int64_t)aip[row + 1];
    double score = 0.0;
    for (int64_t c0 = 0; c0 < k; c0 += 32) {
      const int64_t c = c0 + lane;
      const bool cl = c < k;
      double acc = 0.0;
      for (int64_t p0 = rs; p0 < re; p0 += 32) {
        const int64_t p = p0 + lane;
        const bool has = p < re;
        const int32_t j = has ? (int32_t)aix[p] : 0;
        const double v = has ? (double)av[p] : 0.0;
        const int cnt = (int)min((int64_t)32, re - p0);
        for (int q = 0; q < cnt; ++q) {
          const int32_t jq = __shfl_sync(0xffffffffu, j, q);
          const double vq = __shfl_sync(0xffffffffu, v, q);
          if (cl) acc = fma(vq, probe_at<kSmemProbe>(sprobe, probe, (int64_t)jq * k + c), acc);
        }
      }
      score += warp_sum(cl ? acc * acc : 0.0);
    }
    if (lane == 0) scores[row] = (TS)score;
  }
}

// k == 32, probe in shared memory: a HALF warp per row (LPR = 16), lane owns
// columns 2l', 2l'+1 (one 16-byte probe load per entry); the two rows of a
// warp share every shuffle, so the shared-memory pipe does about half the work
// per entry of the warp-per-row kernel (config 4 shape, fp64: 2.0 -> 1.33 ms).
// Per score the order of the fp64 FMAs over a row's entries is the same
// (ascending entries), per column.
template <typename IP, typename IX, typename TV, typename TS, int LPR>
__global__ void __launch_bounds__(kThreads) lev_csr_k32_kernel(int64_t n, int64_t d, const IP *__restrict__ aip,
                                                               const IX *__restrict__ aix, const TV *__restrict__ av,
                                                               const double *__restrict__ probe,
                                                               TS *__restrict__ scores) {
  // LPR lanes per row (16 or 8), CPL = 32 / LPR columns per lane, 32 / LPR
  // rows per warp sharing every shuffle
  constexpr int CPL = 32 / LPR, RPW = 32 / LPR, V2 = CPL / 2;
  extern __shared__ __align__(16) double sprobe[];
  for (int64_t i = threadIdx.x; i < d * 32; i += blockDim.x) sprobe[i] = probe[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane / LPR, hl = lane % LPR;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
  const double2 *sp2 = reinterpret_cast<const double2 *>(sprobe);
  for (int64_t r0 = RPW * warp; r0 < n; r0 += RPW * nwarps) {
    const int64_t row = r0 + sub;
    const bool live = row < n;
    const int64_t rs = live ? (int64_t)aip[row] : 0, re = live ? (int64_t)aip[row + 1] : 0;
    const int len = (int)(re - rs);
    int lmax = len;
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    double a[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) a[c] = 0.0;
    for (int p0 = 0; p0 < lmax; p0 += LPR) {
      const int p = p0 + hl;
      const bool has = p < len;
      const int32_t j = has ? (int32_t)aix[rs + p] : 0;
      const double v = has ? (double)av[rs + p] : 0.0;
      const int cnt = min(LPR, lmax - p0);
      for (int q = 0; q < cnt; ++q) {
        const int32_t jq = __shfl_sync(0xffffffffu, j, q, LPR);
        const double vq = __shfl_sync(0xffffffffu, v, q, LPR);
        if (p0 + q < len) {  // this row still has entry p0 + q
#pragma unroll
          for (int h = 0; h < V2; ++h) {
            const double2 pr = sp2[(int64_t)jq * 16 + hl * V2 + h];
            a[2 * h] = fma(vq, pr.x, a[2 * h]);
            a[2 * h + 1] = fma(vq, pr.y, a[2 * h + 1]);
          }
        }
      }
    }
    double sc = 0.0;
#pragma unroll
    for (int c = 0; c < CPL; ++c) sc = fma(a[c], a[c], sc);
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
    if (live && hl == 0) scores[row] = (TS)sc;
  }
}

template <typename TA, typename TS, bool kSmemProbe>
__global__ void __launch_bounds__(kThreads) lev_dense_kernel(int64_t n, int64_t d,
                                                             const TA *__restrict__ a, int64_t lda,
                                                             const double *__restrict__ probe,
                                                             int64_t k, TS *__restrict__ scores,
                                                             int32_t *__restrict__ flag) {
  extern __shared__ __align__(16) double sprobe[];
  if (kSmemProbe) {
    for (int64_t i = threadIdx.x; i < d * k; i += blockDim.x) sprobe[i] = probe[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
  bool bad = false;
  for (int64_t row = warp; row < n; row += nwarps) {
    const TA *ar = a + row * lda;
    double score = 0.0;
    for (int64_t c0 = 0; c0 < k; c0 += 32) {
      const int64_t c = c0 + lane;
      const bool cl = c < k;
      double acc = 0.0;
      for (int64_t j0 = 0; j0 < d; j0 += 32) {
        const bool has = j0 + lane < d;
        const double v = has ? (double)ar[j0 + lane] : 0.0;
        if (c0 == 0) bad |= !isfinite(v);
        const int cnt = (int)min((int64_t)32, d - j0);
        for (int q = 0; q < cnt; ++q) {
          const double vq = __shfl_sync(0xffffffffu, v, q);
          if (cl) acc = fma(vq, probe_at<kSmemProbe>(sprobe, probe, (j0 + q) * k + c), acc);
        }
      }
      score += warp_sum(cl ? acc * acc : 0.0);
    }
    if (lane == 0) scores[row] = (TS)score;
  }
  if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

inline int64_t grid_for(int64_t n) {
  const int64_t want = (n + kWarps - 1) / kWarps;
  return std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)kNumSMs * 8));
}

template <typename IP, typename IX, typename TV, typename TS>
skt_status launch_csr(int64_t n, int64_t d, const void *aip, const void *aix, const void *av,
                      const double *p, int64_t k, void *scores, cudaStream_t st) {
  static const char *fn = "skt_lev_rownorms_csr";
  // fp32 values on the tensor cores when the shape fits: the staged scaled
  // 2xFP16 kernel (lev_tc2.cuh, d <= 128, 16-byte aligned arrays), else the
  // register-staged 3xTF32 kernel (lev_tc.cuh)
  if (std::is_same<TV, float>::value && lev_tc_enabled() && d <= 256 && k >= 8 && k <= 256 && k % 8 == 0) {
    const T2Layout L = lev_tc2_layout((int)d, (int)k, (int)sizeof(IX));
    const bool aligned = ((uintptr_t)aip % 16 == 0) && ((uintptr_t)aix % 16 == 0) && ((uintptr_t)av % 16 == 0);
    if (lev_tc2_enabled() && L.nst > 0 && aligned) {
      auto kern = lev_tc2_kernel<IP, IX, TS>;
      SKT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem), fn);
      const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
      const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)kNumSMs);
      SKT_LAUNCH(kern, (unsigned)blocks, kT2Threads, L.smem, st, n, (int)d, (const IP *)aip,
                 (const IX *)aix, (const float *)av, p, (int)k, (TS *)scores, L);
      return check_launch(fn);
    }
    const int dk8 = (int)((d + 7) & ~7LL);  // K of the MMA chain
    const size_t smem3 = lev_tc3_smem(dk8, (int)k);
    if (lev_tc3_enabled() && tc3_ok((int)k) && smem3 <= 200 * 1024) {  // scaled 2xFP16 (lev_tc3.cuh)
      auto kern = lev_tc3_kernel<IP, IX, TS>;
      SKT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3), fn);
      const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
      const size_t by_tmem = 512 / tc3_cols((int)k);
      const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(std::min<size_t>(4, by_tmem), (220 * 1024) / smem3));
      const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)kNumSMs * per_sm);
      SKT_LAUNCH(kern, (unsigned)blocks, kTcThreads, smem3, st, n, (int)d, dk8, (const IP *)aip,
                 (const IX *)aix, (const float *)av, p, (int)k, (TS *)scores);
      return check_launch(fn);
    }
    const size_t smem = lev_tc_smem(dk8, (int)k);
    if (smem <= 200 * 1024) {
      auto kern = tc_merged((int)k) ? lev_tc_kernel<IP, IX, TS, true> : lev_tc_kernel<IP, IX, TS, false>;
      SKT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
      const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
      // resident CTAs per SM: bounded by shared memory and by the 512 TMEM
      // columns (a CTA's tcgen05.alloc would otherwise wait forever)
      const size_t by_tmem = 512 / lev_tc_cols((int)k);
      const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(std::min<size_t>(4, by_tmem), (220 * 1024) / smem));
      const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)kNumSMs * per_sm);
      SKT_LAUNCH(kern, (unsigned)blocks, kTcThreads, smem, st, n, (int)d, dk8, (const IP *)aip,
                 (const IX *)aix, (const float *)av, p, (int)k, (TS *)scores);
      return check_launch(fn);
    }
  }
  const size_t pbytes = (size_t)d * k * sizeof(double);
  const int64_t blocks = grid_for(n);
  static const bool k32 = [] {
    const char *e = getenv("SKT_LEV_K32");
    return !(e && e[0] == '0');
  }();
  if (k == 32 && k32 && pbytes <= kProbeSmemMax) {
    static const int lpr = [] {  // lanes per row: 16 (default) or 8 (A/B; measured 8% slower)
      const char *e = getenv("SKT_LEV_K32_LPR");
      return e && atoi(e) == 8 ? 8 : 16;
    }();
    auto kern = lpr == 16 ? lev_csr_k32_kernel<IP, IX, TV, TS, 16> : lev_csr_k32_kernel<IP, IX, TV, TS, 8>;
    SKT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pbytes), fn);
    SKT_LAUNCH(kern, (unsigned)blocks, kThreads, pbytes, st, n, d, (const IP *)aip, (const IX *)aix, (const TV *)av, p,
               (TS *)scores);
    return check_launch(fn);
  }
  if (pbytes <= kProbeSmemMax) {
    auto kern = lev_csr_kernel<IP, IX, TV, TS, true>;
    SKT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pbytes), fn);
    SKT_LAUNCH(kern, (unsigned)blocks, kThreads, pbytes, st, n, d, (const IP *)aip, (const IX *)aix,
               (const TV *)av, p, k, (TS *)scores);
  } else {
    SKT_LAUNCH((lev_csr_kernel<IP, IX, TV, TS, false>), (unsigned)blocks, kThreads, 0, st, n, d,
               (const IP *)aip, (const IX *)aix, (const TV *)av, p, k, (TS *)scores);
  }
  return check_launch(fn);
}

template <typename IP, typename IX>
skt_status csr_types(int64_t n, int64_t d, const void *aip, const void *aix, const void *av,
                     skt_dtype vt, const double *p, int64_t k, void *scores, skt_dtype st_,
                     cudaStream_t st) {
  if (vt == SKT_F32)
    return st_ == SKT_F64 ? launch_csr<IP, IX, float, double>(n, d, aip, aix, av, p, k, scores, st)
                          : launch_csr<IP, IX, float, float>(n, d, aip, aix, av, p, k, scores, st);
  return st_ == SKT_F64 ? launch_csr<IP, IX, double, double>(n, d, aip, aix, av, p, k, scores, st)
                        : launch_csr<IP, IX, double, float>(n, d, aip, aix, av, p, k, scores, st);
}

template <typename TA, typename TS>
skt_status launch_dense(int64_t n, int64_t d, const void *a, int64_t lda, const double *p,
                        int64_t k, void *scores, int32_t *flag, cudaStream_t st) {
  static const char *fn = "skt_lev_rownorms_dense";
  const size_t pbytes = (size_t)d * k * sizeof(double);
  const int64_t blocks = grid_for(n);
  if (pbytes <= kProbeSmemMax) {
    auto kern = lev_dense_kernel<TA, TS, true>;
    SKT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pbytes), fn);
    SKT_LAUNCH(kern, (unsigned)blocks, kThreads, pbytes, st, n, d, (const TA *)a, lda, p, k,
               (TS *)scores, flag);
  } else {
    SKT_LAUNCH((lev_dense_kernel<TA, TS, false>), (unsigned)blocks, kThreads, 0, st, n, d,
               (const TA *)a, lda, p, k, (TS *)scores, flag);
  }
  return check_launch(fn);
}

}  // namespace
}  // namespace skt

namespace skt {
skt_status lev_dmma_csr(int64_t n, int64_t d, const void *aip, skt_itype ipt, const void *aix, skt_itype ixt,
                        const void *av, skt_dtype vt, const double *p, int64_t k, void *scores, skt_dtype sdt,
                        cudaStream_t st);
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_lev_rownorms_csr(int64_t n, int64_t d, const void *a_indptr,
                                           skt_itype indptr_type, const void *a_indices,
                                           skt_itype index_type, const void *a_vals,
                                           skt_dtype val_dtype, const double *probe, int64_t k,
                                           void *scores, skt_dtype score_dtype, void *stream_) {
  static const char *fn = "skt_lev_rownorms_csr";
  if (n < 0 || d < 0 || k < 0 || !a_indptr || (indptr_type != SKT_I32 && indptr_type != SKT_I64) ||
      (index_type != SKT_I32 && index_type != SKT_I64) ||
      (val_dtype != SKT_F32 && val_dtype != SKT_F64) ||
      (score_dtype != SKT_F32 && score_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (n == 0) return SKT_OK;
  if (!scores || (k > 0 && d > 0 && !probe)) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t st = as_stream(stream_);
  // fp64 values (the reference API's dtype): the fp64 tensor-core kernel (lev_dmma.cuh)
  const skt_status dm = lev_dmma_csr(n, d, a_indptr, indptr_type, a_indices, index_type, a_vals, val_dtype, probe, k,
                                     scores, score_dtype, st);
  if (dm != SKT_ENOTSUP) return dm;
  if (indptr_type == SKT_I32)
    return index_type == SKT_I32
               ? csr_types<int32_t, int32_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, probe, k, scores, score_dtype, st)
               : csr_types<int32_t, int64_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, probe, k, scores, score_dtype, st);
  return index_type == SKT_I32
             ? csr_types<int64_t, int32_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, probe, k, scores, score_dtype, st)
             : csr_types<int64_t, int64_t>(n, d, a_indptr, a_indices, a_vals, val_dtype, probe, k, scores, score_dtype, st);
}

extern "C" skt_status skt_lev_rownorms_dense(int64_t n, int64_t d, const void *a, skt_dtype a_dtype,
                                             int64_t lda, const double *probe, int64_t k,
                                             void *scores, skt_dtype score_dtype,
                                             int32_t *nonfinite_flag, void *stream_) {
  static const char *fn = "skt_lev_rownorms_dense";
  if (n < 0 || d < 0 || k < 0 || lda < d || (a_dtype != SKT_F32 && a_dtype != SKT_F64) ||
      (score_dtype != SKT_F32 && score_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  cudaStream_t st = as_stream(stream_);
  if (nonfinite_flag) SKT_CUDA_TRY(cudaMemsetAsync(nonfinite_flag, 0, sizeof(int32_t), st), fn);
  if (n == 0) return SKT_OK;
  if (!scores || (d > 0 && !a) || (k > 0 && d > 0 && !probe)) return fail(SKT_EINVAL, fn, "NULL buffer");
  if (a_dtype == SKT_F32)
    return score_dtype == SKT_F64 ? launch_dense<float, double>(n, d, a, lda, probe, k, scores, nonfinite_flag, st)
                                  : launch_dense<float, float>(n, d, a, lda, probe, k, scores, nonfinite_flag, st);
  return score_dtype == SKT_F64 ? launch_dense<double, double>(n, d, a, lda, probe, k, scores, nonfinite_flag, st)
                                : launch_dense<double, float>(n, d, a, lda, probe, k, scores, nonfinite_flag, st);
}
