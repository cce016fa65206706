// apply_dense.cu -- K3: SA = S.A for dense row-major A (reference sketch.py:165,
// scipy csr_matvecs over the t x n plan, after as_dense's finiteness scan
// _validation.py:16-27).
//
// Work item = (bucket b, column chunk).  A group of G lanes (G | 32) owns one
// work item; lane g of the group owns VEC consecutive columns and keeps VEC
// fp64 accumulators in registers.  The group walks the bucket's rows in plan
// order (ascending row id) and adds s_i * A[i, cols] sequentially from +0.0,
// i.e. exactly the reference's per-element accumulation order, so the fp64
// result is bit-identical.  Rows are gathered with 128-bit non-allocating
// loads, kUnroll rows in flight per lane before the ordered accumulation.
// The non-finite check of as_dense is fused (exponent-all-ones test).
#include <cstdlib>

#include "common.cuh"
#include "dense_g4.cuh"
#include "dense_tma.cuh"

namespace skt {
namespace {

constexpr int kThreads = 256;
// Tuned on config 3 (tools/dense_ceiling.py, A/B builds on one box): one
// batch of 4 rows in flight per warp (plan words one batch ahead), 60
// registers, >= 4 resident blocks (32 warps) per SM -- 2% faster than the
// software-pipelined gather (SKT_DENSE_PIPE=1: batch k+1 in flight while batch
// k is accumulated, 80 registers, 24 warps per SM): more warps beat a deeper
// per-warp pipeline, as in the CSR tile kernel.
#ifndef SKT_DENSE_PIPE
#define SKT_DENSE_PIPE 0
#endif
#ifndef SKT_DENSE_MINB
#define SKT_DENSE_MINB 4
#endif

template <typename T, int VEC>
struct Vec;
template <>
struct Vec<float, 4> {
  using type = float4;
};
template <>
struct Vec<float, 2> {
  using type = float2;
};
template <>
struct Vec<float, 1> {
  using type = float;
};
template <>
struct Vec<double, 2> {
  using type = double2;
};
template <>
struct Vec<double, 1> {
  using type = double;
};

__device__ __forceinline__ float4 ldstream(const float4 *p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ldstream(const float2 *p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float ldstream(const float *p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ldstream(const double2 *p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double ldstream(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ bool nonfinite(float x) {
  return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}
__device__ __forceinline__ bool nonfinite(double x) {
  return ((uint32_t)(__double_as_longlong(x) >> 32) & 0x7ff00000u) == 0x7ff00000u;
}

template <typename TIn, typename TOut, int VEC, int G, int kUnroll>
__global__ void __launch_bounds__(kThreads, SKT_DENSE_MINB) apply_dense_kernel(
    const int64_t *__restrict__ indptr, const uint32_t *__restrict__ rows, int64_t n_items,
    int64_t n_chunks, const TIn *__restrict__ a, int64_t d, int64_t lda, TOut *__restrict__ sa,
    int64_t ldsa, int32_t *__restrict__ flag) {
  using V = typename Vec<TIn, VEC>::type;
  constexpr int kGroups = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, glane = lane % G;
  // persistent warps: grid-stride over work items (no per-block launch /
  // start-up bubbles between buckets)
  const int64_t warp0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
  bool bad = false;
  for (int64_t warp = warp0; warp * kGroups < n_items; warp += nwarps) {
  const int64_t item = warp * kGroups + grp;
  const bool live = item < n_items;
  const int64_t bucket = live ? item / n_chunks : 0;
  const int64_t chunk = live ? item % n_chunks : 0;
  const int64_t col = chunk * (int64_t)(G * VEC) + (int64_t)glane * VEC;
  const bool active = live && col < d;

  double acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) acc[k] = 0.0;

  const int64_t beg = live ? indptr[bucket] : 0;
  const int64_t end = live ? indptr[bucket + 1] : 0;
  const TIn *acol = a + col;
#if SKT_DENSE_PIPE
  // software pipeline: the rows of batch k+1 are in flight while batch k is
  // accumulated; plan words run one further batch ahead.
  auto words = [&](int64_t k0, uint32_t(&w)[kUnroll]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) w[u] = (k0 + u < end) ? __ldg(rows + k0 + u) : 0u;
  };
  auto gather = [&](int64_t k0, const uint32_t(&w)[kUnroll], V(&v)[kUnroll]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      v[u] = (active && k0 + u < end)
                 ? ldstream(reinterpret_cast<const V *>(acol + (int64_t)(w[u] & 0x7fffffffu) * lda))
                 : V{};
  };
  uint32_t wa[kUnroll], wb[kUnroll];
  V va[kUnroll];
  words(beg, wa);
  gather(beg, wa, va);
  words(beg + kUnroll, wb);
  for (int64_t k0 = beg; k0 < end; k0 += kUnroll) {
    V vb[kUnroll];
    uint32_t wc[kUnroll];
    gather(k0 + kUnroll, wb, vb);
    words(k0 + 2 * kUnroll, wc);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (k0 + u < end) {
        const bool neg = (wa[u] >> 31) != 0;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          const TIn x = reinterpret_cast<const TIn *>(&va[u])[k];
          bad |= nonfinite(x);
          const double xd = (double)x;
          acc[k] += neg ? -xd : xd;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      wa[u] = wb[u];
      va[u] = vb[u];
      wb[u] = wc[u];
    }
  }
#else
  // plan words of the next kUnroll rows are loaded one iteration ahead, so
  // each iteration waits for one DRAM round trip (the row gather) only
  uint32_t wn[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) wn[u] = (beg + u < end) ? __ldg(rows + beg + u) : 0u;
  for (int64_t k0 = beg; k0 < end; k0 += kUnroll) {
    uint32_t w[kUnroll];
    V v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) w[u] = wn[u];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (active && k0 + u < end)
        v[u] = ldstream(reinterpret_cast<const V *>(acol + (int64_t)(w[u] & 0x7fffffffu) * lda));
      else
        v[u] = V{};
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t k = k0 + kUnroll + u;
      wn[u] = (k < end) ? __ldg(rows + k) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (k0 + u < end) {
        const bool neg = (w[u] >> 31) != 0;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          const TIn x = reinterpret_cast<const TIn *>(&v[u])[k];
          bad |= nonfinite(x);
          const double xd = (double)x;
          acc[k] += neg ? -xd : xd;
        }
      }
    }
  }
#endif
  if (active) {
    TOut *o = sa + bucket * ldsa + col;
    if (col + VEC <= d) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) o[k] = (TOut)acc[k];
    } else {
      for (int k = 0; k < VEC && col + k < d; ++k) o[k] = (TOut)acc[k];
    }
  }
  }  // persistent loop
  if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

template <typename TIn, typename TOut, int VEC, int G>
skt_status launch(const int64_t *indptr, const uint32_t *rows, uint64_t t, const TIn *a,
                  int64_t d, int64_t lda, TOut *sa, int64_t ldsa, int32_t *flag,
                  cudaStream_t stream) {
  const int64_t n_chunks = (d + G * VEC - 1) / (G * VEC);
  const int64_t n_items = (int64_t)t * n_chunks;
  const int64_t warps = (n_items + (32 / G) - 1) / (32 / G);
#ifndef SKT_DENSE_BLOCKS_PER_SM
#define SKT_DENSE_BLOCKS_PER_SM 0  // persistent grids measured slower on config 3
#endif
  // persistent grid: SKT_DENSE_BLOCKS_PER_SM resident blocks per SM (0 = one block per 8 items)
  const int64_t need = (warps * 32 + kThreads - 1) / kThreads;
  const int64_t blocks = SKT_DENSE_BLOCKS_PER_SM > 0
                             ? std::min<int64_t>(need, (int64_t)kNumSMs * SKT_DENSE_BLOCKS_PER_SM)
                             : need;
#ifndef SKT_DENSE_UNROLL8
#define SKT_DENSE_UNROLL8 8
#endif
  constexpr int kUnroll = (sizeof(TIn) * VEC >= 16) ? 4 : SKT_DENSE_UNROLL8;
  SKT_LAUNCH((apply_dense_kernel<TIn, TOut, VEC, G, kUnroll>), (unsigned)blocks, kThreads, 0, stream,
             indptr, rows, n_items, n_chunks, a, d, lda, sa, ldsa, flag);
  return check_launch("skt_apply_dense");
}

template <typename TIn, typename TOut, int VEC>
skt_status dispatch_g(const int64_t *indptr, const uint32_t *rows, uint64_t t, const TIn *a,
                      int64_t d, int64_t lda, TOut *sa, int64_t ldsa, int32_t *flag,
                      cudaStream_t stream) {
  const int64_t lanes = (d + VEC - 1) / VEC;
  if (lanes <= 1) return launch<TIn, TOut, VEC, 1>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
  if (lanes <= 2) return launch<TIn, TOut, VEC, 2>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
  if (lanes <= 4) return launch<TIn, TOut, VEC, 4>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
  if (lanes <= 8) return launch<TIn, TOut, VEC, 8>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
  if (lanes <= 16) return launch<TIn, TOut, VEC, 16>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
  return launch<TIn, TOut, VEC, 32>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
}

// SKT_DENSE_G4=0 disables the TMA gather4 kernel (A/B measurement).
inline bool g4_enabled() {
  static const bool on = [] {
    const char *e = getenv("SKT_DENSE_G4");
    return !(e && e[0] == '0');
  }();
  return on;
}

// SKT_DENSE_TMA=0 selects the register-gather kernel (A/B measurement).
inline bool tma_enabled() {
  static const bool on = [] {
    const char *e = getenv("SKT_DENSE_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename TIn, typename TOut>
skt_status dispatch_vec(const int64_t *indptr, const uint32_t *rows, uint64_t t, const void *a_,
                        int64_t d, int64_t lda, void *sa_, int64_t ldsa, int32_t *flag,
                        cudaStream_t stream, int64_t n_rows_hint) {
  const TIn *a = (const TIn *)a_;
  TOut *sa = (TOut *)sa_;
  const uintptr_t ap = (uintptr_t)a;
  auto ok = [&](int vec) {
    return d % vec == 0 && lda % vec == 0 && ap % (sizeof(TIn) * vec) == 0;
  };
  // bulk-copy (TMA 1D) gather for rows of 1-2 KB (16-byte multiples).  Shorter
  // rows stay on the register gather: a 1D bulk copy costs ~46 SM cycles of TMA
  // issue, which caps 512 B rows at ~3.8 TB/s (measured, profiles/).
  const int64_t row_bytes = d * (int64_t)sizeof(TIn), lda_bytes = lda * (int64_t)sizeof(TIn);
  // TMA gather4 (four random rows per TMA instruction): rows of 512 B .. 2 KB
  // (16-byte multiples; one box of <= 256 elements or two equal boxes), row
  // stride a 16-byte multiple.  Measured (tools/dense_rowsize.py, 8.6 GB
  // inputs): 512 B rows 1.24 ms vs 1.41 ms for the register gather, 1 KB 1.24
  // vs 5.5 ms (1D bulk copies); 256 B rows break even and 128 B rows are
  // faster on the register gather.
  const int nbox = g4_boxes(d, (int64_t)sizeof(TIn));
  if (g4_enabled() && nbox > 0 && lda_bytes % 16 == 0 && ap % 16 == 0 && n_rows_hint > 0 &&
      n_rows_hint < (1LL << 31)) {
    CUtensorMap map;
    if (make_row_map(&map, a, sizeof(TIn) == 8, n_rows_hint, d, lda_bytes, d / nbox)) {
      const size_t smem = dense_g4_smem((int)row_bytes);
      const int64_t blocks = ((int64_t)t + kG4Warps - 1) / kG4Warps;
      auto k = row_bytes == 512    ? dense_g4_kernel<TIn, TOut, 1, true>
               : row_bytes == 1024 ? dense_g4_kernel<TIn, TOut, 2, true>
               : row_bytes == 2048 ? dense_g4_kernel<TIn, TOut, 4, true>
               : row_bytes < 1024  ? dense_g4_kernel<TIn, TOut, 2, false>
                                   : dense_g4_kernel<TIn, TOut, 4, false>;
      SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "skt_apply_dense");
      SKT_LAUNCH(k, (unsigned)blocks, kG4Warps * 32, smem, stream, map, indptr, rows, t, (int)row_bytes, (int)d, sa,
                 ldsa, flag, (const unsigned char *)a, lda_bytes, 0.0, nbox, PushTable{});
      return check_launch("skt_apply_dense");
    }
  }
  if (tma_enabled() && row_bytes % 16 == 0 && lda_bytes % 16 == 0 && ap % 16 == 0 && row_bytes >= 1024 &&
      row_bytes <= 2048 && dense_tma_smem((int)row_bytes) <= 200 * 1024) {  // (its ring outgrows smem above 1.6 KB)
    const int kchunks = (int)((row_bytes + 511) / 512);
    const size_t smem = dense_tma_smem((int)row_bytes);
    const int64_t blocks = ((int64_t)t + kTmaWarps - 1) / kTmaWarps;
    auto k = kchunks <= 1 ? dense_tma_kernel<TIn, TOut, 1>
                          : kchunks <= 2 ? dense_tma_kernel<TIn, TOut, 2> : dense_tma_kernel<TIn, TOut, 4>;
    SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "skt_apply_dense");
    SKT_LAUNCH(k, (unsigned)blocks, kTmaWarps * 32, smem, stream, indptr, rows, t, (const char *)a,
               (int)row_bytes, lda_bytes, (int)d, sa, ldsa, flag);
    return check_launch("skt_apply_dense");
  }
#ifndef SKT_DENSE_MAXVEC
#define SKT_DENSE_MAXVEC 4
#endif
  if (SKT_DENSE_MAXVEC >= 4 && sizeof(TIn) == 4 && ok(4))
    return dispatch_g<TIn, TOut, (sizeof(TIn) == 4 ? 4 : 2)>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
  if (ok(2)) return dispatch_g<TIn, TOut, 2>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
  return dispatch_g<TIn, TOut, 1>(indptr, rows, t, a, d, lda, sa, ldsa, flag, stream);
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_apply_dense(const int64_t *indptr, const uint32_t *rows, uint64_t t,
                                      int64_t n, const void *a, skt_dtype a_dtype, int64_t d,
                                      int64_t lda, void *sa, skt_dtype sa_dtype, int64_t ldsa,
                                      int32_t *nonfinite_flag, void *stream_) {
  static const char *fn = "skt_apply_dense";
  if (!indptr || t < 1 || t > (1ull << 32) || n < 0 || d < 0 || lda < d || ldsa < d ||
      (a_dtype != SKT_F32 && a_dtype != SKT_F64) || (sa_dtype != SKT_F32 && sa_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  cudaStream_t stream = as_stream(stream_);
  if (nonfinite_flag) SKT_CUDA_TRY(cudaMemsetAsync(nonfinite_flag, 0, sizeof(int32_t), stream), fn);
  if (d == 0) return SKT_OK;
  if (!sa || (n > 0 && (!a || !rows))) return fail(SKT_EINVAL, fn, "NULL buffer");
  if (a_dtype == SKT_F32)
    return sa_dtype == SKT_F64
               ? dispatch_vec<float, double>(indptr, rows, t, a, d, lda, sa, ldsa, nonfinite_flag, stream, n)
               : dispatch_vec<float, float>(indptr, rows, t, a, d, lda, sa, ldsa, nonfinite_flag, stream, n);
  return sa_dtype == SKT_F64
             ? dispatch_vec<double, double>(indptr, rows, t, a, d, lda, sa, ldsa, nonfinite_flag, stream, n)
             : dispatch_vec<double, float>(indptr, rows, t, a, d, lda, sa, ldsa, nonfinite_flag, stream, n);
}

// ---- fused exchange (row-sharded multi-GPU): K3 that pushes partial rows to
// their owner ranks' receive buffers, and the owner's fixed-order slot sum
namespace skt {
namespace {
template <typename TIn, typename TOut>
skt_status launch_push(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n, const void *a_,
                       int64_t d, int64_t lda, const PushTable &pt, int32_t *flag, cudaStream_t stream) {
  static const char *fn = "skt_apply_dense_push";
  const TIn *a = (const TIn *)a_;
  const int64_t row_bytes = d * (int64_t)sizeof(TIn), lda_bytes = lda * (int64_t)sizeof(TIn);
  const int nbox = g4_boxes(d, (int64_t)sizeof(TIn));
  CUtensorMap map;
  if (nbox == 0 || lda_bytes % 16 != 0 || (uintptr_t)a % 16 != 0 || n < 1 || n >= (1LL << 31) ||
      !make_row_map(&map, a, sizeof(TIn) == 8, n, d, lda_bytes, d / nbox))
    return fail(SKT_ENOTSUP, fn, "fused push needs rows the gather4 kernel takes (512 B .. 2 KB, 16-byte aligned)");
  const size_t smem = dense_g4_smem((int)row_bytes);
  const int64_t blocks = ((int64_t)t + kG4Warps - 1) / kG4Warps;
  auto k = row_bytes == 512    ? dense_g4_kernel<TIn, TOut, 1, true, false, true>
           : row_bytes == 1024 ? dense_g4_kernel<TIn, TOut, 2, true, false, true>
           : row_bytes == 2048 ? dense_g4_kernel<TIn, TOut, 4, true, false, true>
           : row_bytes < 1024  ? dense_g4_kernel<TIn, TOut, 2, false, false, true>
                               : dense_g4_kernel<TIn, TOut, 4, false, false, true>;
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
  SKT_LAUNCH(k, (unsigned)blocks, kG4Warps * 32, smem, stream, map, indptr, rows, t, (int)row_bytes, (int)d,
             (TOut *)nullptr, (int64_t)0, flag, (const unsigned char *)a, lda_bytes, 0.0, nbox, pt);
  return check_launch(fn);
}
}  // namespace
}  // namespace skt

extern "C" skt_status skt_apply_dense_push(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                                           const void *a, skt_dtype a_dtype, int64_t d, int64_t lda,
                                           skt_dtype out_dtype, void *const *peers, const int64_t *bounds,
                                           int32_t nranks, int32_t me, int64_t cap, int64_t ldr, int64_t b0,
                                           int32_t *nonfinite_flag, void *stream_) {
  static const char *fn = "skt_apply_dense_push";
  if (!indptr || t < 1 || n < 0 || d < 1 || lda < d || !peers || !bounds || nranks < 1 ||
      nranks > kPushMaxRanks || me < 0 || me >= nranks || cap < 1 || ldr < d || b0 < 0 ||
      (a_dtype != SKT_F32 && a_dtype != SKT_F64) || (out_dtype != SKT_F32 && out_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  PushTable pt{};
  for (int g = 0; g < nranks; ++g) {
    if (!peers[g] || bounds[g + 1] < bounds[g] || bounds[g + 1] - bounds[g] > cap)
      return fail(SKT_EINVAL, fn, "bad peer table");
    pt.peer[g] = peers[g];
  }
  for (int g = 0; g <= nranks; ++g) pt.bounds[g] = bounds[g];
  if (b0 + (int64_t)t > bounds[nranks]) return fail(SKT_EINVAL, fn, "buckets beyond the owner ranges");
  pt.cap = cap;
  pt.ldr = ldr;
  pt.nranks = nranks;
  pt.me = me;
  pt.b0 = b0;
  cudaStream_t stream = as_stream(stream_);
  if (nonfinite_flag) SKT_CUDA_TRY(cudaMemsetAsync(nonfinite_flag, 0, sizeof(int32_t), stream), fn);
  if (n > 0 && (!a || !rows)) return fail(SKT_EINVAL, fn, "NULL buffer");
  if (a_dtype == SKT_F32)
    return out_dtype == SKT_F64 ? launch_push<float, double>(indptr, rows, t, n, a, d, lda, pt, nonfinite_flag, stream)
                                : launch_push<float, float>(indptr, rows, t, n, a, d, lda, pt, nonfinite_flag, stream);
  return out_dtype == SKT_F64 ? launch_push<double, double>(indptr, rows, t, n, a, d, lda, pt, nonfinite_flag, stream)
                              : launch_push<double, float>(indptr, rows, t, n, a, d, lda, pt, nonfinite_flag, stream);
}

extern "C" skt_status skt_slot_sum(const void *recv, skt_dtype dtype, int32_t nslots, int64_t rows, int64_t d,
                                   int64_t slot_stride, int64_t ldr, void *out, int64_t ldo, void *stream_) {
  static const char *fn = "skt_slot_sum";
  if (!recv || !out || nslots < 1 || rows < 0 || d < 0 || ldr < d || ldo < d || slot_stride < rows * ldr ||
      (dtype != SKT_F32 && dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (rows == 0 || d == 0) return SKT_OK;
  const int64_t total = rows * d;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)kNumSMs * 16));
  cudaStream_t st = as_stream(stream_);
  if (dtype == SKT_F32)
    SKT_LAUNCH(slot_sum_kernel<float>, (unsigned)blocks, 256, 0, st, (const float *)recv, nslots, rows, d,
               slot_stride, ldr, (float *)out, ldo);
  else
    SKT_LAUNCH(slot_sum_kernel<double>, (unsigned)blocks, 256, 0, st, (const double *)recv, nslots, rows, d,
               slot_stride, ldr, (double *)out, ldo);
  return check_launch(fn);
}
