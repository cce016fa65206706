// dense_tma.cuh -- K3 bulk-copy variant: SA = S.A for dense row-major A whose
// rows are 16-byte multiples of 256 B .. 2 KB (BASELINE config 3: 512 B rows).
//
// One warp per bucket.  The bucket's rows (plan order = ascending row id) are
// fetched R at a time into a kStages-deep ring of shared-memory stages with the
// Blackwell bulk-copy engine (cp.async.bulk global->shared, one 1D copy per
// row, completion counted in bytes on an mbarrier per stage), so ~kStages*R
// rows per warp are in flight without holding registers.  The lanes consume a
// landed stage row by row: lane l owns the 16-byte column chunks l, l+32, ...
// of a row and keeps fp64 accumulators for them, adding s_i * A[i, cols] in
// ascending row order from +0.0 -- the reference's csr_matvecs order, so the
// fp64 result is bit-identical.  The non-finite scan of as_dense is fused.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

constexpr int kTmaWarps = 4;
constexpr int kTmaRows = 8;    // rows per stage
constexpr int kTmaStages = 4;  // stages per warp

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <typename T>
struct Chunk16;
template <>
struct Chunk16<float> {
  static constexpr int kElems = 4;
  __device__ static void add(const uint4 &u, bool neg, double *acc, bool &bad) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bad |= (w[k] & 0x7f800000u) == 0x7f800000u;
      const double x = (double)__uint_as_float(w[k]);
      acc[k] += neg ? -x : x;
    }
  }
};
template <>
struct Chunk16<double> {
  static constexpr int kElems = 2;
  __device__ static void add(const uint4 &u, bool neg, double *acc, bool &bad) {
    const uint32_t hi[2] = {u.y, u.w};
    const uint64_t w[2] = {((uint64_t)u.y << 32) | u.x, ((uint64_t)u.w << 32) | u.z};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      bad |= (hi[k] & 0x7ff00000u) == 0x7ff00000u;
      const double x = __longlong_as_double((long long)w[k]);
      acc[k] += neg ? -x : x;
    }
  }
};

// K = 16-byte chunks per lane per row (row_bytes <= K * 512)
template <typename TIn, typename TOut, int K>
__global__ void __launch_bounds__(kTmaWarps * 32) dense_tma_kernel(
    const int64_t *__restrict__ indptr, const uint32_t *__restrict__ rows, uint64_t t,
    const char *__restrict__ a, int row_bytes, int64_t lda_bytes, int d, TOut *__restrict__ sa,
    int64_t ldsa, int32_t *__restrict__ flag) {
  constexpr int E = Chunk16<TIn>::kElems;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[kTmaWarps][kTmaStages];
  __shared__ uint32_t signs[kTmaWarps][kTmaStages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t bucket = (int64_t)blockIdx.x * kTmaWarps + w;
  if (bucket >= (int64_t)t) return;
  unsigned char *ring = smem_raw + (size_t)w * kTmaStages * kTmaRows * row_bytes;
  if (lane == 0)
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[w][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();

  const int64_t beg = indptr[bucket], end = indptr[bucket + 1];
  const int64_t nchunks = (end - beg + kTmaRows - 1) / kTmaRows;
  auto issue = [&](int64_t c, int s) {
    const int64_t k = beg + c * kTmaRows + lane;
    const bool has = lane < kTmaRows && k < end;
    const uint32_t wrd = has ? __ldg(rows + k) : 0u;
    const uint32_t neg = __ballot_sync(0xffffffffu, has && (wrd >> 31));
    const int cnt = (int)min((int64_t)kTmaRows, end - beg - c * kTmaRows);
    if (lane == 0) {
      signs[w][s] = neg;
      mbar_arrive_tx(&bars[w][s], (uint32_t)(cnt * row_bytes));
    }
    __syncwarp();
    if (has)
      bulk_g2s(ring + ((size_t)s * kTmaRows + lane) * row_bytes,
               a + (int64_t)(wrd & 0x7fffffffu) * lda_bytes, (uint32_t)row_bytes, &bars[w][s]);
  };
  for (int s = 0; s < kTmaStages && s < nchunks; ++s) issue(s, s);

  double acc[K][E];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int e = 0; e < E; ++e) acc[k][e] = 0.0;
  bool bad = false;
  int s = 0;
  uint32_t phase = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    mbar_wait(&bars[w][s], phase);
    const int cnt = (int)min((int64_t)kTmaRows, end - beg - c * kTmaRows);
    const uint32_t neg = signs[w][s];
    const unsigned char *st = ring + (size_t)s * kTmaRows * row_bytes;
#pragma unroll
    for (int r = 0; r < kTmaRows; ++r) {
      if (r < cnt) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int off = (k * 32 + lane) * 16;
          if (off < row_bytes) {
            const uint4 u = *reinterpret_cast<const uint4 *>(st + r * row_bytes + off);
            Chunk16<TIn>::add(u, (neg >> r) & 1u, acc[k], bad);
          }
        }
      }
    }
    __syncwarp();  // every lane is done with stage s before it is refilled
    if (c + kTmaStages < nchunks) issue(c + kTmaStages, s);
    if (++s == kTmaStages) {
      s = 0;
      phase ^= 1u;
    }
  }
  TOut *o = sa + bucket * ldsa;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int col = (k * 32 + lane) * E;
    if (col < d) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (col + e < d) o[col + e] = (TOut)acc[k][e];
    }
  }
  if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

inline size_t dense_tma_smem(int row_bytes) {
  return (size_t)kTmaWarps * kTmaStages * kTmaRows * row_bytes;
}

}  // namespace
}  // namespace skt
