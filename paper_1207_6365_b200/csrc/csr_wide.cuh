// csr_wide.cuh -- K4 for CSR A too wide for on-chip bucket accumulators
// (BASELINE config 5: d = 262,144, m = 400 -> a 2 MB fp64 SA row per bucket).
//
// csr_rowseq_kernel (deterministic, bit-identical): one warp per bucket walks
// the bucket's rows in plan (ascending row) order and accumulates directly into
// the bucket's SA row in global memory (zeroed first).  Inside a canonical row
// the columns are distinct, so the row's read-modify-writes never collide;
// successive rows are ordered by __syncwarp (+ the same-address coherence of a
// single warp's accesses), so per SA element the additions run in ascending row
// order -- the reference's bincount order.  Latency-bound (one warp per bucket).
//
// csr_atomic_kernel (fast mode, flag SKT_CSR_FAST, NOT deterministic): warps
// take plan positions in order (all warps work on the same few buckets at a
// time, whose SA rows stay in L2) and add s_i * v with fire-and-forget global
// atomics (RED.ADD f32/f64).  The summation order per element is unspecified:
// results match the reference to rounding (fp64: ~1e-16 relative, fp32 SA:
// one fp32 rounding per addition -> ~1e-7 relative), not bit-for-bit.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

template <typename IP, typename IX, typename TV, typename TOut>
__global__ void __launch_bounds__(256) csr_atomic_kernel(const int64_t *__restrict__ pindptr,
                                                         const uint32_t *__restrict__ prow,
                                                         uint64_t t, int64_t n,
                                                         const IP *__restrict__ aip,
                                                         const IX *__restrict__ aix,
                                                         const TV *__restrict__ av,
                                                         TOut *__restrict__ sa, int64_t ldsa) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // plan positions of buckets [0, t) of the (possibly offset) indptr: a
  // bucket range [b0, b1) of the operator is indptr + b0, t = b1 - b0
  const int64_t k_end = __ldg(pindptr + t);
  (void)n;
  for (int64_t k = __ldg(pindptr) + warp; k < k_end; k += nwarps) {
    // bucket of plan position k: last b with indptr[b] <= k (warp-uniform)
    int64_t lo = 0, hi = (int64_t)t;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(pindptr + mid) <= k) lo = mid; else hi = mid;
    }
    const uint32_t wrd = __ldg(prow + k);
    const int64_t row = wrd & 0x7fffffffu;
    const bool neg = (wrd >> 31) != 0;
    TOut *out = sa + lo * ldsa;
    const int64_t rs = (int64_t)aip[row], re = (int64_t)aip[row + 1];
    for (int64_t p = rs + lane; p < re; p += 32) {
      const TOut v = (TOut)__ldg(av + p);
      atomicAdd(out + (int64_t)__ldg(aix + p), neg ? -v : v);
    }
  }
}

template <typename IP, typename IX, typename TV, typename TOut>
__global__ void __launch_bounds__(128) csr_rowseq_kernel(const int64_t *__restrict__ pindptr,
                                                         const uint32_t *__restrict__ prow,
                                                         uint64_t t, const IP *__restrict__ aip,
                                                         const IX *__restrict__ aix,
                                                         const TV *__restrict__ av, int64_t d,
                                                         double *__restrict__ acc64,
                                                         TOut *__restrict__ sa, int64_t ldsa) {
  const int lane = threadIdx.x & 31;
  const int64_t bucket = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (bucket >= (int64_t)t) return;
  // fp64 accumulation row: the output itself when it is fp64, else scratch
  double *acc = acc64 ? acc64 + bucket * d : (double *)(sa + bucket * ldsa);
  for (int64_t c = lane; c < d; c += 32) acc[c] = 0.0;
  __syncwarp();
  const int64_t beg = pindptr[bucket], end = pindptr[bucket + 1];
  uint32_t wn = beg < end ? __ldg(prow + beg) : 0u;
  for (int64_t k = beg; k < end; ++k) {
    const uint32_t wrd = wn;
    if (k + 1 < end) wn = __ldg(prow + k + 1);
    const int64_t row = wrd & 0x7fffffffu;
    const double sg = (wrd >> 31) ? -1.0 : 1.0;
    const int64_t rs = (int64_t)aip[row], re = (int64_t)aip[row + 1];
    for (int64_t p0 = rs; p0 < re; p0 += 128) {
      // up to 4 independent 32-wide chunks of the row in flight
      int64_t col[4];
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t p = p0 + 32 * u + lane;
        col[u] = p < re ? (int64_t)__ldg(aix + p) : -1;
        v[u] = p < re ? sg * (double)__ldg(av + p) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (col[u] >= 0) acc[col[u]] += v[u];
    }
    __syncwarp();
    __threadfence_block();
  }
  if (acc64) {
    __syncwarp();
    TOut *o = sa + bucket * ldsa;
    for (int64_t c = lane; c < d; c += 32) o[c] = (TOut)acc[c];
  }
}

}  // namespace
}  // namespace skt
