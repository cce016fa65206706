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

// Deterministic wide-d kernel, one BLOCK per bucket (config 5: t = 400
// buckets of ~655 rows, d = 262,144): the block walks the bucket's rows in
// ascending order; a row's stored entries (distinct columns in canonical
// CSR) are spread over all 256 threads, each adding s_i * v into the fp64
// output row with a fire-and-forget reduction (RED.ADD.F64, performed in L2
// as acc + v, round to nearest), and a fence + block barrier separates
// consecutive rows -- so every output element still receives its additions
// in ascending row order (bit-identical).  The next row's indices / values
// are loaded before the barrier, from row descriptors staged 256 at a time in
// shared memory.  400 blocks x 8 warps keep ~20x more loads in flight than a
// warp per bucket, and no thread waits on a read of the accumulator.  The
// kernel then runs at the random read-modify-write rate of HBM (the 839 MB of
// accumulators do not fit L2; measured: dropping the fence changes < 2%).
constexpr int kRowseqThreads = 256;

template <typename IP, typename IX, typename TV>
__global__ void __launch_bounds__(kRowseqThreads) csr_rowseq_block_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, uint64_t t,
    const IP *__restrict__ aip, const IX *__restrict__ aix, const TV *__restrict__ av, int64_t d,
    double *__restrict__ sa, int64_t ldsa) {
  constexpr int kPer = 4;  // entries per thread per step (rows up to 1024 entries in one pass)
  const int64_t bucket = blockIdx.x;
  if (bucket >= (int64_t)t) return;
  double *acc = sa + bucket * ldsa;
  for (int64_t c = threadIdx.x; c < d; c += kRowseqThreads) acc[c] = 0.0;
  const int64_t beg = pindptr[bucket], end = pindptr[bucket + 1];
  // row descriptors (start, end, sign) of the next kRowseqThreads plan
  // positions, fetched one per thread in parallel: the per-row critical path
  // is then a single dependent load (the entries), not plan -> indptr -> entries
  __shared__ int64_t s_rs[kRowseqThreads], s_re[kRowseqThreads];
  __shared__ double s_sg[kRowseqThreads];
  auto load_desc = [&](int64_t k0) {
    const int64_t k = k0 + threadIdx.x;
    int64_t rs = 0, re = 0;
    double sg = 1.0;
    if (k < end) {
      const uint32_t wrd = __ldg(prow + k);
      const int64_t row = wrd & 0x7fffffffu;
      sg = (wrd >> 31) ? -1.0 : 1.0;
      rs = (int64_t)aip[row];
      re = (int64_t)aip[row + 1];
    }
    s_rs[threadIdx.x] = rs;
    s_re[threadIdx.x] = re;
    s_sg[threadIdx.x] = sg;
  };
  int64_t col[kPer];
  double val[kPer];
  // row k's entries for this thread: positions rs + threadIdx.x + j * 256
  auto load_entries = [&](int64_t b0, int64_t b1, double s) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t p = b0 + threadIdx.x + (int64_t)j * kRowseqThreads;
      col[j] = p < b1 ? (int64_t)__ldg(aix + p) : -1;
      val[j] = p < b1 ? s * (double)__ldg(av + p) : 0.0;
    }
  };
  auto first = [&](int64_t rs, int64_t re) {
    return rs + (re - rs < kPer * kRowseqThreads ? re - rs : kPer * kRowseqThreads);
  };
  load_desc(beg);
  __syncthreads();  // descriptors + zeroed row visible
  int64_t rs = s_rs[0], re = s_re[0];
  double sg = s_sg[0];
  load_entries(rs, first(rs, re), sg);
  for (int64_t k = beg; k < end; ++k) {
    // row k's additions as fire-and-forget fp64 reductions (RED.ADD: one per
    // column per row, columns distinct inside a canonical row)
    for (int64_t p0 = rs + kPer * kRowseqThreads; p0 < re; p0 += kRowseqThreads) {
      const int64_t p = p0 + threadIdx.x;
      if (p < re) atomicAdd(acc + (int64_t)__ldg(aix + p), sg * (double)__ldg(av + p));
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (col[j] >= 0) atomicAdd(acc + col[j], val[j]);
    const int64_t k1 = k + 1;
    const int slot = (int)((k1 - beg) % kRowseqThreads);
    if (slot == 0 && k1 < end) {
      __syncthreads();  // everyone done reading the old descriptors
      load_desc(k1);
      __syncthreads();
    }
    // the next row's entries go in flight before the barrier
    if (k1 < end) {
      rs = s_rs[slot];
      re = s_re[slot];
      sg = s_sg[slot];
      load_entries(rs, first(rs, re), sg);
    }
    // row k's reductions performed before any of row k+1's: per output
    // element the additions stay in ascending row order (bit-identical)
    __threadfence();
    __syncthreads();
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
