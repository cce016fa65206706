// csr_group.cuh -- K4 grouped-sweep kernel for canonical CSR with narrow d and
// short rows (<= 8 nonzeros on average; BASELINE config 2 shape).
//
#pragma once

#include "common.cuh"

namespace skt {
namespace {

// K4 sweep kernel (canonical CSR, narrow d).  One warp owns a bucket GROUP
// (2^shift consecutive buckets) and keeps the group's SA rows as fp64
// accumulators in shared memory.  It walks the group's rows in ascending row
// order (the grouped plan), so all warps sweep A from low to high rows at about
// the same rate: rows being read at any moment are clustered, sectors shared by
// adjacent rows and DRAM pages are fetched once and hit in L2 for the others.
// A chunk of 32 rows is gathered with G lanes per row (all loads in flight at
// once, prefetched descriptors); then S = 32/G rows are added per warp step
// when their buckets differ, or serialised in row order when they share one --
// per SA element the additions run in ascending row order, bit-identical to
// the reference's bincount.  Rows longer than G finish with a whole-warp tail.
// ---------------------------------------------------------------------------
constexpr int kGroupWarps = 8;

template <typename IP, typename IX, typename TV, typename TOut, int G>
__global__ void __launch_bounds__(kGroupWarps * 32) csr_group_kernel(
    const int64_t *__restrict__ gptr, const uint32_t *__restrict__ grow,
    const uint8_t *__restrict__ gblo, int64_t ngroups, int shift, uint64_t t,
    const IP *__restrict__ aip, const IX *__restrict__ aix, const TV *__restrict__ av, int d,
    TOut *__restrict__ sa, int64_t ldsa) {
  constexpr int S = 32 / G;   // rows per warp step
  constexpr int kSteps = G;   // steps per chunk of 32 rows
  extern __shared__ __align__(16) double sacc[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t group = (int64_t)blockIdx.x * kGroupWarps + w;
  if (group >= ngroups) return;
  const int gb = 1 << shift;
  double *acc = sacc + (size_t)w * gb * d;
  for (int i = lane; i < gb * d; i += 32) acc[i] = 0.0;
  const int g = lane / G, gl = lane % G;

  const int64_t beg = gptr[group], end = gptr[group + 1];
  // descriptors of the current chunk (lane j <-> row j): row start, length,
  // packed (bucket-in-group | neg << 8); plan words of the next chunk.
  uint32_t wc = beg + lane < end ? __ldg(grow + beg + lane) : 0u;
  uint32_t bc = beg + lane < end ? (uint32_t)(gblo ? __ldg(gblo + beg + lane) : 0) : 0u;
  int64_t rs_c;
  int len_c;
  row_extent_paired(aip, beg + lane < end ? (int64_t)(wc & 0x7fffffffu) : (int64_t)-1, lane, rs_c, len_c);
  uint32_t wn = beg + 32 + lane < end ? __ldg(grow + beg + 32 + lane) : 0u;
  uint32_t bn = beg + 32 + lane < end ? (uint32_t)(gblo ? __ldg(gblo + beg + 32 + lane) : 0) : 0u;

  for (int64_t k0 = beg; k0 < end; k0 += 32) {
    const int nrows = (int)((end - k0) < 32 ? (end - k0) : 32);
    const uint32_t pk_c = bc | ((wc >> 31) << 8);
    // ---- gather this chunk (all loads issued before any use)
    IX cc[kSteps];
    TV vv[kSteps];
#pragma unroll
    for (int i = 0; i < kSteps; ++i) {
      const int r = i * S + g;
      const int64_t rs_r = __shfl_sync(0xffffffffu, rs_c, r);
      const int len_r = __shfl_sync(0xffffffffu, len_c, r);
      cc[i] = (IX)-1;
      if (r < nrows && gl < len_r) {
        cc[i] = __ldg(aix + rs_r + gl);
        vv[i] = __ldg(av + rs_r + gl);
      }
    }
    const uint32_t longm = __ballot_sync(0xffffffffu, lane < nrows && len_c > G);
    // ---- prefetch: descriptors of the next chunk, plan words of the one after
    int64_t rs_n;
    int len_n;
    row_extent_paired(aip, k0 + 32 + lane < end ? (int64_t)(wn & 0x7fffffffu) : (int64_t)-1, lane, rs_n, len_n);
    const int64_t k2 = k0 + 64;
    const uint32_t wn2 = k2 + lane < end ? __ldg(grow + k2 + lane) : 0u;
    const uint32_t bn2 = k2 + lane < end ? (uint32_t)(gblo ? __ldg(gblo + k2 + lane) : 0) : 0u;
    // ---- accumulate in row order.  Rows of a step (lanes i*S .. i*S+S-1 of
    // the chunk) that share a bucket serialise that step in row order: one
    // match over (bucket, step) flags every clashing step of the chunk at once.
    const uint32_t ckey = lane < nrows ? ((bc & 0xffu) | ((uint32_t)(lane / S) << 8)) : (0x10000u | (uint32_t)lane);
    const uint32_t clash_lanes = __ballot_sync(0xffffffffu, __popc(__match_any_sync(0xffffffffu, ckey)) > 1);
#pragma unroll
    for (int i = 0; i < kSteps; ++i) {
      if (i * S < nrows) {  // warp-uniform
        const int r = i * S + g;
        const uint32_t pk_r = __shfl_sync(0xffffffffu, pk_c, r);
        const int bl_r = (int)(pk_r & 0xffu);
        const bool neg_r = (pk_r >> 8) != 0;
        const bool clash = ((clash_lanes >> (i * S)) & ((1u << S) - 1u)) != 0;
        const uint32_t steplong = (longm >> (i * S)) & ((1u << S) - 1u);
        const bool serial = clash || steplong != 0;
        const int rank = serial ? g : 0;
        const int rounds = serial ? S : 1;
        for (int rr = 0; rr < rounds; ++rr) {
          if (rank == rr && cc[i] != (IX)-1) {
            const double v = (double)vv[i];
            acc[bl_r * d + (int)cc[i]] += neg_r ? -v : v;
          }
          __syncwarp();
          if (steplong & (1u << rr)) {  // tail of a long row, right after its head
            const int rt = i * S + rr;
            const int64_t rs_t = __shfl_sync(0xffffffffu, rs_c, rt);
            const int len_t = __shfl_sync(0xffffffffu, len_c, rt);
            const uint32_t pk_t = __shfl_sync(0xffffffffu, pk_c, rt);
            for (int q = G + lane; q < len_t; q += 32) {
              const double v = (double)__ldg(av + rs_t + q);
              acc[(int)(pk_t & 0xffu) * d + (int)__ldg(aix + rs_t + q)] += (pk_t >> 8) ? -v : v;
            }
            __syncwarp();
          }
        }
      }
    }
    wc = wn;
    bc = bn;
    rs_c = rs_n;
    len_c = len_n;
    wn = wn2;
    bn = bn2;
  }
  __syncwarp();
  for (int b = 0; b < gb; ++b) {
    const uint64_t bucket = (uint64_t)group * gb + b;
    if (bucket >= t) break;
    TOut *o = sa + bucket * ldsa;
    for (int c = lane; c < d; c += 32) o[c] = (TOut)acc[b * d + c];
  }
}

}  // namespace
}  // namespace skt
