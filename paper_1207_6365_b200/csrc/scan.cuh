// scan.cuh -- device-wide exclusive prefix sum of uint32 (reduce-then-scan,
// three launches, no atomics, deterministic).  Used by K1 (accepted-draw
// offsets under Lemire rejection) and K2 (radix-sort digit offsets).
#pragma once

#include "common.cuh"

namespace skt {
namespace {  // internal linkage: each translation unit gets its own copy

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total (all threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total) {
  __shared__ uint32_t warp_sums[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  uint32_t incl = warp_incl_scan(v);
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t x = lane < nwarps ? warp_sums[lane] : 0u;
    uint32_t xi = warp_incl_scan(x);
    warp_sums[lane] = xi - x;
    if (lane == 31) warp_sums[31] = xi;  // lane 31 slot is unused when nwarps < 32
  }
  __syncthreads();
  // nwarps <= 8 here, so slot 31 holds the total; guard for 32 warps anyway
  uint32_t base = warp_sums[wid];
  *total = warp_sums[31];
  __syncthreads();
  return base + incl - v;
}

__global__ void scan_reduce_kernel(const uint32_t *__restrict__ data, int64_t count,
                                   uint32_t *__restrict__ partials) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < count) s += data[base + k];
  uint32_t tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// single block: exclusive scan of partials[0..nb) in place, total in partials[nb]
__global__ void scan_partials_kernel(uint32_t *__restrict__ partials, int64_t nb) {
  uint32_t carry = 0;
  for (int64_t off = 0; off < nb; off += kScanTile) {
    const int64_t base = off + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      v[k] = base + k < nb ? partials[base + k] : 0u;
      s += v[k];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan(s, &tot) + carry;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (base + k < nb) partials[base + k] = ex;
      ex += v[k];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) partials[nb] = carry;
}

__global__ void scan_apply_kernel(uint32_t *__restrict__ data, int64_t count,
                                  const uint32_t *__restrict__ partials) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < count ? data[base + k] : 0u;
    s += v[k];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan(s, &tot) + partials[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < count) data[base + k] = ex;
    ex += v[k];
  }
}

inline int64_t scan_partials_len(int64_t count) {
  return (count + kScanTile - 1) / kScanTile + 1;
}

// In-place exclusive scan of data[0..count); partials needs
// scan_partials_len(count) words; the grand total lands in partials[nb].
inline skt_status exclusive_scan_u32(uint32_t *data, int64_t count, uint32_t *partials,
                                     cudaStream_t stream, const char *fn) {
  const int64_t nb = (count + kScanTile - 1) / kScanTile;
  if (nb > 0) SKT_LAUNCH(scan_reduce_kernel, (unsigned)nb, kScanThreads, 0, stream, data, count, partials);
  SKT_LAUNCH(scan_partials_kernel, 1, kScanThreads, 0, stream, partials, nb);
  if (nb > 0) SKT_LAUNCH(scan_apply_kernel, (unsigned)nb, kScanThreads, 0, stream, data, count, partials);
  return check_launch(fn);
}

}  // namespace
}  // namespace skt
