// common.cuh -- shared helpers of the sm_100a CountSketch library:
// error plumbing for the C ABI, launch accounting, 128-bit PCG64 arithmetic.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <string>

#include "sketch_b200.h"

namespace skt {

// ---- error plumbing ------------------------------------------------------
void set_error(const std::string &msg);
std::atomic<uint64_t> &launch_counter();

inline skt_status fail(skt_status st, const char *fn, const std::string &msg) {
  set_error(std::string(fn) + ": " + msg);
  return st;
}

inline skt_status check_launch(const char *fn) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SKT_ECUDA, fn, cudaGetErrorString(e));
  return SKT_OK;
}

#define SKT_CUDA_TRY(expr, fn)                                     \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return ::skt::fail(SKT_ECUDA, fn, cudaGetErrorString(_e)); \
  } while (0)

// Every kernel launch goes through this macro so skt_launch_count() is exact.
#define SKT_LAUNCH(kernel, grid, block, smem, stream, ...)                     \
  do {                                                                         \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                \
    ::skt::launch_counter().fetch_add(1, std::memory_order_relaxed);           \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

// ---- L2 residency hints ---------------------------------------------------
// Loads that should stay in L2 while a stream of read-once data passes through
// it (the CSR row pointers next to the gathered index / value segments).
#ifdef __CUDACC__
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ld_l2_keep(const int32_t *a, uint64_t pol) {
  int32_t v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_l2_keep(const int64_t *a, uint64_t pol) {
  int64_t v;
  asm("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
#endif

// ---- CSR row extents of 32 scattered rows ----------------------------------
// Lane l holds row id `row` (< 0: none) and gets (start, length) of that row.
// indptr[row] and indptr[row + 1] share a 128-byte line, so instead of one
// gather of the 32 starts and one of the 32 ends (32 lines each), the first
// load reads start and end of the rows of lanes 0..15 (lanes l and l + 16 read
// the pair of row l) and the second those of lanes 16..31: 16 lines per load.
#ifdef __CUDACC__
template <typename IP>
__device__ __forceinline__ void row_extent_paired(const IP *__restrict__ aip, int64_t row, int lane, int64_t &rs,
                                                  int &len) {
  const int64_t other = __shfl_xor_sync(0xffffffffu, row, 16);
  const int hi = lane >> 4;  // 0: this half reads starts, 1: ends
  const int64_t r1 = hi ? other : row, r2 = hi ? row : other;
  const int64_t x1 = r1 >= 0 ? (int64_t)aip[r1 + hi] : 0;
  const int64_t x2 = r2 >= 0 ? (int64_t)aip[r2 + hi] : 0;
  const int64_t s1 = __shfl_xor_sync(0xffffffffu, x1, 16), s2 = __shfl_xor_sync(0xffffffffu, x2, 16);
  rs = hi ? s2 : x1;
  len = row >= 0 ? (int)((hi ? x2 : s1) - rs) : 0;
  if (row < 0) rs = 0;
}
#endif

// ---- 128-bit PCG64 -------------------------------------------------------
typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | (u128)lo;
}

// numpy pcg64 default multiplier (PCG_DEFAULT_MULTIPLIER_128)
__host__ __device__ __forceinline__ u128 pcg_mult() {
  return mk128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull);
}

// XSL-RR output of a (post-step) state
__host__ __device__ __forceinline__ uint64_t pcg_output(u128 st) {
  uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
  unsigned rot = (unsigned)(st >> 122);
  uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Affine LCG map x -> mult * x + plus, composed delta times (pcg_advance_lcg_128).
struct Affine128 {
  u128 mult, plus;
};
__host__ __device__ __forceinline__ Affine128 lcg_power(uint64_t delta, u128 inc) {
  u128 cur_mult = pcg_mult(), cur_plus = inc;
  u128 acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return Affine128{acc_mult, acc_plus};
}

}  // namespace skt
