// csr_quad.cuh -- K4 "densify" kernel for canonical CSR with fp32 values, int32
// column indices and d <= 64 (BASELINE config 4's shape), 128-bit loads
// (sketch.py:155-164, bit-identical).
//
// The arithmetic is csr_tile.cuh's: one warp per bucket, a batch of 32 rows of
// the bucket (plan order) scattered into a zeroed 32 x 64 fp32 tile in shared
// memory (columns are distinct inside a canonical row: no conflicts), lane l
// adds tile[r][2l, 2l+1] into fp64 register accumulators for r = 0..31 -- per
// output column the bucket's rows in ascending order, absent entries adding
// +0.0 (exact) -- and the tile is cleared.  What differs is the data path:
//   * row descriptors stay in registers, lane per row (start rounded down to a
//     16-byte boundary, offset of the first entry, length, sign), read as
//     (start, end) pairs (row_extent_paired) and handed to the loading lanes
//     by shuffles: no descriptor staging in shared memory;
//   * four lanes per row, each one 128-bit load of indices and one of values:
//     the 16 aligned slots that contain the row's first entry cover rows of
//     <= 13 entries at any alignment and rows of 16 on a 16-byte boundary; 8
//     load instructions per 32 rows instead of 32, all issued before use and
//     in flight while the previous batch is accumulated;
//   * rows reaching up to 4 slots past the 16 (rows of 14-16 entries off a
//     16-byte boundary) take one more 128-bit slot group, longer rows the whole
//     warp per row from slot 16, both when the batch is scattered.
// Pipeline: batch b scattered / accumulated / cleared, batch b+1's nonzeros in
// flight, batch b+2's row extents, batch b+3's plan words.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

#ifndef SKT_QUAD_L2HINT
#define SKT_QUAD_L2HINT 1
#endif
#ifndef SKT_QUAD_MINB
#define SKT_QUAD_MINB 4
#endif
#ifndef SKT_QUAD_WARPS
#define SKT_QUAD_WARPS 4
#endif
constexpr int kQuadWarps = SKT_QUAD_WARPS;
constexpr int kQuadD = 64;                       // tile width (d <= 64)
constexpr int kQuadTileBytes = 32 * kQuadD * 4;  // per warp

// Slots 16..19 of the rows of a batch that reach up to 4 slots past their 16
// (rows of 14-16 entries off a 16-byte boundary): one more 128-bit load of
// indices and values by the row's first lane, scattered into the tile.
template <typename IP>
__device__ __noinline__ void quad_extra_slots(float *tile, const int32_t *__restrict__ aix,
                                              const float *__restrict__ av, IP b0, int mt0, int mt1, int mt2, int mt3,
                                              int g, int q) {
  const int mt[4] = {mt0, mt1, mt2, mt3};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const IP b = __shfl_sync(0xffffffffu, b0, 8 * i + g);
    const int m = mt[i];
    const int stop = ((m >> 8) & 3) + (m & 0xff);
    if (q == 0 && stop > 16 && stop <= 20) {
      const int4 c = __ldg(reinterpret_cast<const int4 *>(aix + b + 16));
      const float4 v = __ldg(reinterpret_cast<const float4 *>(av + b + 16));
      const uint32_t sg = (uint32_t)(m >> 16) << 31;
      float *trow = tile + (8 * i + g) * 64;
      const int cs[4] = {c.x, c.y, c.z, c.w};
      const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (16 + j < stop) trow[cs[j]] = __uint_as_float(__float_as_uint(vs[j]) ^ sg);
    }
  }
}

template <typename IP, typename TOut>
__global__ void __launch_bounds__(kQuadWarps * 32, SKT_QUAD_MINB) csr_quad_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, uint64_t t,
    const IP *__restrict__ aip, const int32_t *__restrict__ aix, const float *__restrict__ av, int d,
    TOut *__restrict__ sa, int64_t ldsa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t bucket = (int64_t)blockIdx.x * kQuadWarps + w;
  if (bucket >= (int64_t)t) return;
  float *tile = reinterpret_cast<float *>(smem_raw + (size_t)w * kQuadTileBytes);
  {
    uint4 *z = reinterpret_cast<uint4 *>(tile);
#pragma unroll
    for (int i = 0; i < kQuadTileBytes / 16 / 32; ++i) z[i * 32 + lane] = make_uint4(0, 0, 0, 0);
  }
  double acc0 = 0.0, acc1 = 0.0;
  const int g = lane >> 2, q = lane & 3;
  const int64_t beg = pindptr[bucket], end = pindptr[bucket + 1];

  // lane-per-row descriptor of a batch: base = row start rounded down to 4
  // entries, meta = length | offset of the first entry << 8 | sign << 16.
  // The extents are read as (start, end) pairs (see row_extent_paired); the
  // loads are issued one batch before the values are exchanged, so nothing
  // waits on them.
  const int hi = lane >> 4;
#if SKT_QUAD_L2HINT
  const uint64_t keep = l2_keep_policy();
#endif
  auto plan_word = [&](int64_t k0) -> uint32_t { return k0 + lane < end ? __ldg(prow + k0 + lane) : 0u; };
  auto extent_issue = [&](int64_t k0, uint32_t wd, IP &x1, IP &x2) {  // raw loads, untouched until finish
    const int64_t row = k0 + lane < end ? (int64_t)(wd & 0x7fffffffu) : (int64_t)-1;
    const int64_t other = __shfl_xor_sync(0xffffffffu, row, 16);
    const int64_t r1 = hi ? other : row, r2 = hi ? row : other;
    x1 = 0;
    x2 = 0;
#if SKT_QUAD_L2HINT
    if (r1 >= 0) x1 = ld_l2_keep(aip + r1 + hi, keep);
    if (r2 >= 0) x2 = ld_l2_keep(aip + r2 + hi, keep);
#else
    if (r1 >= 0) x1 = aip[r1 + hi];
    if (r2 >= 0) x2 = aip[r2 + hi];
#endif
  };
  auto extent_finish = [&](int64_t k0, uint32_t wd, IP x1, IP x2, IP &base, int &meta) {
    const IP s1 = __shfl_xor_sync(0xffffffffu, x1, 16), s2 = __shfl_xor_sync(0xffffffffu, x2, 16);
    const IP rs = hi ? s2 : x1;
    const int len = k0 + lane < end ? (int)((hi ? x2 : s1) - rs) : 0;
    base = len ? rs & ~(IP)3 : (IP)0;
    meta = len | ((int)(rs & 3) << 8) | ((int)(wd >> 31) << 16);
  };
  int4 ci[4];
  float4 cv[4];
  int mt[4];  // meta of rows 8 i + g of the batch in ci / cv
  auto load = [&](IP base, int meta) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = 8 * i + g;
      const IP b = __shfl_sync(0xffffffffu, base, r);
      const int m = __shfl_sync(0xffffffffu, meta, r);
      mt[i] = m;
      // unconditional loads: lanes whose slots lie past the row's end re-read its first
      // slots, empty rows the arrays' first (nnz > 0 here); the scatter ignores both
      const IP at = b + (4 * q < ((m >> 8) & 3) + (m & 0xff) ? 4 * q : 0);
#if SKT_QUAD_L2HINT
      ci[i] = __ldcs(reinterpret_cast<const int4 *>(aix + at));  // read once: evict first
      cv[i] = __ldcs(reinterpret_cast<const float4 *>(av + at));
#else
      ci[i] = __ldg(reinterpret_cast<const int4 *>(aix + at));
      cv[i] = __ldg(reinterpret_cast<const float4 *>(av + at));
#endif
    }
  };

  uint32_t w0 = plan_word(beg), w1 = plan_word(beg + 32), w2 = plan_word(beg + 64);
  IP b0, x1, x2;
  int m0;
  extent_issue(beg, w0, x1, x2);
  extent_finish(beg, w0, x1, x2, b0, m0);
  extent_issue(beg + 32, w1, x1, x2);
  load(b0, m0);

  for (int64_t k0 = beg; k0 < end; k0 += 32) {
    const int nrows = (int)((end - k0) < 32 ? (end - k0) : 32);
    // ---- scatter batch b: slot j of this lane is entry 4 q + j - offset of its row
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = mt[i];
      const int lo = ((m >> 8) & 3) - 4 * q, hi = lo + (m & 0xff);
      const uint32_t sg = (uint32_t)(m >> 16) << 31;
      float *trow = tile + (8 * i + g) * kQuadD;
      const int cs[4] = {ci[i].x, ci[i].y, ci[i].z, ci[i].w};
      const float vs[4] = {cv[i].x, cv[i].y, cv[i].z, cv[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j >= lo && j < hi) trow[cs[j]] = __uint_as_float(__float_as_uint(vs[j]) ^ sg);
    }
    // rows reaching past their 16 slots: up to 20 (rows of 14-16 entries off a 16-byte
    // boundary) one more 128-bit slot group, read by the row's first lane; longer rows the
    // whole warp per row from slot 16
    const int used = ((m0 >> 8) & 3) + (m0 & 0xff);  // slots of row `lane`
    if (__ballot_sync(0xffffffffu, used > 16 && used <= 20))  // warp-uniform; out of line: rare on aligned data
      quad_extra_slots<IP>(tile, aix, av, b0, mt[0], mt[1], mt[2], mt[3], g, q);
    for (uint32_t longm = __ballot_sync(0xffffffffu, used > 20); longm; longm &= longm - 1) {
      const int r = __ffs(longm) - 1;
      const IP b = __shfl_sync(0xffffffffu, b0, r);
      const int m = __shfl_sync(0xffffffffu, m0, r);
      const int stop = ((m >> 8) & 3) + (m & 0xff);
      const uint32_t sg = (uint32_t)(m >> 16) << 31;
      for (int e = 16 + lane; e < stop; e += 32)
        tile[r * kQuadD + __ldg(aix + b + e)] = __uint_as_float(__float_as_uint(__ldg(av + b + e)) ^ sg);
    }
    // ---- batch b+1 in flight, extent loads of b+2, plan words of b+3
    IP b1;
    int m1;
    extent_finish(k0 + 32, w1, x1, x2, b1, m1);
    load(b1, m1);
    extent_issue(k0 + 64, w2, x1, x2);
    const uint32_t w3 = plan_word(k0 + 96);
    __syncwarp();
    // ---- accumulate batch b in row order
    const float *tcol = tile + 2 * lane;
    if (nrows == 32) {
#pragma unroll
      for (int r0 = 0; r0 < 32; r0 += 8) {  // 8 rows' loads in flight, then the ordered adds
        float2 x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) x[r] = *reinterpret_cast<const float2 *>(tcol + (r0 + r) * kQuadD);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          acc0 += (double)x[r].x;
          acc1 += (double)x[r].y;
        }
      }
    } else {
      for (int r = 0; r < nrows; ++r) {
        const float2 x = *reinterpret_cast<const float2 *>(tcol + r * kQuadD);
        acc0 += (double)x.x;
        acc1 += (double)x.y;
      }
    }
    __syncwarp();
    // ---- clear the batch's rows of the tile
    {
      uint4 *z = reinterpret_cast<uint4 *>(tile);
      for (int i = lane; i < nrows * (kQuadD / 4); i += 32) z[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();  // the clear lands before the next batch's scatter
    b0 = b1;
    m0 = m1;
    w1 = w2;
    w2 = w3;
  }
  TOut *o = sa + bucket * ldsa;
  if (2 * lane < d) o[2 * lane] = (TOut)acc0;
  if (2 * lane + 1 < d) o[2 * lane + 1] = (TOut)acc1;
}

}  // namespace
}  // namespace skt
