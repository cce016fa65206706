// csr_tile.cuh -- K4 "densify" kernel for canonical CSR with narrow d and
// rows of ~8+ nonzeros (BASELINE config 4 shape).
//
// One warp per bucket.  A batch of R rows of the bucket (plan order) is
// scattered into a zeroed R x d tile in shared memory (signed values; columns
// are distinct inside a canonical row, so the scatter has no conflicts), then
// lane l adds tile[r][2l, 2l+1 (+64k)] into fp64 register accumulators for
// r = 0..R-1, and the written entries are re-zeroed.  Per output column the
// additions run over the bucket's rows in ascending order; absent entries add
// +0.0, an exact identity (the accumulator is never -0.0: it starts at +0.0 and
// x + y = -0.0 only if both are -0.0), so the result is bit-identical to the
// reference's bincount.
//
// Software pipeline (three batches deep): while batch b is scattered,
// accumulated and re-zeroed, the nonzeros of batch b+1 are already in flight
// into registers, the row descriptors (indptr pairs) of batch b+2 and the plan
// words of batch b+3.  A batch's nonzeros are fetched G lanes per row (G =
// 4/8/16 by the batch's longest row); the first G of every row are prefetched,
// longer rows' tails are fetched by the whole warp when the batch is scattered.
// The random row order makes this kernel request-rate bound (the index and
// value segments of a row are ~64 B at arbitrary offsets): the ceiling is the
// same access pattern without arithmetic, tools/gather_bench.cu.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace skt {
namespace {

constexpr int kTileWarps = 4;
constexpr int kTileMaxD = 256;
constexpr int kTileDescSlots = 2;  // double-buffered batch descriptors

template <typename TV>
__host__ __device__ constexpr int tile_bytes() { return sizeof(TV) == 4 ? 8192 : 12288; }
template <typename TV>
__host__ __device__ constexpr int tile_slice_bytes() {
  return tile_bytes<TV>() + kTileDescSlots * 32 * (int)sizeof(int4);
}

// The first G nonzeros of every row of a batch into registers, G lanes per
// row; row descriptors from shared memory (broadcast).
template <int G, typename IX, typename TV>
__device__ __forceinline__ void load_rows(const int4 *__restrict__ desc, int nrows, const IX *__restrict__ aix,
                                          const TV *__restrict__ av, int lane, int32_t (&cc)[16], TV (&vv)[16]) {
  constexpr int S = 32 / G;
  const int g = lane / G, gl = lane % G;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int r = i * S + g;
    cc[i] = -1;  // columns < d <= 256: int32 registers for any index type
    if (i * S < nrows) {  // warp-uniform
      const int4 ds = desc[r];
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      if (r < nrows && gl < ds.z) {
        cc[i] = (int32_t)__ldg(aix + rs + gl);
        vv[i] = __ldg(av + rs + gl);
      }
    }
  }
}

template <int G, typename TV>
__device__ __forceinline__ void store_rows(const int4 *__restrict__ desc, TV *tile, int dp, int lane,
                                           const int32_t (&cc)[16], const TV (&vv)[16]) {
  constexpr int S = 32 / G;
  const int g = lane / G;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int r = i * S + g;
    if (cc[i] != -1) tile[r * dp + cc[i]] = desc[r].w ? -vv[i] : vv[i];
  }
}

template <int G, typename TV>
__device__ __forceinline__ void unscatter_rows(TV *tile, int dp, int lane, const int32_t (&cc)[16]) {
  constexpr int S = 32 / G;
  const int g = lane / G;
#pragma unroll
  for (int i = 0; i < G; ++i)
    if (cc[i] != -1) tile[(i * S + g) * dp + cc[i]] = (TV)0;
}

__device__ __forceinline__ int tile_g(int lmax) { return lmax <= 4 ? 4 : lmax <= 8 ? 8 : 16; }

#ifndef SKT_TILE_PAIRED
#define SKT_TILE_PAIRED 1
#endif
#ifndef SKT_TILE_ONEBUF
#define SKT_TILE_ONEBUF 1
#endif
#ifndef SKT_TILE_MINB
#define SKT_TILE_MINB (SKT_TILE_ONEBUF ? 5 : 4)
#endif

template <typename IP, typename IX, typename TV, typename TOut, int kChunks>
__global__ void __launch_bounds__(kTileWarps * 32, SKT_TILE_MINB) csr_tile_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, uint64_t t,
    const IP *__restrict__ aip, const IX *__restrict__ aix, const TV *__restrict__ av, int d,
    int dp, int R, TOut *__restrict__ sa, int64_t ldsa) {
  using V2 = typename std::conditional<sizeof(TV) == 4, float2, double2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t bucket = (int64_t)blockIdx.x * kTileWarps + w;
  if (bucket >= (int64_t)t) return;
  unsigned char *slice = smem_raw + (size_t)w * tile_slice_bytes<TV>();
  int4 *descs = (int4 *)slice;  // [slot][row of the batch]: rs lo, rs hi, len, neg
  TV *tile = (TV *)(slice + kTileDescSlots * 32 * sizeof(int4));
  for (int i = lane; i < R * dp; i += 32) tile[i] = (TV)0;

  double acc[kChunks][2];
#pragma unroll
  for (int k = 0; k < kChunks; ++k) acc[k][0] = acc[k][1] = 0.0;

  const int64_t beg = pindptr[bucket], end = pindptr[bucket + 1];
  auto plan_word = [&](int64_t k0) -> uint32_t {
    return (lane < R && k0 + lane < end) ? __ldg(prow + k0 + lane) : 0u;
  };
  auto row_desc = [&](int64_t k0, uint32_t wd, int64_t &rs, int &len) {
#if SKT_TILE_PAIRED
    row_extent_paired(aip, (lane < R && k0 + lane < end) ? (int64_t)(wd & 0x7fffffffu) : (int64_t)-1, lane, rs, len);
#else
    rs = 0;
    len = 0;
    if (lane < R && k0 + lane < end) {
      const int64_t row = wd & 0x7fffffffu;
      rs = (int64_t)aip[row];
      len = (int)((int64_t)aip[row + 1] - rs);
    }
#endif
  };
  // publish a batch's descriptors (lane r = row r) into a slot; returns G
  auto publish = [&](int slot, int64_t k0, int64_t rs, int len, uint32_t wd) -> int {
    const int nrows = (int)((end - k0) < R ? (end - k0) : R);
    if (lane < nrows) descs[slot * 32 + lane] = make_int4((int)(uint32_t)rs, (int)(rs >> 32), len, (int)(wd >> 31));
    return tile_g(__reduce_max_sync(0xffffffffu, lane < nrows ? len : 0));
  };
  auto load_sw = [&](int G, const int4 *dsc, int nrows, int32_t (&c)[16], TV (&v)[16]) {
    if (G == 4)
      load_rows<4>(dsc, nrows, aix, av, lane, c, v);
    else if (G == 8)
      load_rows<8>(dsc, nrows, aix, av, lane, c, v);
    else
      load_rows<16>(dsc, nrows, aix, av, lane, c, v);
  };

  // ---- prologue: batch 0 descriptors + nonzeros, batch 1 descriptors,
  // batch 2 plan words
  uint32_t w0 = plan_word(beg);
  int64_t rs0;
  int len0;
  row_desc(beg, w0, rs0, len0);
  uint32_t w1 = plan_word(beg + R);
  int64_t rs1;
  int len1;
  row_desc(beg + R, w1, rs1, len1);
  uint32_t w2 = plan_word(beg + 2 * (int64_t)R);
#if SKT_TILE_ONEBUF
  // one register set: batch b is scattered first, then batch b+1's nonzeros
  // are requested into the same registers and stay in flight while batch b
  // is accumulated; the tile is cleared whole (no per-entry columns kept)
  int slot = 0;
  int32_t cc[16];
  TV vv[16];
  int g0 = publish(slot, beg, rs0, len0, w0);
  __syncwarp();
  load_sw(g0, descs + slot * 32, (int)((end - beg) < R ? (end - beg) : R), cc, vv);
  for (int64_t k0 = beg; k0 < end; k0 += R) {
    const int nrows = (int)((end - k0) < R ? (end - k0) : R);
    const int4 *dcur = descs + slot * 32;
    const int64_t k1 = k0 + R, k2 = k0 + 2 * (int64_t)R, k3 = k0 + 3 * (int64_t)R;
    // ---- scatter batch b
    if (g0 == 4)
      store_rows<4>(dcur, tile, dp, lane, cc, vv);
    else if (g0 == 8)
      store_rows<8>(dcur, tile, dp, lane, cc, vv);
    else
      store_rows<16>(dcur, tile, dp, lane, cc, vv);
    uint32_t longm = __ballot_sync(0xffffffffu, lane < nrows && len0 > g0);
    while (longm) {  // rows longer than G: whole warp per row
      const int r = __ffs(longm) - 1;
      longm &= longm - 1;
      const int4 ds = dcur[r];
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      for (int q = g0 + lane; q < ds.z; q += 32) {
        const TV v = __ldg(av + rs + q);
        tile[r * dp + (int)__ldg(aix + rs + q)] = ds.w ? -v : v;
      }
    }
    // ---- batch b+1 in flight, descriptors of b+2, plan words of b+3
    int g1 = 4;
    if (k1 < end) {
      g1 = publish(slot ^ 1, k1, rs1, len1, w1);
      __syncwarp();
      load_sw(g1, descs + (slot ^ 1) * 32, (int)((end - k1) < R ? (end - k1) : R), cc, vv);
    }
    int64_t rs2;
    int len2;
    row_desc(k2, w2, rs2, len2);
    const uint32_t w3 = plan_word(k3);
    __syncwarp();
    // ---- accumulate batch b in row order
    for (int r = 0; r < nrows; ++r) {
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = 64 * k + 2 * lane;
        if (c < dp) {
          const V2 x = *reinterpret_cast<const V2 *>(tile + r * dp + c);
          acc[k][0] += (double)x.x;
          acc[k][1] += (double)x.y;
        }
      }
    }
    __syncwarp();
    // ---- clear the batch's rows of the tile
    {
      uint4 *z = reinterpret_cast<uint4 *>(tile);
      const int words = (int)(((size_t)nrows * dp * sizeof(TV) + 15) / 16);
      for (int i = lane; i < words; i += 32) z[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();  // the clear lands before the next batch's scatter
    g0 = g1;
    len0 = len1;
    rs1 = rs2;
    len1 = len2;
    w1 = w2;
    w2 = w3;
    slot ^= 1;
  }
#else
  int slot = 0;
  int32_t c0[16], c1[16];
  TV v0[16], v1[16];
  int g0 = publish(slot, beg, rs0, len0, w0);
  __syncwarp();
  load_sw(g0, descs + slot * 32, (int)((end - beg) < R ? (end - beg) : R), c0, v0);

  for (int64_t k0 = beg; k0 < end; k0 += R) {
    const int nrows = (int)((end - k0) < R ? (end - k0) : R);
    const int4 *dcur = descs + slot * 32;
    const int64_t k1 = k0 + R, k2 = k0 + 2 * (int64_t)R, k3 = k0 + 3 * (int64_t)R;
    // ---- batch b+1: descriptors published, nonzeros in flight
    int g1 = 4;
    if (k1 < end) {
      g1 = publish(slot ^ 1, k1, rs1, len1, w1);
      __syncwarp();
      load_sw(g1, descs + (slot ^ 1) * 32, (int)((end - k1) < R ? (end - k1) : R), c1, v1);
    }
    // ---- batch b+2 descriptors, batch b+3 plan words
    int64_t rs2;
    int len2;
    row_desc(k2, w2, rs2, len2);
    const uint32_t w3 = plan_word(k3);
    // ---- scatter batch b
    if (g0 == 4)
      store_rows<4>(dcur, tile, dp, lane, c0, v0);
    else if (g0 == 8)
      store_rows<8>(dcur, tile, dp, lane, c0, v0);
    else
      store_rows<16>(dcur, tile, dp, lane, c0, v0);
    uint32_t longm = __ballot_sync(0xffffffffu, lane < nrows && len0 > g0);
    const uint32_t had_long = longm;
    while (longm) {  // rows longer than G: whole warp per row
      const int r = __ffs(longm) - 1;
      longm &= longm - 1;
      const int4 ds = dcur[r];
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      for (int q = g0 + lane; q < ds.z; q += 32) {
        const TV v = __ldg(av + rs + q);
        tile[r * dp + (int)__ldg(aix + rs + q)] = ds.w ? -v : v;
      }
    }
    __syncwarp();
    // ---- accumulate batch b in row order
    for (int r = 0; r < nrows; ++r) {
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = 64 * k + 2 * lane;
        if (c < dp) {
          const V2 x = *reinterpret_cast<const V2 *>(tile + r * dp + c);
          acc[k][0] += (double)x.x;
          acc[k][1] += (double)x.y;
        }
      }
    }
    __syncwarp();
    // ---- re-zero exactly what was written
    if (g0 == 4)
      unscatter_rows<4>(tile, dp, lane, c0);
    else if (g0 == 8)
      unscatter_rows<8>(tile, dp, lane, c0);
    else
      unscatter_rows<16>(tile, dp, lane, c0);
    for (uint32_t m = had_long; m; m &= m - 1) {
      const int r = __ffs(m) - 1;
      for (int c = lane; c < dp; c += 32) tile[r * dp + c] = (TV)0;
    }
    // ---- rotate the pipeline
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      c0[i] = c1[i];
      v0[i] = v1[i];
    }
    g0 = g1;
    len0 = len1;
    rs1 = rs2;
    len1 = len2;
    w1 = w2;
    w2 = w3;
    slot ^= 1;
  }
#endif
  TOut *o = sa + bucket * ldsa;
#pragma unroll
  for (int k = 0; k < kChunks; ++k) {
    const int c = 64 * k + 2 * lane;
    if (c < d) o[c] = (TOut)acc[k][0];
    if (c + 1 < d) o[c + 1] = (TOut)acc[k][1];
  }
}

}  // namespace
}  // namespace skt
