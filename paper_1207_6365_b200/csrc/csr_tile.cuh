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
// reference's bincount.  The row descriptors of batch b+1 and the plan words of
// batch b+2 are in flight while batch b is gathered and accumulated; a batch's
// nonzeros are fetched G lanes per row (G = 4/8/16 by the batch's longest row)
// with all loads issued before the tile stores.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace skt {
namespace {

constexpr int kTileWarps = 4;
constexpr int kTileMaxD = 256;

template <typename TV>
__host__ __device__ constexpr int tile_bytes() { return sizeof(TV) == 4 ? 8192 : 12288; }

// Phase 1 of a batch: the first G nonzeros of every row, G lanes per row, all
// loads issued before the tile stores.  Row descriptors come from shared
// memory (broadcast).  Returns nothing; entries beyond G are left to phase 2.
template <int G, typename IX, typename TV>
__device__ __forceinline__ void scatter_rows(const int4 *__restrict__ desc, int nrows,
                                             const IX *__restrict__ aix,
                                             const TV *__restrict__ av, TV *tile, int dp,
                                             int lane, IX (&cc)[16]) {
  constexpr int S = 32 / G;
  const int g = lane / G, gl = lane % G;
  TV vv[G];
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int r = i * S + g;
    cc[i] = (IX)-1;
    if (i * S < nrows) {  // warp-uniform
      const int4 ds = desc[r];
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      if (r < nrows && gl < ds.z) {
        cc[i] = __ldg(aix + rs + gl);
        vv[i] = __ldg(av + rs + gl);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int r = i * S + g;
    if (cc[i] != (IX)-1) tile[r * dp + (int)cc[i]] = desc[r].w ? -vv[i] : vv[i];
  }
}

template <int G, typename IX, typename TV>
__device__ __forceinline__ void unscatter_rows(const int4 *__restrict__ desc, int nrows,
                                               TV *tile, int dp, int lane, const IX (&cc)[16]) {
  constexpr int S = 32 / G;
  const int g = lane / G;
#pragma unroll
  for (int i = 0; i < G; ++i)
    if (cc[i] != (IX)-1) tile[(i * S + g) * dp + (int)cc[i]] = (TV)0;
}

template <typename IP, typename IX, typename TV, typename TOut, int kChunks>
__global__ void __launch_bounds__(kTileWarps * 32, 6) csr_tile_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, uint64_t t,
    const IP *__restrict__ aip, const IX *__restrict__ aix, const TV *__restrict__ av, int d,
    int dp, int R, TOut *__restrict__ sa, int64_t ldsa) {
  using V2 = typename std::conditional<sizeof(TV) == 4, float2, double2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t bucket = (int64_t)blockIdx.x * kTileWarps + w;
  if (bucket >= (int64_t)t) return;
  unsigned char *slice = smem_raw + (size_t)w * (tile_bytes<TV>() + 32 * sizeof(int4));
  int4 *desc = (int4 *)slice;  // per row of the batch: rs lo, rs hi, len, neg
  TV *tile = (TV *)(slice + 32 * sizeof(int4));
  for (int i = lane; i < R * dp; i += 32) tile[i] = (TV)0;

  double acc[kChunks][2];
#pragma unroll
  for (int k = 0; k < kChunks; ++k) acc[k][0] = acc[k][1] = 0.0;

  const int64_t beg = pindptr[bucket], end = pindptr[bucket + 1];
  // software pipeline: descriptors of batch b+1 and the plan words of batch
  // b+2 are in flight while batch b is gathered and accumulated.
  uint32_t w_cur = (lane < R && beg + lane < end) ? __ldg(prow + beg + lane) : 0u;
  int64_t rs_cur = 0;
  int len_cur = 0;
  if (lane < R && beg + lane < end) {
    const int64_t row = w_cur & 0x7fffffffu;
    rs_cur = (int64_t)aip[row];
    len_cur = (int)((int64_t)aip[row + 1] - rs_cur);
  }
  uint32_t w_nxt = (lane < R && beg + R + lane < end) ? __ldg(prow + beg + R + lane) : 0u;

  for (int64_t k0 = beg; k0 < end; k0 += R) {
    const int nrows = (int)((end - k0) < R ? (end - k0) : R);
    __syncwarp();
    if (lane < nrows) desc[lane] = make_int4((int)(uint32_t)rs_cur, (int)(rs_cur >> 32), len_cur, (int)(w_cur >> 31));
    const int lmax = __reduce_max_sync(0xffffffffu, lane < nrows ? len_cur : 0);
    // prefetch: descriptors of the next batch, plan words of the one after
    int64_t rs_n = 0;
    int len_n = 0;
    const int64_t k1 = k0 + R, k2 = k0 + 2 * (int64_t)R;
    if (lane < R && k1 + lane < end) {
      const int64_t row = w_nxt & 0x7fffffffu;
      rs_n = (int64_t)aip[row];
      len_n = (int)((int64_t)aip[row + 1] - rs_n);
    }
    const uint32_t w_n2 = (lane < R && k2 + lane < end) ? __ldg(prow + k2 + lane) : 0u;
    __syncwarp();
    // ---- gather + scatter into the tile
    IX cc[16];
    int gsel;
    if (lmax <= 4) {
      gsel = 4;
      scatter_rows<4>(desc, nrows, aix, av, tile, dp, lane, cc);
    } else if (lmax <= 8) {
      gsel = 8;
      scatter_rows<8>(desc, nrows, aix, av, tile, dp, lane, cc);
    } else {
      gsel = 16;
      scatter_rows<16>(desc, nrows, aix, av, tile, dp, lane, cc);
    }
    uint32_t longm = __ballot_sync(0xffffffffu, lane < nrows && len_cur > gsel);
    const uint32_t had_long = longm;
    while (longm) {  // rows longer than G: whole warp per row
      const int r = __ffs(longm) - 1;
      longm &= longm - 1;
      const int4 ds = desc[r];
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      for (int q = gsel + lane; q < ds.z; q += 32) {
        const TV v = __ldg(av + rs + q);
        tile[r * dp + (int)__ldg(aix + rs + q)] = ds.w ? -v : v;
      }
    }
    __syncwarp();
    // ---- accumulate the batch in row order
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
    if (gsel == 4)
      unscatter_rows<4>(desc, nrows, tile, dp, lane, cc);
    else if (gsel == 8)
      unscatter_rows<8>(desc, nrows, tile, dp, lane, cc);
    else
      unscatter_rows<16>(desc, nrows, tile, dp, lane, cc);
    for (uint32_t m = had_long; m; m &= m - 1) {
      const int r = __ffs(m) - 1;
      for (int c = lane; c < dp; c += 32) tile[r * dp + c] = (TV)0;
    }
    w_cur = w_nxt;
    rs_cur = rs_n;
    len_cur = len_n;
    w_nxt = w_n2;
  }
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
