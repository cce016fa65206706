// csr_sweep.cuh -- K4 "sweep" kernel for canonical CSR with narrow d and rows
// of ~8+ nonzeros (BASELINE config 4 shape), over the bucket-GROUP plan.
//
// Why: csr_tile (warp per bucket) visits A's rows in bucket order; with t
// buckets in ~t/2960 waves every wave touches rows spread over all of A, so
// each row's ~64 B index / value segments are random DRAM accesses whose
// neighbouring sectors are fetched and thrown away (ncu: ~1.9x algorithmic
// DRAM bytes).  Here one warp owns a group of 2^shift consecutive buckets and
// walks the group's rows in ascending ROW order (K2's grouped plan); with all
// groups resident in one wave every warp advances through A at about the
// same rate, so the rows being read at any moment lie in a narrow window of
// A: sectors shared by adjacent rows (which belong to other groups) hit in L2
// and DRAM pages are read while open (tools/gather_bench.cu: windowed row
// order 0.174 ms vs 0.2435 ms random for config 4's pattern).
//
// Data path per batch of R rows (as csr_tile): the rows' nonzeros (G lanes per
// row) are scattered, signed, into a zeroed R x d tile in shared memory, then
// lane l adds tile[r][2l, 2l+1 (+64k)] into the fp64 register accumulators
// of the row's bucket (bucket-in-group from the plan's blo byte): bucket by
// bucket, each bucket's rows of the batch in ascending order.  Per SA element the additions therefore
// run over the bucket's rows in ascending row order from +0.0, and absent
// entries add +0.0 (an exact identity: the accumulator is never -0.0) --
// bit-identical to the reference's bincount.  While batch b is accumulated,
// batch b+1's nonzeros are in flight (one register set), b+2's descriptors
// and b+3's plan words.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "csr_tile.cuh"

namespace skt {
namespace {

constexpr int kSweepWarps = 4;

// per-warp shared memory: 2 descriptor slots, the R x dp tile, 2^shift x dp
// fp64 accumulators
__host__ __device__ inline size_t sweep_tile_bytes(int R, int dp, int tv_size) {
  return ((size_t)R * dp * tv_size + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t sweep_slice_bytes(int R, int dp, int tv_size) {
  return 2 * 32 * sizeof(int4) + sweep_tile_bytes(R, dp, tv_size);
}

// A batch's first G nonzeros of every row into registers (G lanes per row,
// RT*G/32 row steps), and their scatter (sign in bit 0 of the descriptor's .w)
template <int G, int RT, typename IX, typename TV>
__device__ __forceinline__ void sweep_load(const int4 *__restrict__ desc, int nrows, const IX *__restrict__ aix,
                                           const TV *__restrict__ av, int lane, IX (&cc)[RT / 2], TV (&vv)[RT / 2]) {
  constexpr int S = 32 / G, NI = RT * G / 32;
  const int g = lane / G, gl = lane % G;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
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
}
template <int G, int RT, typename IX, typename TV>
__device__ __forceinline__ void sweep_store(const int4 *__restrict__ desc, TV *tile, int dp, int lane,
                                            const IX (&cc)[RT / 2], const TV (&vv)[RT / 2]) {
  constexpr int S = 32 / G, NI = RT * G / 32;
  const int g = lane / G;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = i * S + g;
    if (cc[i] != (IX)-1) tile[r * dp + (int)cc[i]] = (desc[r].w & 1) ? -vv[i] : vv[i];
  }
}

template <typename IP, typename IX, typename TV, typename TOut, int kChunks, int RT, int SHIFT>
__global__ void __launch_bounds__(kSweepWarps * 32, RT == 16 ? (SHIFT == 1 ? 7 : 6) : 4) csr_sweep_kernel(
    const int64_t *__restrict__ gptr, const uint32_t *__restrict__ grow, const uint8_t *__restrict__ gblo,
    int64_t ngroups, uint64_t t, const IP *__restrict__ aip, const IX *__restrict__ aix,
    const TV *__restrict__ av, int d, int dp, TOut *__restrict__ sa, int64_t ldsa) {
  constexpr int R = RT;
  using V2 = typename std::conditional<sizeof(TV) == 4, float2, double2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t group = (int64_t)blockIdx.x * kSweepWarps + w;
  if (group >= ngroups) return;
  constexpr int GB = 1 << SHIFT;
  unsigned char *slice = smem_raw + (size_t)w * sweep_slice_bytes(R, dp, (int)sizeof(TV));
  int4 *descs = (int4 *)slice;  // [slot][row of the batch]: rs lo, rs hi, len, neg | blo << 1
  TV *tile = (TV *)(slice + 2 * 32 * sizeof(int4));
  for (int i = lane; i < R * dp; i += 32) tile[i] = (TV)0;
  double acc[GB][kChunks][2];
#pragma unroll
  for (int j = 0; j < GB; ++j)
#pragma unroll
    for (int k = 0; k < kChunks; ++k) acc[j][k][0] = acc[j][k][1] = 0.0;

  const int64_t beg = gptr[group], end = gptr[group + 1];
  auto plan_word = [&](int64_t k0, uint32_t &bl) -> uint32_t {
    bl = 0;
    if (lane < R && k0 + lane < end) {
      bl = __ldg(gblo + k0 + lane);
      return __ldg(grow + k0 + lane);
    }
    return 0u;
  };
  auto row_desc = [&](int64_t k0, uint32_t wd, int64_t &rs, int &len) {
    rs = 0;
    len = 0;
    if (lane < R && k0 + lane < end) {
      const int64_t row = wd & 0x7fffffffu;
      rs = (int64_t)aip[row];
      len = (int)((int64_t)aip[row + 1] - rs);
    }
  };
  auto publish = [&](int slot, int64_t k0, int64_t rs, int len, uint32_t wd, uint32_t bl) -> int {
    const int nrows = (int)((end - k0) < R ? (end - k0) : R);
    if (lane < nrows)
      descs[slot * 32 + lane] = make_int4((int)(uint32_t)rs, (int)(rs >> 32), len, (int)((wd >> 31) | (bl << 1)));
    return tile_g(__reduce_max_sync(0xffffffffu, lane < nrows ? len : 0));
  };
  auto load_sw = [&](int G, const int4 *dsc, int nrows, IX (&c)[RT / 2], TV (&v)[RT / 2]) {
    if (G == 4)
      sweep_load<4, RT>(dsc, nrows, aix, av, lane, c, v);
    else if (G == 8)
      sweep_load<8, RT>(dsc, nrows, aix, av, lane, c, v);
    else
      sweep_load<16, RT>(dsc, nrows, aix, av, lane, c, v);
  };

  uint32_t b0, b1, b2;
  uint32_t w0 = plan_word(beg, b0);
  int64_t rs0;
  int len0;
  row_desc(beg, w0, rs0, len0);
  uint32_t w1 = plan_word(beg + R, b1);
  int64_t rs1;
  int len1;
  row_desc(beg + R, w1, rs1, len1);
  uint32_t w2 = plan_word(beg + 2 * (int64_t)R, b2);
  int slot = 0;
  IX cc[RT / 2];
  TV vv[RT / 2];
  int g0 = publish(slot, beg, rs0, len0, w0, b0);
  __syncwarp();
  load_sw(g0, descs + slot * 32, (int)((end - beg) < R ? (end - beg) : R), cc, vv);
  for (int64_t k0 = beg; k0 < end; k0 += R) {
    const int nrows = (int)((end - k0) < R ? (end - k0) : R);
    const int4 *dcur = descs + slot * 32;
    const int64_t k1 = k0 + R, k2 = k0 + 2 * (int64_t)R, k3 = k0 + 3 * (int64_t)R;
    // ---- scatter batch b (the sign is in bit 0 of .w)
    if (g0 == 4)
      sweep_store<4, RT>(dcur, tile, dp, lane, cc, vv);
    else if (g0 == 8)
      sweep_store<8, RT>(dcur, tile, dp, lane, cc, vv);
    else
      sweep_store<16, RT>(dcur, tile, dp, lane, cc, vv);
    uint32_t longm = __ballot_sync(0xffffffffu, lane < nrows && len0 > g0);
    while (longm) {  // rows longer than G: whole warp per row
      const int r = __ffs(longm) - 1;
      longm &= longm - 1;
      const int4 ds = dcur[r];
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      for (int q = g0 + lane; q < ds.z; q += 32) {
        const TV v = __ldg(av + rs + q);
        tile[r * dp + (int)__ldg(aix + rs + q)] = (ds.w & 1) ? -v : v;
      }
    }
    // ---- batch b+1 in flight, descriptors of b+2, plan words of b+3
    int g1 = 4;
    if (k1 < end) {
      g1 = publish(slot ^ 1, k1, rs1, len1, w1, b1);
      __syncwarp();
      load_sw(g1, descs + (slot ^ 1) * 32, (int)((end - k1) < R ? (end - k1) : R), cc, vv);
    }
    int64_t rs2;
    int len2;
    row_desc(k2, w2, rs2, len2);
    uint32_t b3;
    const uint32_t w3 = plan_word(k3, b3);
    __syncwarp();
    // ---- accumulate batch b: bucket by bucket (accumulators in registers),
    // each bucket's rows in ascending row order
    const uint32_t blr = lane < nrows ? (uint32_t)(dcur[lane].w >> 1) : 0xffu;
#pragma unroll
    for (int j = 0; j < GB; ++j) {
      for (uint32_t m = __ballot_sync(0xffffffffu, blr == (uint32_t)j); m; m &= m - 1) {
        const int r = __ffs(m) - 1;
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = 64 * k + 2 * lane;
          if (c < dp) {
            const V2 x = *reinterpret_cast<const V2 *>(tile + r * dp + c);
            acc[j][k][0] += (double)x.x;
            acc[j][k][1] += (double)x.y;
          }
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
    __syncwarp();
    g0 = g1;
    len0 = len1;
    rs1 = rs2;
    len1 = len2;
    w1 = w2;
    b1 = b2;
    w2 = w3;
    b2 = b3;
    slot ^= 1;
  }
#pragma unroll
  for (int j = 0; j < GB; ++j) {
    const uint64_t bucket = (uint64_t)group * GB + j;
    if (bucket < t) {
      TOut *o = sa + bucket * ldsa;
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = 64 * k + 2 * lane;
        if (c < d) o[c] = (TOut)acc[j][k][0];
        if (c + 1 < d) o[c + 1] = (TOut)acc[j][k][1];
      }
    }
  }
}

}  // namespace
}  // namespace skt
