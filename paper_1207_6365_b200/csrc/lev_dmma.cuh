// lev_dmma.cuh -- K5 (leverage.py:87-91: rows = A @ probe, scores = squared
// row norms) for fp64 CSR A on the fp64 tensor cores: the path the reference
// API takes (as_csr upcasts fp32 values to fp64, _validation.py:30-41).
//
// A CTA owns 128-row tiles of A (persistent over tiles).  A tile is densified
// into shared memory directly in DMMA fragment order -- for 8-row block mb and
// 4-column step ks, the 32 doubles a warp's mma.sync.m8n8k4 A operand reads,
// lane = (row & 7) * 4 + (col & 3) -- so the operand load is one conflict-free
// LDS.64 per lane.  The probe (d x k, d <= 64, k = 8 * NB) stays in registers
// as B fragments for the whole kernel: warp w covers n-blocks of half
// (w & 1) for m-blocks 4 (w >> 1) .. 4 (w >> 1) + 3, so every A fragment feeds
// NB / 2 DMMAs.  Epilogue: squares of the fp64 accumulators, quad shuffle
// reduction, the two halves summed through shared memory.  Zero entries of
// the densified tile add exact zeros (finite probe), so the products equal
// the sparse row's within fp64 rounding (tolerance 1e-12 relative, the
// north-star bar; the reference's own BLAS order is unspecified).
// Duplicate column indices inside a row (non-canonical CSR) are summed in
// stored order by one lane before the tile is used.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

constexpr int kDmRows = 128;
constexpr int kDmWarps = 16;  // warps 0-7: DMMA + epilogue, warps 8-15: densify
constexpr int kDmThreads = kDmWarps * 32;

__device__ __forceinline__ void dmma_m8n8k4(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void nbar_sync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ bool nbar_or(int id, int cnt, bool v) {
  int r;
  asm volatile("{ .reg .pred p, q; setp.ne.s32 p, %1, 0; bar.red.or.pred q, %2, %3, p; selp.s32 %0, 1, 0, q; }"
               : "=r"(r)
               : "r"((int)v), "r"(id), "r"(cnt)
               : "memory");
  return r != 0;
}
// named barriers: 1, 2 = tile buffer s full; 3, 4 = buffer s empty;
// 5, 6 = densify group s; 7 = DMMA warps.  Densify group s (4 warps, 32 rows
// each) fills buffer s with tiles j = s, s + 2, ... (two tiles in flight)
constexpr int kBarFull = 1, kBarEmpty = 3, kBarProd = 5, kBarCons = 7;
constexpr int kDmGroupThreads = 128;
constexpr int kDmIters = 16;  // 32 rows per densify warp, two per iteration

// shared memory: two densified tiles (16 m-blocks x KS k-steps x 32 doubles)
// and 2 x 128 x 2 partial scores
template <int KS>
__host__ __device__ constexpr size_t dmma_tile_doubles() {
  return (size_t)(kDmRows / 8) * KS * 32;
}
template <int KS>
__host__ __device__ constexpr size_t dmma_smem() {
  return (2 * dmma_tile_doubles<KS>() + 2 * kDmRows * 2) * sizeof(double);
}

template <typename IX>
__device__ __forceinline__ int frag_pos(int trow, IX c, int KS) {
  return ((trow >> 3) * KS + ((int)c >> 2)) * 32 + ((trow & 7) << 2 | ((int)c & 3));
}

// One densify group (4 warps) fills a tile buffer.  (rs_l, re_l): row range
// of row 32 pw + lane of this tile, loaded one tile ahead by the caller.
template <typename IP, typename IX, typename TV, int KS>
__device__ __forceinline__ void dmma_densify(double *tile, int64_t r0, int64_t n, int pw, int lane, int bar,
                                             int64_t rs_l, int64_t re_l, const IP *__restrict__ aip,
                                             const IX *__restrict__ aix, const TV *__restrict__ av) {
  const int sl = lane & 15, hf = lane >> 4;
  // the first 16 entries of every row of the warp in flight at once (issued
  // before the zeroing so their latency overlaps it)
  IX cc[kDmIters];
  TV vv[kDmIters];
#pragma unroll
  for (int it = 0; it < kDmIters; ++it) {
    const int lr = 2 * it + hf;
    const int64_t rs = __shfl_sync(0xffffffffu, rs_l, lr), re = __shfl_sync(0xffffffffu, re_l, lr);
    cc[it] = (IX)-1;
    vv[it] = (TV)0;
    if (rs + sl < re) {
      cc[it] = __ldg(aix + rs + sl);
      vv[it] = __ldg(av + rs + sl);
    }
  }
  {
    double2 *z = reinterpret_cast<double2 *>(tile);
    for (int i = pw * 32 + lane; i < (kDmRows / 8) * KS * 16; i += kDmGroupThreads) z[i] = make_double2(0.0, 0.0);
  }
  nbar_sync(bar, kDmGroupThreads);
  bool dirty = false;
#pragma unroll
  for (int it = 0; it < kDmIters; ++it) {
    const int trow = 32 * pw + 2 * it + hf;
    // canonical check: strictly increasing columns inside the row
    const IX prevc = __shfl_up_sync(0xffffffffu, cc[it], 1);
    if (sl > 0 && cc[it] != (IX)-1 && !(cc[it] > prevc)) dirty = true;
    if (cc[it] != (IX)-1) tile[frag_pos(trow, cc[it], KS)] = (double)vv[it];
  }
  // rows longer than 16 entries (config 4: the 1% dense rows): the whole warp
  // per row, entries 16 .. 79 in flight at once, longer rows loop
  for (uint32_t m = __ballot_sync(0xffffffffu, re_l - rs_l > 16); m; m &= m - 1) {
    const int lr = __ffs(m) - 1, trow = 32 * pw + lr;
    const int64_t rs = __shfl_sync(0xffffffffu, rs_l, lr), re = __shfl_sync(0xffffffffu, re_l, lr);
    for (int64_t p0 = rs + 16; p0 < re; p0 += 64) {
      const int64_t pa = p0 + lane, pb = p0 + 32 + lane;
      IX ca = (IX)-1, cb = (IX)-1, prev = (IX)-1;
      TV va = 0, vb = 0;
      if (pa < re) {
        ca = __ldg(aix + pa);
        va = __ldg(av + pa);
        prev = __ldg(aix + pa - 1);
      }
      if (pb < re) {
        cb = __ldg(aix + pb);
        vb = __ldg(av + pb);
      }
      const IX prevb = __shfl_up_sync(0xffffffffu, cb, 1);
      const IX ca31 = __shfl_sync(0xffffffffu, ca, 31);
      if (ca != (IX)-1 && !(ca > prev)) dirty = true;
      if (cb != (IX)-1 && !(cb > (lane == 0 ? ca31 : prevb))) dirty = true;
      if (ca != (IX)-1) tile[frag_pos(trow, ca, KS)] = (double)va;
      if (cb != (IX)-1) tile[frag_pos(trow, cb, KS)] = (double)vb;
    }
  }
  // non-canonical rows (duplicate or unsorted columns): rebuilt in stored
  // order, one lane per row, duplicates summed
  if (nbar_or(bar, kDmGroupThreads, dirty)) {
    if (r0 + 32 * pw + lane < n) {
      const int trow = 32 * pw + lane;
      for (int64_t p = rs_l; p < re_l; ++p) tile[frag_pos(trow, __ldg(aix + p), KS)] = 0.0;
      for (int64_t p = rs_l; p < re_l; ++p) tile[frag_pos(trow, __ldg(aix + p), KS)] += (double)__ldg(av + p);
    }
  }
}

template <typename IP, typename IX, typename TV, typename TS, int KS, int NB>
__global__ void __launch_bounds__(kDmThreads, 1) lev_dmma_kernel(int64_t n, int d, const IP *__restrict__ aip,
                                                                  const IX *__restrict__ aix,
                                                                  const TV *__restrict__ av,
                                                                  const double *__restrict__ probe, int k,
                                                                  TS *__restrict__ scores) {
  static_assert(NB % 2 == 0, "k must be a multiple of 16");
  constexpr int NBW = NB / 2;
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t ntiles = (n + kDmRows - 1) / kDmRows;

  if (w >= 8) {  // ---------------- densify groups (producers)
    const int s = (w - 8) >> 2, pw = (w - 8) & 3;
    auto rows_of = [&](int64_t ti, int64_t &rs, int64_t &re) {
      rs = re = 0;
      const int64_t r = ti * kDmRows + 32 * pw + lane;
      if (ti < ntiles && r < n) {
        rs = (int64_t)aip[r];
        re = (int64_t)aip[r + 1];
      }
    };
    int64_t rs_l, re_l;
    rows_of(blockIdx.x + (int64_t)s * gridDim.x, rs_l, re_l);
    for (int64_t tile_i = blockIdx.x + (int64_t)s * gridDim.x; tile_i < ntiles; tile_i += 2 * (int64_t)gridDim.x) {
      int64_t rs_n, re_n;  // the group's next tile, one tile ahead
      rows_of(tile_i + 2 * (int64_t)gridDim.x, rs_n, re_n);
      nbar_sync(kBarEmpty + s, kDmGroupThreads + 256);  // the DMMA warps released buffer s
      dmma_densify<IP, IX, TV, KS>(dsm + s * dmma_tile_doubles<KS>(), tile_i * kDmRows, n, pw, lane, kBarProd + s,
                                   rs_l, re_l, aip, aix, av);
      nbar_arrive(kBarFull + s, kDmGroupThreads + 256);
      rs_l = rs_n;
      re_l = re_n;
    }
    return;
  }
  // ---------------- DMMA warps (consumer)
  const int nh = w & 1, ms = w >> 1;
  double *part = dsm + 2 * dmma_tile_doubles<KS>();
  // B fragments (probe rows 4 ks + (lane & 3), column 8 nb + (lane >> 2)), zero past d
  double b[NBW][KS];
#pragma unroll
  for (int jj = 0; jj < NBW; ++jj)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int r = 4 * ks + (lane & 3), c = 8 * (nh * NBW + jj) + (lane >> 2);
      b[jj][ks] = r < d ? __ldg(probe + (int64_t)r * k + c) : 0.0;
    }
  nbar_arrive(kBarEmpty + 0, kDmGroupThreads + 256);  // both buffers start empty
  nbar_arrive(kBarEmpty + 1, kDmGroupThreads + 256);
  int j = 0;
  for (int64_t tile_i = blockIdx.x; tile_i < ntiles; tile_i += gridDim.x, ++j) {
    const int s = j & 1;
    const double *tile = dsm + s * dmma_tile_doubles<KS>();
    nbar_sync(kBarFull + s, kDmGroupThreads + 256);
    double acc[4][NBW][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int jj = 0; jj < NBW; ++jj) acc[m][jj][0] = acc[m][jj][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double a = tile[((4 * ms + m) * KS + ks) * 32 + lane];
#pragma unroll
        for (int jj = 0; jj < NBW; ++jj) dmma_m8n8k4(acc[m][jj][0], acc[m][jj][1], a, b[jj][ks]);
      }
    nbar_arrive(kBarEmpty + s, kDmGroupThreads + 256);  // buffer s free for tile j + 2
    // epilogue: sum of squares per row (row = 8 mb + lane / 4)
    double *pp = part + s * kDmRows * 2;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      double sq = 0.0;
#pragma unroll
      for (int jj = 0; jj < NBW; ++jj) sq += acc[m][jj][0] * acc[m][jj][0] + acc[m][jj][1] * acc[m][jj][1];
      sq += __shfl_xor_sync(0xffffffffu, sq, 1);
      sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      if ((lane & 3) == 0) pp[(8 * (4 * ms + m) + (lane >> 2)) * 2 + nh] = sq;
    }
    nbar_sync(kBarCons, 256);
    const int64_t r0 = tile_i * kDmRows;
    if (threadIdx.x < kDmRows && r0 + threadIdx.x < n)
      scores[r0 + threadIdx.x] = (TS)(pp[2 * threadIdx.x] + pp[2 * threadIdx.x + 1]);
  }
}

}  // namespace
}  // namespace skt
