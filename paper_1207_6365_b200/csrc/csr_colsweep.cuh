// csr_colsweep.cuh -- deterministic K4 for CSR A too wide for on-chip
// accumulators of whole SA rows (BASELINE config 5: d = 262,144 columns,
// t = 400 buckets -> 2 MB of fp64 per SA row), with sorted column indices per
// row (canonical CSR, as_csr's output).  Replaces sketch.py:155-164 for that
// shape; bit-identical: every SA element receives s_i * v in ascending row
// order from +0.0 (the reference's bincount order).
//
// Work item = one CTA per (bucket b, column block): the block's columns are
// swept in super-steps of kCsStep = 8192 columns whose fp64 accumulators live
// in shared memory (64 KB), warp w owning the 1024-column cell
// [cs + 1024 w, cs + 1024 (w + 1)).  Every row of the bucket keeps a cursor
// (first entry not yet consumed; global workspace, initialised per column
// block by csr_colsweep_init_kernel with a binary search).  Per super-step and
// group of <= kCsRG rows:
//   1. boundary pass: 16 lanes per row load the next 16 column indices from
//      the cursor; since a row's columns are sorted, the entries of cell w are
//      the contiguous run whose (col - cs) >> 10 == w, so the 8 run ends are
//      the lanes where that value changes (a row with more than 16 entries in
//      the super-step loads the next 16, rarely);
//   2. accumulate pass: warp w flattens its cell's runs over 32 rows at a
//      time (a row's run, then the next row's: ascending row order), loads
//      (col, val) and adds s_i * v into its accumulators; lanes that hit the
//      same column in one step (two rows of the bucket sharing it) are
//      serialised in lane = row order with __match_any_sync;
//   3. after the last group: the 8192 sums are written to SA row b (fp32 or
//      fp64 output, one rounding) and the accumulators re-zeroed.
// No global atomics; A is read once, SA written once.
#pragma once

#include <climits>

#include "common.cuh"

namespace skt {
namespace {

constexpr int kCsWarps = 8;
constexpr int kCsThreads = kCsWarps * 32;
constexpr int kCsCellShift = 10;                   // 1024 columns per warp cell
constexpr int kCsStep = kCsWarps << kCsCellShift;  // 8192 columns per super-step
constexpr int kCsRG = 1024;                        // rows per group
constexpr int kCsRowsPerWarp = kCsRG / kCsWarps;   // 128 (boundary pass)
constexpr int kCsBI = 16;                          // boundary iterations in flight
constexpr int kCsSteps = 8;                        // accumulate: 32-row steps per load batch

struct CsSmem {
  double acc[kCsStep];               // 64 KB
  int64_t rs[kCsRG];                 // row start (entry index); bit 63 = negative sign
  int32_t rlen[kCsRG];               // row length
  int32_t cur[kCsRG];                // cursor (relative to the row start) at the super-step start
  uint16_t ends[kCsRG][kCsWarps];    // end of cell w's run, relative to cur
};

// cursor[cb][p] = first entry of plan position p's row with column >= cb * blk_cols
template <typename IP, typename IX>
__global__ void __launch_bounds__(256) csr_colsweep_init_kernel(const uint32_t *__restrict__ prow, int64_t np,
                                                                int nblk, int64_t blk_cols,
                                                                const IP *__restrict__ aip,
                                                                const IX *__restrict__ aix,
                                                                int32_t *__restrict__ cursor) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np * nblk) return;
  const int cb = (int)(i / np);
  const int64_t p = i - (int64_t)cb * np;
  if (cb == 0) {
    cursor[i] = 0;
    return;
  }
  const int64_t row = __ldg(prow + p) & 0x7fffffffu;
  const int64_t rs = (int64_t)aip[row], re = (int64_t)aip[row + 1];
  const int64_t key = (int64_t)cb * blk_cols;
  int64_t lo = rs, hi = re;  // first index with col >= key
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(aix + mid) < key) lo = mid + 1; else hi = mid;
  }
  cursor[i] = (int32_t)(lo - rs);
}

template <typename IP, typename IX, typename TV, typename TOut>
__global__ void __launch_bounds__(kCsThreads, 2) csr_colsweep_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, int64_t np, uint64_t t,
    int nblk, int64_t blk_cols, int64_t d, const IP *__restrict__ aip, const IX *__restrict__ aix,
    const TV *__restrict__ av, int32_t *__restrict__ cursor, TOut *__restrict__ sa, int64_t ldsa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CsSmem &S = *reinterpret_cast<CsSmem *>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = blockIdx.x / nblk;
  const int cb = (int)(blockIdx.x - b * nblk);
  const int64_t c_lo = (int64_t)cb * blk_cols, c_hi = min(d, c_lo + blk_cols);
  const int64_t p0 = pindptr[b], p1 = pindptr[b + 1];
  const int64_t nr = p1 - p0;
  int32_t *gcur = cursor + (int64_t)cb * np + p0;
  const bool resident = nr <= kCsRG;

  for (int i = threadIdx.x; i < kCsStep; i += kCsThreads) S.acc[i] = 0.0;

  const int sl = lane & 15, half = lane >> 4;

  for (int64_t cs = c_lo; cs < c_hi; cs += kCsStep) {
    const int64_t ce = min(c_hi, cs + kCsStep);
    for (int64_t g0 = 0; g0 < max(nr, (int64_t)1); g0 += kCsRG) {
      const int ng = (int)min((int64_t)kCsRG, nr - g0);
      if (ng <= 0) break;
      // ---- row descriptors (once for a resident bucket) and cursors
      if (!resident || cs == c_lo) {
        __syncthreads();
        for (int r = threadIdx.x; r < ng; r += kCsThreads) {
          const uint32_t wd = __ldg(prow + p0 + g0 + r);
          const int64_t row = wd & 0x7fffffffu;
          const int64_t rs = (int64_t)aip[row];
          S.rs[r] = rs | ((int64_t)(wd >> 31) << 63);
          S.rlen[r] = (int32_t)((int64_t)aip[row + 1] - rs);
          S.cur[r] = gcur[g0 + r];
        }
        __syncthreads();
      }
      // ---- 1. boundary pass: run ends of the 8 cells per row; row pairs
      // interleaved over the warps (pair q -> warp q % 8), kCsBI pairs in flight
      const int npairs = (ng + 1) >> 1;
      for (int q0 = w; q0 < npairs; q0 += kCsWarps * kCsBI) {
        int cols[kCsBI];
#pragma unroll
        for (int it = 0; it < kCsBI; ++it) {
          const int r = 2 * (q0 + it * kCsWarps) + half;
          cols[it] = INT_MAX;
          if (r < ng) {
            const int c = S.cur[r] + sl;
            if (c < S.rlen[r]) cols[it] = (int)__ldg(aix + (S.rs[r] & 0x7fffffffffffffffLL) + c);
          }
        }
#pragma unroll
        for (int it = 0; it < kCsBI; ++it) {
          const int r = 2 * (q0 + it * kCsWarps) + half;
          if (q0 + it * kCsWarps >= npairs) break;  // warp-uniform
          bool active = r < ng;
          int col = cols[it], off = 0, prevc = 0;
          for (;;) {
            // cell of each loaded entry; 8 = beyond the super-step or the row
            // (the cursor sits on the first entry with col >= cs)
            const int k = (active && col < ce) ? (int)((col - cs) >> kCsCellShift) : kCsWarps;
            const int kp = __shfl_up_sync(0xffffffffu, k, 1);
            const int prev = sl == 0 ? prevc : kp;
            // cells [prev, k) end at this position (columns sorted in the row)
            if (active)
              for (int q = prev; q < k; ++q) S.ends[r][q] = (uint16_t)(off + sl);
            const int klast = __shfl_sync(0xffffffffu, k, (lane & 16) | 15);
            const bool cont = active && klast < kCsWarps;
            if (!__any_sync(0xffffffffu, cont)) break;
            // all 16 loaded entries inside the super-step: the next 16 (rare)
            active = cont;
            prevc = klast;
            off += 16;
            col = INT_MAX;
            if (active) {
              const int c = S.cur[r] + off + sl;
              if (c < S.rlen[r]) col = (int)__ldg(aix + (S.rs[r] & 0x7fffffffffffffffLL) + c);
            }
          }
        }
      }
      __syncthreads();
      // ---- 2. accumulate pass: warp w, cell [cs + 1024 w, ...).  Rows in
      // steps of 32 (lane = row), 8 steps at a time: the first two 32-entry
      // batches of every step are loaded before any is added (16 batches in
      // flight), longer steps continue unbatched; adds in step order.
      const int64_t cbase = cs + ((int64_t)w << kCsCellShift);
      double *acc = S.acc + (w << kCsCellShift);
      for (int rg = 0; rg < ng; rg += 32 * kCsSteps) {
        int excl[kCsSteps], tot[kCsSteps], curr[kCsSteps];
        bool one[kCsSteps], has1[kCsSteps];
        int64_t rsr[kCsSteps];
#pragma unroll
        for (int g = 0; g < kCsSteps; ++g) {
          const int r = rg + 32 * g + lane;
          int a = 0, cnt = 0;
          rsr[g] = 0;
          curr[g] = 0;
          if (r < ng) {
            a = w ? S.ends[r][w - 1] : 0;
            cnt = (int)S.ends[r][w] - a;
            rsr[g] = S.rs[r];
            curr[g] = S.cur[r] + a;
          }
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          excl[g] = incl - cnt;
          tot[g] = __shfl_sync(0xffffffffu, incl, 31);
          one[g] = __all_sync(0xffffffffu, cnt <= 1);
          has1[g] = cnt == 1;
        }
        // flattened entry f of step g -> (row lane j, entry index)
        auto locate = [&](int g, int f, int64_t &idx, bool &neg) {
          int j = 0;
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            const int e = __shfl_sync(0xffffffffu, excl[g], (j + step) & 31);
            if (j + step < 32 && e <= f) j += step;
          }
          const int64_t rsj = __shfl_sync(0xffffffffu, rsr[g], j);
          const int curj = __shfl_sync(0xffffffffu, curr[g], j);
          const int exj = __shfl_sync(0xffffffffu, excl[g], j);
          idx = (rsj & 0x7fffffffffffffffLL) + curj + (f - exj);
          neg = rsj < 0;
        };
        int kk[2 * kCsSteps];
        double vv[2 * kCsSteps];
#pragma unroll
        for (int g = 0; g < kCsSteps; ++g)
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int f = 32 * h2 + lane;
            kk[2 * g + h2] = -1 - lane;  // unique per lane when idle
            vv[2 * g + h2] = 0.0;
            if (h2 == 0 && one[g]) {
              // every row of the step has at most one entry in the cell: the
              // flattened order is the lane order, entry = the row's own
              if (has1[g]) {
                const int64_t idx = (rsr[g] & 0x7fffffffffffffffLL) + curr[g];
                kk[2 * g] = (int)((int64_t)__ldg(aix + idx) - cbase);
                const double v = (double)__ldg(av + idx);
                vv[2 * g] = rsr[g] < 0 ? -v : v;
              }
            } else if (32 * h2 < tot[g]) {  // warp-uniform
              int64_t idx;
              bool neg;
              locate(g, f, idx, neg);
              if (f < tot[g]) {
                kk[2 * g + h2] = (int)((int64_t)__ldg(aix + idx) - cbase);
                const double v = (double)__ldg(av + idx);
                vv[2 * g + h2] = neg ? -v : v;
              }
            }
          }
        auto add_batch = [&](int key, double v, bool has) {
          const uint32_t peers = __match_any_sync(0xffffffffu, key);
          if (__all_sync(0xffffffffu, peers == (1u << lane))) {
            if (has) acc[key] += v;
          } else {
            const int rank = __popc(peers & ((1u << lane) - 1u));
            const int rounds = __reduce_max_sync(0xffffffffu, has ? rank + 1 : 0);
            for (int q = 0; q < rounds; ++q) {
              if (has && rank == q) acc[key] += v;
              __syncwarp();
            }
          }
          __syncwarp();
        };
#pragma unroll
        for (int g = 0; g < kCsSteps; ++g) {
          if (one[g]) {  // lane = row; rows without an entry idle
            if (tot[g]) add_batch(kk[2 * g], vv[2 * g], kk[2 * g] >= 0);
            continue;
          }
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2)
            if (32 * h2 < tot[g]) add_batch(kk[2 * g + h2], vv[2 * g + h2], 32 * h2 + lane < tot[g]);
          for (int f0 = 64; f0 < tot[g]; f0 += 32) {  // long steps (dense cells), unbatched
            const int f = f0 + lane;
            int64_t idx;
            bool neg;
            locate(g, f, idx, neg);
            int key = -1 - lane;
            double v = 0.0;
            if (f < tot[g]) {
              key = (int)((int64_t)__ldg(aix + idx) - cbase);
              v = (double)__ldg(av + idx);
              if (neg) v = -v;
            }
            add_batch(key, v, f < tot[g]);
          }
        }
      }
      __syncthreads();
      // ---- cursors past this super-step
      for (int r = threadIdx.x; r < ng; r += kCsThreads) {
        const int nc = S.cur[r] + (int)S.ends[r][kCsWarps - 1];
        S.cur[r] = nc;
        if (!resident) gcur[g0 + r] = nc;
      }
    }
    __syncthreads();
    // ---- 3. SA row b, columns [cs, ce): one rounding, re-zero
    TOut *o = sa + b * ldsa + cs;
    const int ncol = (int)(ce - cs);
    for (int i = threadIdx.x; i < ncol; i += kCsThreads) {
      o[i] = (TOut)S.acc[i];
      S.acc[i] = 0.0;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace skt
