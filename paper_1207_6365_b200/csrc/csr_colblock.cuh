// csr_colblock.cuh -- deterministic K4 for canonical CSR A whose SA rows are
// too wide for on-chip accumulators (BASELINE config 5: d = 262,144, t = 400),
// replacing sketch.py:155-164 for that shape, bit-identical: every SA element
// is the fp64 sum of s_i * v over the bucket's rows in ascending row order
// from +0.0 (the reference's bincount order).
//
// 1. csr_colblock_bounds_kernel (one streaming read of the column indices):
//    for every row, the offsets of its first entry in each 16384-column block
//    (the row's columns are sorted, so a block's entries are one run).
// 2. csr_colblock_kernel, one CTA per (bucket b, column block q), fp64
//    accumulators of the block's 16384 columns in shared memory (128 KB):
//    a. count: every entry of the bucket's rows inside the block sets its
//       column in three bitmaps (seen once / twice / three times or more);
//    b. add: a column seen once gets a plain store of s_i * v (0 + x = x),
//       a column seen twice two fp64 adds from +0.0 in either order
//       (fl(fl(0 + x) + y) = fl(x + y) = fl(y + x): IEEE addition is
//       commutative), so neither needs the row order; entries of columns
//       seen three or more times are appended to a list with their row rank;
//    c. the list (~3% of the columns for config 5) is sorted by (column,
//       rank) with a block radix sort and each column's entries are summed
//       in rank order by one thread -- the reference's order exactly;
//    d. the block's SA columns are written once (0 where nothing landed).
//    Lists that overflow shared memory, or buckets of 2^17+ rows, take an
//    ordered single-warp sweep for the columns seen three or more times.
// No global atomics; A is read twice (boundaries: indices only), SA once.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

constexpr int kCbShift = 14;
constexpr int kCbCols = 1 << kCbShift;  // 16384 columns per block
constexpr int kCbThreads = 512;
constexpr int kBndBatch = 9;  // bounds kernel: 288 column indices of a row in flight
constexpr int kCbList = 2048;                   // entries of columns with >= 3 contributions
constexpr int kCbChain = 32;                    // longest per-column chain sorted in registers
constexpr int kCbRows = 2048;                   // row descriptors staged per chunk
constexpr int kCbUnroll = 8;                    // row pairs per warp with loads in flight

// bnd[row * (nblk - 1) + (q - 1)] = offset (relative to the row start) of the
// row's first entry with column >= q * 16384, q = 1 .. nblk - 1
template <typename IP, typename IX>
__global__ void __launch_bounds__(256) csr_colblock_bounds_kernel(int64_t n, int nblk, const IP *__restrict__ aip,
                                                                   const IX *__restrict__ aix,
                                                                   int32_t *__restrict__ bnd) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nb1 = nblk - 1;
  for (int64_t row = warp; row < n; row += nwarps) {
    const int64_t rs = (int64_t)aip[row], re = (int64_t)aip[row + 1];
    int32_t *o = bnd + row * nb1;
    int prevq = 0;  // block of the entry before this lane's
    for (int64_t b0 = rs; b0 < re; b0 += 32 * kBndBatch) {
      int qs[kBndBatch];  // kBndBatch x 32 column indices in flight
#pragma unroll
      for (int j = 0; j < kBndBatch; ++j) {
        const int64_t p = b0 + 32 * j + lane;
        qs[j] = p < re ? (int)((int64_t)__ldg(aix + p) >> kCbShift) : nblk;
      }
#pragma unroll
      for (int j = 0; j < kBndBatch; ++j) {
        if (b0 + 32 * j >= re) break;  // warp-uniform
        const int64_t p = b0 + 32 * j + lane;
        const int q = qs[j];
        const int qp = __shfl_up_sync(0xffffffffu, q, 1);
        const int prev = lane == 0 ? prevq : qp;
        // blocks (prev, q] start at this entry
        for (int k = max(prev + 1, 1); k <= min(q, nb1); ++k) o[k - 1] = (int32_t)(p - rs);
        prevq = __shfl_sync(0xffffffffu, q, 31);
      }
    }
    // blocks after the row's last entry start at its end
    for (int k = max(prevq + 1, 1) + lane; k <= nb1; k += 32) o[k - 1] = (int32_t)(re - rs);
  }
}

struct CbSmem {
  double acc[kCbCols];            // 128 KB
  uint32_t seen[3][kCbCols / 32]; // >= 1, >= 2, >= 3 contributions
  uint32_t lrank[kCbList];        // row rank inside the bucket
  int32_t lnext[kCbList];         // per-column chains (heads kept in acc[c])
  double lval[kCbList];
  int64_t es[kCbRows];            // first entry in the block (bit 63: negative sign)
  int32_t len[kCbRows];           // entries in the block
  int count;
  int overflow;
};

template <typename IP, typename IX, typename TV, typename TOut>
__global__ void __launch_bounds__(kCbThreads, 1) csr_colblock_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, int nblk, int64_t d,
    const IP *__restrict__ aip, const IX *__restrict__ aix, const TV *__restrict__ av,
    const int32_t *__restrict__ bnd, TOut *__restrict__ sa, int64_t ldsa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CbSmem &S = *reinterpret_cast<CbSmem *>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t b = blockIdx.x / nblk;
  const int q = (int)(blockIdx.x - b * nblk);
  const int64_t c0 = (int64_t)q << kCbShift;
  const int ncols = (int)min((int64_t)kCbCols, d - c0);
  const int64_t p0 = pindptr[b], p1 = pindptr[b + 1];
  const int64_t nr = p1 - p0;
  const int nb1 = nblk - 1;

  for (int i = tid; i < 3 * kCbCols / 32; i += kCbThreads) (&S.seen[0][0])[i] = 0u;
  if (tid == 0) {
    S.count = 0;
    S.overflow = nr >= (1LL << 31);
  }
  __syncthreads();

  const int sl = lane & 15, hf = lane >> 4;
  // the block's entry range of plan position p (absolute entry indices), sign
  auto row_range = [&](int64_t p, int64_t &es, int64_t &ee, bool &neg) {
    const uint32_t wd = __ldg(prow + p);
    const int64_t row = wd & 0x7fffffffu;
    const int64_t rs = (int64_t)aip[row];
    es = rs + (q == 0 ? 0 : (int64_t)__ldg(bnd + row * nb1 + (q - 1)));
    ee = q == nb1 ? (int64_t)aip[row + 1] : rs + (int64_t)__ldg(bnd + row * nb1 + q);
    neg = (wd >> 31) != 0;
  };
  // stage the descriptors of rows [g0, g0 + ng) of the bucket (all loads in flight)
  auto stage = [&](int64_t g0, int ng) {
    for (int r = tid; r < ng; r += kCbThreads) {
      int64_t es, ee;
      bool neg;
      row_range(p0 + g0 + r, es, ee, neg);
      S.es[r] = es | ((int64_t)neg << 63);
      S.len[r] = (int32_t)(ee - es);
    }
  };
  // visit every entry of the staged rows: warp w takes row pairs w, w + 16, ..;
  // kCbUnroll pairs with their first 16 entries loaded before use
  auto sweep = [&](int ng, bool vals, auto &&body) {
    for (int pr0 = 2 * w; pr0 < ng; pr0 += 2 * (kCbThreads / 32) * kCbUnroll) {
      int cc[kCbUnroll][2];
      double vv[kCbUnroll][2];
#pragma unroll
      for (int u = 0; u < kCbUnroll; ++u) {
        const int r = pr0 + 2 * (kCbThreads / 32) * u + hf;
        const int L = r < ng ? S.len[r] : 0;
        const int64_t e = r < ng ? (S.es[r] & 0x7fffffffffffffffLL) : 0;
        const bool ng_ = r < ng && S.es[r] < 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          cc[u][h] = -1;
          vv[u][h] = 0.0;
          if (sl + 16 * h < L) {
            cc[u][h] = (int)((int64_t)__ldg(aix + e + sl + 16 * h) - c0);
            if (vals) {
              const double v = (double)__ldg(av + e + sl + 16 * h);
              vv[u][h] = ng_ ? -v : v;
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kCbUnroll; ++u) {
        const int r = pr0 + 2 * (kCbThreads / 32) * u + hf;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (cc[u][h] >= 0) body(cc[u][h], vv[u][h], r);
        // rows with more than 32 entries in the block: the rest
        const int L = r < ng ? S.len[r] : 0;
        for (int k = 32 + sl; __any_sync(0xffffffffu, k < L); k += 16) {
          if (k < L) {
            const int64_t e = S.es[r] & 0x7fffffffffffffffLL;
            const int c = (int)((int64_t)__ldg(aix + e + k) - c0);
            double v = 0.0;
            if (vals) {
              v = (double)__ldg(av + e + k);
              if (S.es[r] < 0) v = -v;
            }
            body(c, v, r);
          }
        }
      }
    }
  };
  const bool one_chunk = nr <= kCbRows;
  // ---- a. count contributions per column
  for (int64_t g0 = 0; g0 < nr; g0 += kCbRows) {
    const int ng = (int)min((int64_t)kCbRows, nr - g0);
    __syncthreads();
    stage(g0, ng);
    __syncthreads();
    sweep(ng, false, [&](int c, double, int) {
      const uint32_t m = 1u << (c & 31);
      if (atomicOr(&S.seen[0][c >> 5], m) & m)
        if (atomicOr(&S.seen[1][c >> 5], m) & m) atomicOr(&S.seen[2][c >> 5], m);
    });
  }
  __syncthreads();
  // columns seen exactly twice start from +0.0 (two order-free adds); columns
  // seen three or more times hold the head of their entry chain (-1: empty)
  for (int i = tid; i < kCbCols / 32; i += kCbThreads) {
    uint32_t m = S.seen[1][i];
    const uint32_t m3 = S.seen[2][i];
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      if (m3 & (1u << bit))
        reinterpret_cast<long long *>(S.acc)[32 * i + bit] = -1LL;
      else
        S.acc[32 * i + bit] = 0.0;
    }
  }
  // ---- b. order-free stores / adds; list the columns seen three or more times
  for (int64_t g0 = 0; g0 < nr; g0 += kCbRows) {
    const int ng = (int)min((int64_t)kCbRows, nr - g0);
    __syncthreads();
    if (!one_chunk) stage(g0, ng);
    __syncthreads();
    sweep(ng, true, [&](int c, double v, int r) {
      const uint32_t m = 1u << (c & 31);
      if (!(S.seen[1][c >> 5] & m)) {
        S.acc[c] = v + 0.0;  // the reference's 0.0 + v (maps -0.0 to +0.0)
      } else if (!(S.seen[2][c >> 5] & m)) {
        atomicAdd(&S.acc[c], v);  // two adds from +0.0: order-free
      } else {
        const int slot = atomicAdd(&S.count, 1);
        if (slot < kCbList) {
          S.lrank[slot] = (uint32_t)(g0 + r);
          S.lval[slot] = v;
          S.lnext[slot] = (int32_t)atomicExch(reinterpret_cast<unsigned long long *>(S.acc) + c, (unsigned long long)slot);
        }
      }
    });
  }
  __syncthreads();
  const int cnt = S.count;
  if (cnt > kCbList) S.overflow = 1;  // read below after the barrier
  __syncthreads();
  // ---- c. columns seen three or more times: walk the column's chain, sort
  // its entries by row rank (insertion sort in registers), add from +0.0
  if (!S.overflow && cnt > 0) {
    for (int i = tid; i < kCbCols / 32; i += kCbThreads) {
      uint32_t m = S.seen[2][i];
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        const int c = 32 * i + bit;
        uint32_t rk[kCbChain];
        double vl[kCbChain];
        int k = 0;
        for (int e = (int)reinterpret_cast<long long *>(S.acc)[c]; e >= 0; e = S.lnext[e]) {
          if (k == kCbChain) {
            k = -1;
            break;
          }
          const uint32_t r = S.lrank[e];
          const double v = S.lval[e];
          int j = k++;
          while (j > 0 && rk[j - 1] > r) {
            rk[j] = rk[j - 1];
            vl[j] = vl[j - 1];
            --j;
          }
          rk[j] = r;
          vl[j] = v;
        }
        if (k < 0) {
          S.overflow = 1;  // a chain longer than kCbChain: ordered sweep below
          continue;
        }
        double sum = 0.0;
        for (int j = 0; j < k; ++j) sum += vl[j];
        S.acc[c] = sum;
      }
    }
  }
  __syncthreads();
  if (S.overflow) {
    // fallback: one warp sweeps the bucket's rows in order, adding the
    // entries of columns seen three or more times from +0.0
    for (int i = tid; i < kCbCols / 32; i += kCbThreads) {
      uint32_t m = S.seen[2][i];
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        S.acc[32 * i + bit] = 0.0;
      }
    }
    __syncthreads();
    // fallback: one warp sweeps the bucket's rows in order, adding the
    // entries of columns seen three or more times (acc is +0.0 there)
    if (w == 0) {
      for (int64_t pp = 0; pp < nr; ++pp) {
        int64_t es, ee;
        bool neg;
        row_range(p0 + pp, es, ee, neg);
        for (int64_t e = es + lane; e < ee; e += 32) {
          const int c = (int)((int64_t)__ldg(aix + e) - c0);
          if (S.seen[2][c >> 5] & (1u << (c & 31))) {
            const double v = (double)__ldg(av + e);
            S.acc[c] += neg ? -v : v;  // distinct columns inside a row: no clash
          }
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // ---- d. the block's SA columns, one rounding
  TOut *o = sa + b * ldsa + c0;
  for (int i = tid; i < ncols; i += kCbThreads)
    o[i] = (S.seen[0][i >> 5] & (1u << (i & 31))) ? (TOut)S.acc[i] : (TOut)0;
}

}  // namespace
}  // namespace skt
