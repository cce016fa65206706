// csr_partition.cuh -- deterministic K4 for canonical CSR A with very wide SA
// rows (BASELINE config 5), without per-row work in the accumulate stage
// (sketch.py:155-164, bit-identical):
//
//   the bucket's rows (plan order = ascending row) are cut into pieces of
//   <= 512 rows; P1 counts pieces and stored entries per piece, P2 scans them;
//   P3 (CTA per piece) writes the piece's entries to the workspace ordered by
//      (16384-column block, row, column): per row, the entries of one block
//      are one contiguous run (columns sorted), so each row contributes
//      ~16-entry runs; the run lengths are counted by the CTA itself (run
//      starts of each 32-entry batch), scanned over the piece's rows per block;
//      keys are the column inside the block (uint16), values s_i * v;
//   P4 (CTA per (bucket, block)) walks the bucket's pieces in order -- their
//      block-q regions concatenated are the block's entries in ascending row
//      order -- twice with coalesced loads: contribution bitmaps, then
//      order-free stores / adds for columns with <= 2 contributions (IEEE
//      addition is commutative: fl(0 + x) + y = y + x) and per-column chains for
//      columns with >= 3, each chain sorted by position (= row order) and summed
//      from +0.0 -- the reference's order exactly.  Overflowing lists / long
//      chains: one warp sweeps the block in order for those columns.
// No global atomics.  Needs <= 32 column blocks (d <= 524,288).
#pragma once

#include "common.cuh"
#include "csr_colblock.cuh"

namespace skt {
namespace {

constexpr int kPtThreads = 512;
constexpr int kPtPiece = 512;  // rows per piece
constexpr int kPtBatch = 9;    // P3: 32-entry groups of a row in flight (config 5: a whole row)
constexpr int kPtItems = 8;    // P4: consecutive entries per thread per sweep step
constexpr int kPaThreads = 1024;  // P4 threads
constexpr int kPtPieceTab = 32;   // P4 register path: buckets of <= 32 pieces (16 K rows)
constexpr int kPtMaxBlocks = 32;

// P1a: pieces per bucket
__global__ void csr_part_npieces_kernel(const int64_t *__restrict__ pindptr, uint64_t t, int64_t *__restrict__ np) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < (int64_t)t) np[b] = (pindptr[b + 1] - pindptr[b] + kPtPiece - 1) / kPtPiece;
}

// exclusive scan of `cnt` values (one CTA, chunks of 1024); out[cnt] = total
__global__ void __launch_bounds__(1024) csr_part_scan_kernel(const int64_t *__restrict__ in, int64_t cnt,
                                                             int64_t *__restrict__ out) {
  __shared__ int64_t warp_sums[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < cnt; c0 += 1024) {
    const int64_t i = c0 + tid;
    const int64_t v = i < cnt ? in[i] : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t ws = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      warp_sums[lane] = ws;  // inclusive
    }
    __syncthreads();
    const int64_t before = carry + (w ? warp_sums[w - 1] : 0) + x - v;
    if (i < cnt) out[i] = before;
    __syncthreads();
    if (tid == 1023) carry = before + v;
    __syncthreads();
  }
  if (tid == 0) out[cnt] = carry;
}

// piece j -> bucket (last b with pstart[b] <= j)
__device__ __forceinline__ int64_t piece_bucket(const int64_t *__restrict__ pstart, uint64_t t, int64_t j) {
  int64_t lo = 0, hi = (int64_t)t;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (pstart[mid] <= j) lo = mid; else hi = mid;
  }
  return lo;
}

// P1b: stored entries per piece (warp per piece)
template <typename IP>
__global__ void __launch_bounds__(256) csr_part_piece_nnz_kernel(const int64_t *__restrict__ pindptr,
                                                                 const uint32_t *__restrict__ prow, uint64_t t,
                                                                 const int64_t *__restrict__ pstart,
                                                                 const IP *__restrict__ aip, int64_t *__restrict__ pnz) {
  const int lane = threadIdx.x & 31;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= pstart[t]) return;
  const int64_t b = piece_bucket(pstart, t, j);
  const int64_t g0 = pindptr[b] + (j - pstart[b]) * kPtPiece, g1 = min(pindptr[b + 1], g0 + kPtPiece);
  int64_t s = 0;
  for (int64_t p = g0 + lane; p < g1; p += 32) {
    const int64_t row = __ldg(prow + p) & 0x7fffffffu;
    s += (int64_t)aip[row + 1] - (int64_t)aip[row];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) pnz[j] = s;
}

// P3: CTA per piece.  reg[j * (nblk + 1) + q] = first slot of the piece's
// block-q region (q = nblk: the piece's end).
template <typename IP, typename IX, typename TV>
__global__ void __launch_bounds__(kPtThreads) csr_part_scatter_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, uint64_t t,
    const int64_t *__restrict__ pstart, const int64_t *__restrict__ pbase, int nblk, const IP *__restrict__ aip,
    const IX *__restrict__ aix, const TV *__restrict__ av, int64_t *__restrict__ reg, uint16_t *__restrict__ wkey,
    TV *__restrict__ wval) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t *rstart = reinterpret_cast<int64_t *>(smem_raw);        // kPtPiece: row start | sign << 63
  int64_t *rlen = rstart + kPtPiece;                               // kPtPiece
  int64_t *rbase = rlen + kPtPiece;                                // kPtMaxBlocks + 1
  int32_t *cnt = reinterpret_cast<int32_t *>(rbase + kPtMaxBlocks + 1);  // kPtPiece x nblk run lengths
  int32_t *off = cnt + kPtPiece * nblk;                            // kPtPiece x nblk, scanned per block
  __shared__ int32_t wsum[kPtThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t j = blockIdx.x;
  if (j >= pstart[t]) return;
  const int64_t b = piece_bucket(pstart, t, j);
  const int64_t g0 = pindptr[b] + (j - pstart[b]) * kPtPiece;
  const int ng = (int)min((int64_t)kPtPiece, pindptr[b + 1] - g0);
  for (int i = tid; i < kPtPiece * nblk; i += kPtThreads) cnt[i] = 0;
  for (int r = tid; r < ng; r += kPtThreads) {
    const uint32_t wd = __ldg(prow + g0 + r);
    const int64_t row = wd & 0x7fffffffu;
    const int64_t rs = (int64_t)aip[row];
    rstart[r] = rs | ((int64_t)(wd >> 31) << 63);
    rlen[r] = (int64_t)aip[row + 1] - rs;
  }
  __syncthreads();
  // ---- run lengths per (row, block): warp per row, run starts of each batch
  for (int r = w; r < ng; r += kPtThreads / 32) {
    const int64_t rs = rstart[r] & 0x7fffffffffffffffLL, len = rlen[r];
    for (int64_t k0 = 0; k0 < len; k0 += 32 * kPtBatch) {
      int qs[kPtBatch];
#pragma unroll
      for (int u = 0; u < kPtBatch; ++u) {
        const int64_t k = k0 + 32 * u + lane;
        qs[u] = k < len ? (int)((int64_t)__ldg(aix + rs + k) >> kCbShift) : kPtMaxBlocks;  // canonical: q < nblk
      }
#pragma unroll
      for (int u = 0; u < kPtBatch; ++u) {
        if (k0 + 32 * u >= len) break;  // warp-uniform
        const int q = qs[u];
        const int qp = __shfl_up_sync(0xffffffffu, q, 1);
        const uint32_t starts = __ballot_sync(0xffffffffu, q < kPtMaxBlocks && (lane == 0 || q != qp));
        if (q < kPtMaxBlocks && (lane == 0 || q != qp)) {
          // run of block q from this lane to the next run start (or the batch end)
          const uint32_t later = starts & ~((2u << lane) - 1u);
          const int end = later ? __ffs(later) - 1 : 32;
          const int valid = (int)min((int64_t)32, len - (k0 + 32 * u));
          cnt[r * nblk + q] += min(end, valid) - lane;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // ---- per block: exclusive scan of the run lengths over the rows
  for (int q = 0; q < nblk; ++q) {
    const int r = tid;  // kPtThreads == kPtPiece: one row per thread
    const int32_t a = r < ng ? cnt[r * nblk + q] : 0;
    int32_t x = a;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int32_t ws = lane < kPtThreads / 32 ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      if (lane < kPtThreads / 32) wsum[lane] = ws;
    }
    __syncthreads();
    if (r < ng) off[r * nblk + q] = (w ? wsum[w - 1] : 0) + x - a;
    if (tid == 0) rbase[q] = wsum[kPtThreads / 32 - 1];  // block total (turned into a base below)
    __syncthreads();
  }
  if (tid == 0) {
    int64_t acc = pbase[j];
    for (int q = 0; q < nblk; ++q) {
      const int64_t c = rbase[q];
      rbase[q] = acc;
      reg[j * (nblk + 1) + q] = acc;
      acc += c;
    }
    rbase[nblk] = acc;
    reg[j * (nblk + 1) + nblk] = acc;
  }
  __syncthreads();
  // ---- entries: warp per row; lane q < nblk holds block q's slot base minus
  // the run's first entry index inside the row
  for (int r = w; r < ng; r += kPtThreads / 32) {
    const int64_t rsg = rstart[r];
    const int64_t rs = rsg & 0x7fffffffffffffffLL, len = rlen[r];
    const bool neg = rsg < 0;
    const int32_t c_l = lane < nblk ? cnt[r * nblk + lane] : 0;
    int32_t inc = c_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int64_t qbase = lane < nblk ? rbase[lane] + off[r * nblk + lane] - (int64_t)(inc - c_l) : 0;
    for (int64_t k0 = 0; k0 < len; k0 += 32 * kPtBatch) {
      IX cc[kPtBatch];
      TV vv[kPtBatch];
#pragma unroll
      for (int u = 0; u < kPtBatch; ++u) {
        const int64_t k = k0 + 32 * u + lane;
        cc[u] = (IX)-1;
        if (k < len) {
          cc[u] = __ldg(aix + rs + k);
          vv[u] = __ldg(av + rs + k);
        }
      }
#pragma unroll
      for (int u = 0; u < kPtBatch; ++u) {
        const int64_t k = k0 + 32 * u + lane;
        const int q = cc[u] == (IX)-1 ? 0 : (int)((int64_t)cc[u] >> kCbShift);
        const int64_t qb = __shfl_sync(0xffffffffu, qbase, q);
        if (cc[u] != (IX)-1) {
          const int64_t pos = qb + k;
          wkey[pos] = (uint16_t)((int64_t)cc[u] & (kCbCols - 1));
          wval[pos] = neg ? -vv[u] : vv[u];
        }
      }
    }
  }
}

inline size_t part_scatter_smem(int nblk) {
  return (size_t)(2 * kPtPiece + kPtMaxBlocks + 1) * 8 + (size_t)2 * kPtPiece * nblk * 4;
}

// P4: CTA per (bucket, block): the bucket's pieces' block regions, in order
struct PtSmem {
  double acc[kCbCols];
  uint32_t seen[3][kCbCols / 32];
  int64_t pcum[kPtPieceTab];   // entries of the block before piece k (row order)
  int64_t pslot[kPtPieceTab];  // workspace slot of piece k's block region
  int32_t lpos[kCbList];  // region position (= row rank order) of a >= 3 column's entry
  int32_t lnext[kCbList];
  double lval[kCbList];
  int count;
  int overflow;
};

template <typename TV, typename TOut>
__global__ void __launch_bounds__(kPaThreads, 1) csr_part_accum_kernel(int nblk, int64_t d,
                                                                        const int64_t *__restrict__ pstart,
                                                                        const int64_t *__restrict__ reg,
                                                                        const uint16_t *__restrict__ wkey,
                                                                        const TV *__restrict__ wval,
                                                                        TOut *__restrict__ sa, int64_t ldsa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PtSmem &S = *reinterpret_cast<PtSmem *>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t b = blockIdx.x / nblk;
  const int q = (int)(blockIdx.x - b * nblk);
  const int64_t c0 = (int64_t)q << kCbShift;
  const int ncols = (int)min((int64_t)kCbCols, d - c0);
  const int64_t j0 = pstart[b], j1 = pstart[b + 1];
  // the block's entries = the pieces' block-q regions concatenated (row order);
  // `each(fn)` visits them with their position in that order
  int64_t ne = 0;
  for (int64_t j = j0; j < j1; ++j) ne += reg[j * (nblk + 1) + q + 1] - reg[j * (nblk + 1) + q];

  for (int i = tid; i < 3 * kCbCols / 32; i += kPaThreads) (&S.seen[0][0])[i] = 0u;
  if (tid == 0) {
    S.count = 0;
    S.overflow = ne >= (1LL << 31);
    int64_t acc = 0;
    for (int64_t jp = j0; jp < j1 && jp - j0 < kPtPieceTab; ++jp) {
      S.pcum[jp - j0] = acc;
      S.pslot[jp - j0] = reg[jp * (nblk + 1) + q];
      acc += reg[jp * (nblk + 1) + q + 1] - reg[jp * (nblk + 1) + q];
    }
  }
  __syncthreads();
  // register-resident fast path: the block's entries (<= kPaThreads x 2 x
  // kPtItems) are loaded once, both sweeps work from registers
  constexpr int kRes = 2 * kPtItems;
  const bool resident = ne <= (int64_t)kPaThreads * kRes && j1 - j0 <= kPtPieceTab;
  if (resident) {
    int rc[kRes];
    TV rv[kRes];
    // entry u of this thread sits at position f(u) of the block's row order
    auto fpos = [&](int u) -> int64_t {
      return (int64_t)(u / kPtItems) * kPaThreads * kPtItems + (int64_t)tid * kPtItems + (u % kPtItems);
    };
    {
      // pieces of the bucket: [S.pcum[k], S.pcum[k + 1]) of the block's row
      // order start at workspace slot S.pslot[k] (tables built before the sweep)
      const int np = (int)(j1 - j0);
#pragma unroll
      for (int u = 0; u < kRes; ++u) {
        const int64_t f = fpos(u);
        rc[u] = -1;
        if (f < ne) {
          int k = 0;
          while (k + 1 < np && S.pcum[k + 1] <= f) ++k;
          const int64_t i = S.pslot[k] + (f - S.pcum[k]);
          rc[u] = (int)wkey[i];
          rv[u] = wval[i];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kRes; ++u) {
      const int c = rc[u];
      if (c < 0) continue;
      const uint32_t m = 1u << (c & 31);
      if (atomicOr(&S.seen[0][c >> 5], m) & m)
        if (atomicOr(&S.seen[1][c >> 5], m) & m) atomicOr(&S.seen[2][c >> 5], m);
    }
    __syncthreads();
    for (int i = tid; i < kCbCols / 32; i += kPaThreads) {
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
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kRes; ++u) {
      const int c = rc[u];
      if (c < 0) continue;
      const double v = (double)rv[u];
      const uint32_t m = 1u << (c & 31);
      if (!(S.seen[1][c >> 5] & m)) {
        S.acc[c] = v + 0.0;  // the reference's 0.0 + v
      } else if (!(S.seen[2][c >> 5] & m)) {
        atomicAdd(&S.acc[c], v);  // two adds from +0.0: order-free
      } else {
        const int slot = atomicAdd(&S.count, 1);
        if (slot < kCbList) {
          S.lpos[slot] = (int32_t)fpos(u);
          S.lval[slot] = v;
          S.lnext[slot] = (int32_t)atomicExch(reinterpret_cast<unsigned long long *>(S.acc) + c, (unsigned long long)slot);
        }
      }
    }
  } else {
  // ---- a. contributions per column (kPtItems consecutive keys per thread in flight)
  for (int64_t jp = j0; jp < j1; ++jp) {
  const int64_t s0 = reg[jp * (nblk + 1) + q], pn = reg[jp * (nblk + 1) + q + 1] - s0;
  const uint16_t *key = wkey + s0;
  for (int64_t i0 = (int64_t)tid * kPtItems; i0 < pn; i0 += (int64_t)kPaThreads * kPtItems) {
    int cs[kPtItems];
#pragma unroll
    for (int j = 0; j < kPtItems; ++j) cs[j] = i0 + j < pn ? (int)key[i0 + j] : -1;
#pragma unroll
    for (int j = 0; j < kPtItems; ++j) {
      const int c = cs[j];
      if (c < 0) continue;
      const uint32_t m = 1u << (c & 31);
      if (atomicOr(&S.seen[0][c >> 5], m) & m)
        if (atomicOr(&S.seen[1][c >> 5], m) & m) atomicOr(&S.seen[2][c >> 5], m);
    }
  }
  }
  __syncthreads();
  for (int i = tid; i < kCbCols / 32; i += kPaThreads) {
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
  __syncthreads();
  // ---- b. order-free stores / adds; chains for columns seen >= 3 times
  int64_t posb = 0;  // position of the piece's first entry in the block's row order
  for (int64_t jp = j0; jp < j1; ++jp) {
  const int64_t s0 = reg[jp * (nblk + 1) + q], pn = reg[jp * (nblk + 1) + q + 1] - s0;
  const uint16_t *key = wkey + s0;
  const TV *val = wval + s0;
  for (int64_t i0 = (int64_t)tid * kPtItems; i0 < pn; i0 += (int64_t)kPaThreads * kPtItems) {
    int cs[kPtItems];
    double vs[kPtItems];
#pragma unroll
    for (int j = 0; j < kPtItems; ++j) {
      cs[j] = -1;
      if (i0 + j < pn) {
        cs[j] = (int)key[i0 + j];
        vs[j] = (double)val[i0 + j];
      }
    }
#pragma unroll
    for (int j = 0; j < kPtItems; ++j) {
      const int c = cs[j];
      if (c < 0) continue;
      const double v = vs[j];
      const uint32_t m = 1u << (c & 31);
      if (!(S.seen[1][c >> 5] & m)) {
        S.acc[c] = v + 0.0;  // the reference's 0.0 + v
      } else if (!(S.seen[2][c >> 5] & m)) {
        atomicAdd(&S.acc[c], v);  // two adds from +0.0: order-free
      } else {
        const int slot = atomicAdd(&S.count, 1);
        if (slot < kCbList) {
          S.lpos[slot] = (int32_t)(posb + i0 + j);
          S.lval[slot] = v;
          S.lnext[slot] = (int32_t)atomicExch(reinterpret_cast<unsigned long long *>(S.acc) + c, (unsigned long long)slot);
        }
      }
    }
  }
  posb += pn;
  }
  }
  __syncthreads();
  if (S.count > kCbList) S.overflow = 1;
  __syncthreads();
  // ---- c. chains in region order (= row rank order), summed from +0.0
  if (!S.overflow) {
    for (int i = tid; i < kCbCols / 32; i += kPaThreads) {
      uint32_t m = S.seen[2][i];
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        const int c = 32 * i + bit;
        int32_t ps[kCbChain];
        double vl[kCbChain];
        int k = 0;
        for (int e = (int)reinterpret_cast<long long *>(S.acc)[c]; e >= 0; e = S.lnext[e]) {
          if (k == kCbChain) {
            k = -1;
            break;
          }
          const int32_t pz = S.lpos[e];
          const double v = S.lval[e];
          int j = k++;
          while (j > 0 && ps[j - 1] > pz) {
            ps[j] = ps[j - 1];
            vl[j] = vl[j - 1];
            --j;
          }
          ps[j] = pz;
          vl[j] = v;
        }
        if (k < 0) {
          S.overflow = 1;
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
    // ordered fallback for the columns seen >= 3 times: one warp, the region
    // in order, same-column lanes of a batch in lane (= rank) order
    for (int i = tid; i < kCbCols / 32; i += kPaThreads) {
      uint32_t m = S.seen[2][i];
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        S.acc[32 * i + bit] = 0.0;
      }
    }
    __syncthreads();
    if (w == 0) {
      for (int64_t jp = j0; jp < j1; ++jp) {
      const int64_t s0 = reg[jp * (nblk + 1) + q], pn = reg[jp * (nblk + 1) + q + 1] - s0;
      const uint16_t *key = wkey + s0;
      const TV *val = wval + s0;
      for (int64_t i0 = 0; i0 < pn; i0 += 32) {
        const int64_t i = i0 + lane;
        int c = -1 - lane;
        double v = 0.0;
        bool has = false;
        if (i < pn) {
          const int cc = key[i];
          if (S.seen[2][cc >> 5] & (1u << (cc & 31))) {
            c = cc;
            v = (double)val[i];
            has = true;
          }
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, c);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int rounds = __reduce_max_sync(0xffffffffu, has ? rank + 1 : 0);
        for (int r = 0; r < rounds; ++r) {
          if (has && rank == r) S.acc[c] += v;
          __syncwarp();
        }
      }
      }
    }
  }
  __syncthreads();
  TOut *o = sa + b * ldsa + c0;
  for (int i = tid; i < ncols; i += kPaThreads)
    o[i] = (S.seen[0][i >> 5] & (1u << (i & 31))) ? (TOut)S.acc[i] : (TOut)0;
}

}  // namespace
}  // namespace skt
