// csr_fine.cuh -- deterministic K4 for canonical CSR A with very wide SA rows
// (BASELINE config 5), fine column blocks (sketch.py:155-164, bit-identical):
//
//   the bucket's rows (plan order = ascending row) are cut into pieces of
//   <= 32 rows; F1 counts pieces and stored entries per piece (rounded up to 8
//   so every piece starts on a 16-byte boundary of the workspace), F2 scans;
//   F3 (CTA per piece) orders the piece's entries by (1024-column block, row,
//      column): every (row, block) run's first and past-the-end entry index
//      marked by the lanes where the block changes, scanned over the rows per
//      block; entries placed in a shared-memory image of the piece's workspace
//      region and written out as one contiguous stream (pieces too large for
//      the image are placed directly in the workspace); keys are the column
//      inside the block (uint16), values s_i * v;
//   F4 (WARP per (bucket, block)) walks the block's entries -- the block's
//      regions of the bucket's pieces, concatenated = ascending row order --
//      32 at a time and adds them into 1024 fp64 accumulators in shared memory
//      with plain read-add-write; a step whose lanes share a column (found by
//      writing lane ids into a per-column tag byte and reading them back) adds
//      the sharing lanes one after the other in lane (= row) order.
//      Every output is the reference's sum: from +0.0, ascending row.
// No atomics of any kind, no CTA barriers in F4.  Needs <= 512 column blocks
// (d <= 524,288).
#pragma once

#include "common.cuh"
#include "csr_partition.cuh"  // csr_part_scan_kernel, piece_bucket

namespace skt {
namespace {

#ifndef SKT_FB_SHIFT
#define SKT_FB_SHIFT 10
#endif
#ifndef SKT_FA_WARPS
#define SKT_FA_WARPS 2
#endif
constexpr int kFbShift = SKT_FB_SHIFT;
constexpr int kFbCols = 1 << kFbShift;  // 1024 columns per block (2048: 1.05 ms vs 0.94 ms on config 5)
constexpr int kFbMaxBlocks = 512;
#ifndef SKT_FP_ROWS
#define SKT_FP_ROWS 32
#endif
constexpr int kFpRows = SKT_FP_ROWS;  // rows per piece (<= 32: lane per row)
#ifndef SKT_FS_THREADS
#define SKT_FS_THREADS 512
#endif
constexpr int kFsThreads = SKT_FS_THREADS;  // F3 threads
#ifndef SKT_FS_UNROLL_MARK
#define SKT_FS_UNROLL_MARK 8
#endif
#ifndef SKT_FS_UNROLL
#define SKT_FS_UNROLL 8
#endif
constexpr int kFsUnroll = SKT_FS_UNROLL;           // F3: 32-entry batches of a row in flight (entries)
constexpr int kFsUnrollMark = SKT_FS_UNROLL_MARK;  // ... (run marks)
constexpr int kFaWarps = SKT_FA_WARPS;  // F4 warps (units) per CTA
#ifndef SKT_FA_UNROLL
#define SKT_FA_UNROLL 4
#endif
constexpr int kFaUnroll = SKT_FA_UNROLL;  // F4: steps with loads in flight (x2: double-buffered)
constexpr int kFaWarpBytes = kFbCols * 8 + kFbCols + 512;  // accumulators, column tags, region tables

// entries of a piece staged in shared memory (F3)
template <typename TV>
__host__ __device__ constexpr int fine_cap() { return kFpRows * (sizeof(TV) == 4 ? 384 : 256); }

inline int fine_nblk(int64_t d) { return (int)std::max<int64_t>(1, (d + kFbCols - 1) / kFbCols); }

// F1a: pieces per bucket
__global__ void csr_fine_npieces_kernel(const int64_t *__restrict__ pindptr, uint64_t t, int64_t *__restrict__ np) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < (int64_t)t) np[b] = (pindptr[b + 1] - pindptr[b] + kFpRows - 1) / kFpRows;
}

// F1b: stored entries per piece, rounded up to a multiple of 8 (lane per row)
template <typename IP>
__global__ void __launch_bounds__(256) csr_fine_piece_nnz_kernel(const int64_t *__restrict__ pindptr,
                                                                 const uint32_t *__restrict__ prow, uint64_t t,
                                                                 const int64_t *__restrict__ pstart,
                                                                 const IP *__restrict__ aip, int64_t *__restrict__ pnz) {
  const int lane = threadIdx.x & 31;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= pstart[t]) return;
  const int64_t b = piece_bucket(pstart, t, j);
  const int64_t g = pindptr[b] + (j - pstart[b]) * kFpRows + lane;
  int64_t s = 0;
  if (lane < kFpRows && g < pindptr[b + 1]) {
    const int64_t row = __ldg(prow + g) & 0x7fffffffu;
    s = (int64_t)aip[row + 1] - (int64_t)aip[row];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) pnz[j] = (s + 7) & ~(int64_t)7;
}

inline size_t fine_scatter_smem(int nblk, size_t vsize) {
  const size_t head = (size_t)kFpRows * 8 + (size_t)kFpRows * 4 + (size_t)((nblk + 1 + 3) & ~3) * 4;
  const size_t cap = vsize == 4 ? fine_cap<float>() : fine_cap<double>();
  return head + (size_t)kFpRows * nblk * 4 + cap * (2 + vsize);
}

// F3: CTA per piece.  reg[j * (nblk + 1) + q] = first workspace slot of the
// piece's block-q region (q = nblk: the end of the piece's entries).
template <typename IP, typename IX, typename TV>
__global__ void __launch_bounds__(kFsThreads, 1024 / kFsThreads) csr_fine_scatter_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, uint64_t t,
    const int64_t *__restrict__ pstart, const int64_t *__restrict__ pbase, int nblk, const IP *__restrict__ aip,
    const IX *__restrict__ aix, const TV *__restrict__ av, int64_t *__restrict__ reg, uint16_t *__restrict__ wkey,
    TV *__restrict__ wval) {
  constexpr int kCap = fine_cap<TV>();
  constexpr int kWarps = kFsThreads / 32;
  constexpr int U = kFsUnroll;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t *rstart = reinterpret_cast<int64_t *>(smem_raw);     // kFpRows: row start | sign << 63
  int32_t *rlen = reinterpret_cast<int32_t *>(rstart + kFpRows);  // kFpRows
  int32_t *bbase = rlen + kFpRows;                             // nblk + 1: block regions inside the piece
  int32_t *start = bbase + ((nblk + 1 + 3) & ~3);              // kFpRows x nblk: run start k, then slot - k
  unsigned char *stage = reinterpret_cast<unsigned char *>(start + kFpRows * nblk);
  uint16_t *skey = reinterpret_cast<uint16_t *>(stage);
  TV *sval = reinterpret_cast<TV *>(stage + (size_t)kCap * 2);
  int32_t *kend = reinterpret_cast<int32_t *>(stage);          // kFpRows x nblk run ends (before the image is filled)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t j = blockIdx.x;
  if (j >= pstart[t]) return;
  __shared__ int64_t bucket_of_piece;
  if (tid == 0) bucket_of_piece = piece_bucket(pstart, t, j);
  __syncthreads();
  const int64_t b = bucket_of_piece;
  const int64_t g0 = pindptr[b] + (j - pstart[b]) * kFpRows;
  const int ng = (int)min((int64_t)kFpRows, pindptr[b + 1] - g0);
  {
    uint4 *z0 = reinterpret_cast<uint4 *>(start), *z1 = reinterpret_cast<uint4 *>(kend);
    for (int i = tid; i < kFpRows * nblk / 4; i += kFsThreads) z0[i] = z1[i] = make_uint4(0, 0, 0, 0);
  }
  if (tid < ng) {
    const uint32_t wd = __ldg(prow + g0 + tid);
    const int64_t row = wd & 0x7fffffffu;
    const int64_t rs = (int64_t)aip[row];
    rstart[tid] = rs | ((int64_t)(wd >> 31) << 63);
    rlen[tid] = (int32_t)((int64_t)aip[row + 1] - rs);
  }
  __syncthreads();
  // ---- per (row, block): the run's first and past-the-end entry index inside
  // the row (columns ascend, so a block's entries are one run); warp per row
  for (int r = w; r < ng; r += kWarps) {
    const IX *ix = aix + (rstart[r] & 0x7fffffffffffffffLL) + lane;
    const int len = rlen[r];
    int32_t *ks = start + r * nblk, *ke = kend + r * nblk;
    int carry = -1;  // block of the entry before this batch
    auto mark = [&](int q, int k) {  // q < 0: past the row's end
      int qp = __shfl_up_sync(0xffffffffu, q, 1);
      if (lane == 0) qp = carry;
      if (q >= 0 && q != qp) {
        ks[q] = k;
        if (qp >= 0) ke[qp] = k;
      }
      if (k == len - 1) ke[q] = len;
      carry = __shfl_sync(0xffffffffu, q, 31);
    };
    int k0 = 0;
    for (; k0 + 32 * kFsUnrollMark <= len; k0 += 32 * kFsUnrollMark) {
      int qs[kFsUnrollMark];
#pragma unroll
      for (int u = 0; u < kFsUnrollMark; ++u)
        qs[u] = (int)((int64_t)__ldg(ix + k0 + 32 * u) >> kFbShift);  // canonical: < nblk
#pragma unroll
      for (int u = 0; u < kFsUnrollMark; ++u) mark(qs[u], k0 + 32 * u + lane);
    }
    for (; k0 < len; k0 += 32) {
      const int k = k0 + lane;
      mark(k < len ? (int)((int64_t)__ldg(ix + k0) >> kFbShift) : -1, k);
    }
  }
  __syncthreads();
  // ---- per block: entries of earlier rows; start[r][q] = that - run start,
  // so entry k of row r goes to bbase[q] + start[r][q] + k
  for (int q = tid; q < nblk; q += kFsThreads) {
    int32_t run = 0;
    for (int r = 0; r < ng; ++r) {
      const int32_t k0 = start[r * nblk + q];
      start[r * nblk + q] = run - k0;
      run += kend[r * nblk + q] - k0;
    }
    bbase[q] = run;
  }
  __syncthreads();
  const int64_t pb = pbase[j];
  if (w == 0) {
    int32_t carry = 0;
    for (int c0 = 0; c0 < nblk; c0 += 32) {
      const int q = c0 + lane;
      const int32_t c = q < nblk ? bbase[q] : 0;
      int32_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (q < nblk) {
        bbase[q] = carry + x - c;
        reg[j * (nblk + 1) + q] = pb + carry + x - c;
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
      bbase[nblk] = carry;
      reg[j * (nblk + 1) + nblk] = pb + carry;
    }
  }
  __syncthreads();
  const int total = bbase[nblk];
  const bool staged = total <= kCap;
  // ---- entries: warp per row
  for (int r = w; r < ng; r += kWarps) {
    const int64_t rsg = rstart[r];
    const int64_t rs = rsg & 0x7fffffffffffffffLL;
    const IX *ix = aix + rs + lane;
    const TV *vp = av + rs + lane;
    const int len = rlen[r];
    const bool neg = rsg < 0;
    const int32_t *srow = start + r * nblk;
    auto place = [&](int32_t c, TV v, int k) {
      const int q = c >> kFbShift;
      const int pos = bbase[q] + srow[q] + k;
      const uint16_t key = (uint16_t)(c & (kFbCols - 1));
      if (neg) v = -v;
      if (staged) {
        skey[pos] = key;
        sval[pos] = v;
      } else {
        wkey[pb + pos] = key;
        wval[pb + pos] = v;
      }
    };
    int k0 = 0;
    for (; k0 + 32 * U <= len; k0 += 32 * U) {
      int32_t cc[U];
      TV vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        cc[u] = (int32_t)__ldg(ix + k0 + 32 * u);  // columns < d < 2^31
        vv[u] = __ldg(vp + k0 + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) place(cc[u], vv[u], k0 + 32 * u + lane);
    }
    for (; k0 < len; k0 += 32)
      if (k0 + lane < len) place((int32_t)__ldg(ix + k0), __ldg(vp + k0), k0 + lane);
  }
  if (!staged) return;
  __syncthreads();
  // ---- the image -> workspace, 16 bytes per thread (pb is a multiple of 8)
  {
    const uint4 *s = reinterpret_cast<const uint4 *>(skey);
    uint4 *g = reinterpret_cast<uint4 *>(wkey + pb);
    const int nv = (total * 2 + 15) / 16;
    for (int i = tid; i < nv; i += kFsThreads) g[i] = s[i];
  }
  {
    const uint4 *s = reinterpret_cast<const uint4 *>(sval);
    uint4 *g = reinterpret_cast<uint4 *>(wval + pb);
    const int nv = (int)(((size_t)total * sizeof(TV) + 15) / 16);
    for (int i = tid; i < nv; i += kFsThreads) g[i] = s[i];
  }
}

// F4: warp per (bucket, block)
template <typename TV, typename TOut>
__global__ void __launch_bounds__(kFaWarps * 32, 8) csr_fine_accum_kernel(int nblk, int64_t d, uint64_t t,
                                                                        const int64_t *__restrict__ pstart,
                                                                        const int64_t *__restrict__ reg,
                                                                        const uint16_t *__restrict__ wkey,
                                                                        const TV *__restrict__ wval,
                                                                        TOut *__restrict__ sa, int64_t ldsa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t unit = (int64_t)blockIdx.x * kFaWarps + w;
  if (unit >= (int64_t)t * nblk) return;
  const int64_t b = unit / nblk;
  const int q = (int)(unit - b * nblk);
  unsigned char *mine = smem_raw + (size_t)w * kFaWarpBytes;
  double *acc = reinterpret_cast<double *>(mine);                       // kFbCols
  uint8_t *tag = mine + kFbCols * 8;                                    // kFbCols: last lane that named the column
  int64_t *rbase = reinterpret_cast<int64_t *>(mine + kFbCols * 9);     // 32: slot of region entry 0 - entries before
  int32_t *rcum = reinterpret_cast<int32_t *>(mine + kFbCols * 9 + 256);  // 33: entries before region i
  {
    double2 *z = reinterpret_cast<double2 *>(acc);
    for (int i = lane; i < kFbCols / 2; i += 32) z[i] = make_double2(0.0, 0.0);
  }
  const int64_t j0 = pstart[b], j1 = pstart[b + 1];
  for (int64_t jg = j0; jg < j1; jg += 32) {  // the bucket's pieces, 32 regions at a time
    const int64_t j = jg + lane;
    int64_t s0 = 0;
    int32_t len = 0;
    if (j < j1) {
      s0 = reg[j * (nblk + 1) + q];
      len = (int32_t)(reg[j * (nblk + 1) + q + 1] - s0);
    }
    int32_t x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __syncwarp();  // the previous group's tables are no longer read
    rcum[lane + 1] = x;
    if (lane == 0) rcum[0] = 0;
    rbase[lane] = s0 - (int64_t)(x - len);
    __syncwarp();
    const int total = __shfl_sync(0xffffffffu, x, 31);
    // this lane's region (its entries are visited in increasing order): the
    // first entry past it, and the workspace arrays shifted so that entry v of
    // the block sits at pk[v] / pv[v]
    int ri = 0;
    int32_t rnext = rcum[1];
    const uint16_t *pk = wkey + rbase[0];
    const TV *pv = wval + rbase[0];
    auto fetch = [&](int v0, int32_t (&key)[kFaUnroll], TV (&val)[kFaUnroll]) {
#pragma unroll
      for (int u = 0; u < kFaUnroll; ++u) {
        const int v = v0 + 32 * u + lane;
        key[u] = 0x10000 | lane;  // idle lanes: distinct, never a column
        if (v < total) {
          if (v >= rnext) {
            do rnext = rcum[++ri + 1];
            while (v >= rnext);
            const int64_t rb = rbase[ri];
            pk = wkey + rb;
            pv = wval + rb;
          }
          key[u] = (int32_t)pk[v];
          val[u] = pv[v];
        }
      }
    };
    auto add = [&](int v0, const int32_t (&key)[kFaUnroll], const TV (&val)[kFaUnroll]) {
#pragma unroll
      for (int u = 0; u < kFaUnroll; ++u) {
        if (v0 + 32 * u >= total) break;  // warp-uniform
        const int32_t c = key[u];
        const bool act = c < 0x10000;
        if (act) tag[c] = (uint8_t)lane;
        __syncwarp();
        // lanes that lost their column's tag share it with a later writer
        uint32_t lost = __ballot_sync(0xffffffffu, act && tag[c] != (uint8_t)lane);
        bool alone = act;
        while (lost) {  // per shared column: its lanes add in lane (= row) order
          const int32_t cs = __shfl_sync(0xffffffffu, c, __ffs(lost) - 1);
          uint32_t peers = __ballot_sync(0xffffffffu, c == cs);
          lost &= ~peers;
          if (c == cs) alone = false;
          for (; peers; peers &= peers - 1) {
            if (lane == __ffs(peers) - 1) acc[c] += (double)val[u];
            __syncwarp();
          }
        }
        if (alone) acc[c] += (double)val[u];
        // no barrier here: the next step's adds come after its own tag barrier
      }
    };
    int32_t ka[kFaUnroll], kb[kFaUnroll];
    TV va[kFaUnroll], vb[kFaUnroll];
    fetch(0, ka, va);
    for (int v0 = 0; v0 < total; v0 += 64 * kFaUnroll) {  // loads of the next steps in flight
      fetch(v0 + 32 * kFaUnroll, kb, vb);
      add(v0, ka, va);
      fetch(v0 + 64 * kFaUnroll, ka, va);
      add(v0 + 32 * kFaUnroll, kb, vb);
    }
  }
  __syncwarp();
  const int64_t c0 = (int64_t)q << kFbShift;
  const int ncols = (int)min((int64_t)kFbCols, d - c0);
  TOut *o = sa + b * ldsa + c0;
  if (ncols == kFbCols && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
    constexpr int kPer = 16 / (int)sizeof(TOut);  // outputs per 16-byte store
    for (int i = lane * kPer; i < kFbCols; i += 32 * kPer) {
      if constexpr (sizeof(TOut) == 4) {
        const double2 a0 = *reinterpret_cast<const double2 *>(acc + i);
        const double2 a1 = *reinterpret_cast<const double2 *>(acc + i + 2);
        *reinterpret_cast<float4 *>(o + i) = make_float4((float)a0.x, (float)a0.y, (float)a1.x, (float)a1.y);
      } else {
        *reinterpret_cast<double2 *>(o + i) = *reinterpret_cast<const double2 *>(acc + i);
      }
    }
  } else {
    for (int i = lane; i < ncols; i += 32) o[i] = (TOut)acc[i];
  }
}

}  // namespace
}  // namespace skt
