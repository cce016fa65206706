// csr_window.cuh -- K4 "row-window" kernel for canonical CSR with narrow d and
// rows of ~16 nonzeros (BASELINE config 4): A is STREAMED once in row order
// instead of gathered in bucket order.
//
// The bucket-ordered kernels (csr_tile.cuh) visit rows in plan order, i.e. at
// random: every row costs an indptr pair plus two ~64-byte segments at
// arbitrary offsets, and the chip serves such requests at a request rate, not
// a byte rate.  Here the rows are cut into windows of W
// consecutive rows, and one persistent kernel runs two kinds of warps against
// each other, window by window:
//
//  * scatter side (kWinScat warps per CTA): the CTA's contiguous block of the
//    window is fetched 32 rows at a time with the bulk-copy engine
//    (cp.async.bulk global -> shared, completion counted in bytes on an
//    mbarrier, two stages per warp; the block two windows ahead is prefetched
//    into L2), and every row is written as ONE aligned 128-byte slot -- 16
//    (column, signed fp32 value) pairs -- at the position the WINDOW PLAN
//    gives it: the rows of a window stably sorted by bucket.  Stores carry no
//    dependency chain; the slot buffers (a ring of kWinBufs windows) stay in
//    L2.
//  * accumulate side (kWinAcc warps per CTA): warp g owns buckets
//    [g*bpw, (g+1)*bpw) with their fp64 accumulators in shared memory.  In a
//    window its rows are one contiguous slot range, read with coalesced
//    128-bit loads, scattered into a zeroed 16-row tile and added row by row
//    in ascending row order (absent entries add +0.0, an exact identity), so
//    every SA element is summed in exactly the reference's order: bit-identical
//    to the bincount of sketch.py:155-164.
//
// Windows are handed over through two counters per window in global memory
// (scattered / consumed; release-acquire, no data atomics).  Rows longer than
// 16 nonzeros leave a marker slot (row start, length, sign) and the
// accumulating warp reads them straight from A.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace skt {
namespace {

constexpr int kWinScat = 8;     // consumer warps of the scatter side
constexpr int kWinAcc = 14;     // accumulating warps
constexpr int kWinWarps = kWinScat + kWinAcc;
constexpr int kWinThreads = kWinWarps * 32;
#ifndef SKT_WIN_SPW
#define SKT_WIN_SPW 2
#endif
#ifndef SKT_WIN_TILE_ROWS
#define SKT_WIN_TILE_ROWS 16
#endif
constexpr int kWinSpw = SKT_WIN_SPW;  // bulk-copy stages per scatter warp
constexpr int kWinCap = 576;    // entries per stage (index + value arrays)
static_assert(kWinCap * 4 == 2304, "the scatter loop hard-codes the value offset of a stage");
constexpr int kWinStageBytes = kWinCap * 8 + 288 + 128 + 96;  // 5120: entries, indptr (<= 36 x 8 B), plan words
constexpr int kWinSlot = 16;    // entries per slot (128 bytes)
constexpr int kWinTileRows = SKT_WIN_TILE_ROWS;
constexpr uint32_t kWinEmpty = 0xffffffffu, kWinLong = 0xfffffffeu;

struct WinParams {
  const void *aip;
  const int32_t *aix;
  const float *av;
  int64_t n, nnz;
  int d, dp;
  uint64_t t;
  const uint32_t *pos;  // [n]: slot of the row inside its window | sign << 31
  const int32_t *wpi;   // [nwin][t + 1]: first slot of bucket b in window w
  unsigned char *slots; // nbuf x W x 128 bytes
  uint32_t *scat_done, *acc_done;  // [nwin] each, zeroed before the launch
  int32_t W, nwin, nbuf, cpb, bpw;
  void *sa;
  int64_t ldsa;
};

__device__ __forceinline__ uint32_t wn_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wn_mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(wn_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void wn_mbar_expect(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(wn_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wn_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(wn_smem(bar)) : "memory");
}
__device__ __forceinline__ void wn_mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
          wn_smem(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ uint64_t wn_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t wn_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void wn_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          wn_smem(dst)),
      "l"(src), "r"(bytes), "r"(wn_smem(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void wn_prefetch_l2(const void *src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void wn_st_slot4(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a), "r"(b), "r"(c),
               "r"(d), "l"(pol));
}
__device__ __forceinline__ uint4 wn_ld_slot(const void *p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t wn_ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wn_fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void wn_red_release(uint32_t *p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
// the whole warp polls (no divergence) until *p >= want
__device__ __forceinline__ void wn_wait_count(const uint32_t *p, uint32_t want) {
  uint32_t ns = 32;
  while (wn_ld_relaxed(p) < want) {
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
  }
  wn_fence_acquire();
}

template <typename IP, typename TOut, int kChunks>
__global__ void __launch_bounds__(kWinThreads, 1) csr_window_kernel(const WinParams p) {
  extern __shared__ __align__(128) unsigned char wn_smem_raw[];
  __shared__ __align__(8) uint64_t full[kWinScat * kWinSpw];
  __shared__ uint32_t scat_cnt[8], acc_cnt[8];  // per-window arrival counters of the CTA's warps
  __shared__ int acc_offs[kWinAcc][32];  // bucket boundaries of the current window, per accumulating warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = (int)gridDim.x, cta = (int)blockIdx.x;
  const IP *__restrict__ aip = (const IP *)p.aip;
  const int32_t *__restrict__ aix = p.aix;
  const float *__restrict__ av = p.av;
  // [scatter warp][stage]: index entries, value entries, 36 indptr values, 32 plan words
  double *acc_all = (double *)(wn_smem_raw + (size_t)kWinScat * kWinSpw * kWinStageBytes);  // [acc warp][bpw][dp]
  float *tile_all = (float *)(acc_all + (size_t)kWinAcc * p.bpw * p.dp);  // [acc warp][rows][dp]

  if (threadIdx.x < 8) scat_cnt[threadIdx.x] = acc_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWinScat * kWinSpw; ++s) wn_mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t n = p.n;
  const int W = p.W, cpb = p.cpb, nwin = p.nwin;

  if (warp < kWinScat) {
    // ------------------------------------------------------------ scatter
    // This warp's chunks: c = warp + kWinScat * i of the CTA's block of every
    // window, i < cpw; flattened over the windows as J.  Chunk J lands in the
    // warp's stage J % kWinSpw (index / value entries, the 33 indptr values
    // and the 32 plan words of its rows, four bulk copies on one mbarrier);
    // the copy of chunk J + kWinSpw is issued when chunk J has been consumed.
    // Lane i < cpw keeps the entry range of chunk i of windows w, w+1, w+2
    // (h, g, f), loaded two windows ahead, so no global load sits on the
    // warp's critical path.
    typedef typename std::conditional<sizeof(IP) == 4, int32_t, int64_t>::type E;
    const int sw = warp;
    const int sub = lane >> 3, part = lane & 7;  // 4 rows per step, 8 lanes per row, 2 entries per lane
    const int cpw = cpb / kWinScat;
    uint64_t *bars = full + sw * kWinSpw;
    unsigned char *stage_w = wn_smem_raw + (size_t)sw * kWinSpw * kWinStageBytes;
    struct Cur {
      int w, i;
      int64_t row;
    };
    const int64_t wrap = (int64_t)W - (int64_t)cpw * kWinScat * 32;
    auto adv = [&](Cur &c) {
      c.row += kWinScat * 32;
      if (++c.i == cpw) {
        c.i = 0;
        ++c.w;
        c.row += wrap;
      }
    };
    const E nnz_al = (E)(p.nnz & ~(int64_t)3);
    // the 16-byte-aligned entry range [a0, a0 + cnt) a chunk [e0, e1) of rows
    // [row, row + 32) is copied as; false = the chunk is read from global memory
    // (does not fit a stage / unaligned tail of the arrays / last rows of A)
    auto chunk_range = [&](int64_t row, E e0, E e1, E &a0, uint32_t &cnt) -> bool {
      a0 = e0 & ~(E)3;
      const E a1 = (e1 + 3) & ~(E)3;
      cnt = 0;
      if (row + 36 > n) return false;
      if (e1 <= e0) return true;
      if (a1 > nnz_al || a1 - a0 > (E)kWinCap) return false;
      cnt = (uint32_t)(a1 - a0);
      return true;
    };
    auto load_range = [&](int w, E &e0, E &e1) {  // lane i < cpw: chunk i of window w
      e0 = e1 = 0;
      const int64_t row = (int64_t)w * W + ((int64_t)cta * cpb + sw + kWinScat * lane) * 32;
      if (lane < cpw && w < nwin && row < n) {
        e0 = (E)aip[row];
        e1 = (E)aip[(row + 32 < n) ? row + 32 : n];
      }
    };
    const uint64_t pol_stream = wn_policy_evict_first(), pol_keep = wn_policy_evict_last();
    auto issue = [&](int s, const Cur &c, E e0, E e1) {  // whole warp: lane 0 arms the barrier, lanes 0-3 copy
      if (c.w >= nwin) return;
      E a0;
      uint32_t cnt;
      unsigned char *st = stage_w + (size_t)s * kWinStageBytes;
      if (c.row < n && chunk_range(c.row, e0, e1, a0, cnt)) {
        if (lane == 0) wn_mbar_expect(&bars[s], cnt * 8u + 36u * (uint32_t)sizeof(IP) + 128u);
        __syncwarp();
        if (lane == 0 && cnt > 0) wn_bulk_g2s(st, aix + a0, cnt * 4u, &bars[s], pol_stream);
        if (lane == 1 && cnt > 0) wn_bulk_g2s(st + kWinCap * 4, av + a0, cnt * 4u, &bars[s], pol_stream);
        if (lane == 2) wn_bulk_g2s(st + kWinCap * 8, aip + c.row, 36u * (uint32_t)sizeof(IP), &bars[s], pol_stream);
        if (lane == 3) wn_bulk_g2s(st + kWinCap * 8 + 288, p.pos + c.row, 128u, &bars[s], pol_stream);
      } else if (lane == 0) {
        wn_mbar_arrive(&bars[s]);
      }
    };
    E h0, h1, g0, g1, f0, f1;
    load_range(0, h0, h1);
    load_range(1, g0, g1);
    auto range_of = [&](const Cur &c, int w, E &e0, E &e1) {  // all lanes; c.w in [w, w + 2]
      const int dw = c.w - w;
      const E x0 = dw == 0 ? h0 : dw == 1 ? g0 : f0, x1 = dw == 0 ? h1 : dw == 1 ? g1 : f1;
      e0 = __shfl_sync(0xffffffffu, x0, c.i);
      e1 = __shfl_sync(0xffffffffu, x1, c.i);
    };
    Cur cc{0, 0, ((int64_t)cta * cpb + sw) * 32};
    Cur ci = cc;
    f0 = f1 = 0;
#pragma unroll
    for (int s = 0; s < kWinSpw; ++s) {
      E e0, e1;
      range_of(ci, 0, e0, e1);  // needs cpw >= kWinSpw (the host checks cpb)
      issue(s, ci, e0, e1);
      adv(ci);
    }
    int J = 0;
    for (int w = 0; w < nwin; ++w) {
      load_range(w + 2, f0, f1);  // used from the end of this window on
      if (w >= p.nbuf) wn_wait_count(p.acc_done + (w - p.nbuf), (uint32_t)G);
      unsigned char *slotlane = p.slots + (size_t)(w % p.nbuf) * (size_t)W * 128 + part * 16;
      for (int i = 0; i < cpw; ++i, ++J) {
        const int s = J % kWinSpw;
        const uint32_t ph = (uint32_t)(J / kWinSpw) & 1u;
        const int64_t rowc = cc.row;
        const int nrows = (int)(rowc >= n ? 0 : (n - rowc < 32 ? n - rowc : 32));
        const bool valid = lane < nrows;
        const E ce0 = __shfl_sync(0xffffffffu, h0, i), ce1 = __shfl_sync(0xffffffffu, h1, i);
        E a0;
        uint32_t cnt;
        const bool staged = nrows > 0 && chunk_range(rowc, ce0, ce1, a0, cnt);
        const unsigned char *st = stage_w + (size_t)s * kWinStageBytes;
        wn_mbar_wait(&bars[s], ph);
        E rs = 0, re = 0;
        uint32_t pw = 0;
        if (staged) {
          const IP *sip = reinterpret_cast<const IP *>(st + kWinCap * 8);
          rs = (E)sip[lane];
          re = (E)sip[lane + 1];
          pw = reinterpret_cast<const uint32_t *>(st + kWinCap * 8 + 288)[lane];
        } else if (valid) {
          rs = (E)aip[rowc + lane];
          re = (E)aip[rowc + lane + 1];
          pw = __ldg(p.pos + rowc + lane);
        }
        const E len = re - rs;
        const bool is_long = len > kWinSlot;
        // row descriptor: byte offset of the row in the stage (14 bits), entries to copy (5),
        // sign (bit 19), long row (20), valid (21)
        const uint32_t meta = valid ? ((((uint32_t)(rs - a0) * 4u) & 0x3fffu) | ((is_long ? 0u : (uint32_t)len) << 14) |
                                       ((pw >> 31) << 19) | ((uint32_t)is_long << 20) | (1u << 21))
                                    : 0u;
        const uint32_t dst = (pw & 0x7fffffffu) * 128u;
        if (staged) {
          // branch-free: every lane reads its two entries (garbage past the row's
          // end stays inside the stage) and selects the empty marker
          const uint32_t sb = wn_smem(st) + part * 8;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int r = 4 * it + sub;
            const uint32_t m1 = __shfl_sync(0xffffffffu, meta, r), ds = __shfl_sync(0xffffffffu, dst, r);
            const uint32_t l = (m1 >> 14) & 31u, neg = (m1 << 12) & 0x80000000u;
            const uint32_t a = sb + (m1 & 0x3fffu);
            uint32_t x0, y0, x1, y1;
            asm("ld.shared.u32 %0, [%1];" : "=r"(x0) : "r"(a));
            asm("ld.shared.u32 %0, [%1+2304];" : "=r"(y0) : "r"(a));
            asm("ld.shared.u32 %0, [%1+4];" : "=r"(x1) : "r"(a));
            asm("ld.shared.u32 %0, [%1+2308];" : "=r"(y1) : "r"(a));
            const bool p0 = (uint32_t)(2 * part) < l, p1 = (uint32_t)(2 * part + 1) < l;
            const uint32_t c0 = p0 ? x0 : kWinEmpty, v0 = p0 ? (y0 ^ neg) : 0u;
            const uint32_t c1 = p1 ? x1 : kWinEmpty, v1 = p1 ? (y1 ^ neg) : 0u;
            if ((m1 >> 21) && !(((m1 >> 20) & 1u) && part < 2))
              wn_st_slot4(slotlane + ds, c0, v0, c1, v1, pol_keep);
          }
        } else if (nrows > 0) {
#pragma unroll 1
          for (int it = 0; it < 8; ++it) {
            const int r = 4 * it + sub;
            const E rs_r = __shfl_sync(0xffffffffu, rs, r);
            const uint32_t m1 = __shfl_sync(0xffffffffu, meta, r), ds = __shfl_sync(0xffffffffu, dst, r);
            const uint32_t l = (m1 >> 14) & 31u, neg = (m1 << 12) & 0x80000000u;
            uint32_t c0 = kWinEmpty, v0 = 0, c1 = kWinEmpty, v1 = 0;
            if ((uint32_t)(2 * part) < l) {
              c0 = (uint32_t)__ldg(aix + rs_r + 2 * part);
              v0 = __float_as_uint(__ldg(av + rs_r + 2 * part)) ^ neg;
            }
            if ((uint32_t)(2 * part + 1) < l) {
              c1 = (uint32_t)__ldg(aix + rs_r + 2 * part + 1);
              v1 = __float_as_uint(__ldg(av + rs_r + 2 * part + 1)) ^ neg;
            }
            if ((m1 >> 21) && !(((m1 >> 20) & 1u) && part < 2))
              wn_st_slot4(slotlane + ds, c0, v0, c1, v1, pol_keep);
          }
        }
        if (valid && is_long) {  // marker slot: the accumulating warp reads the row from A
          unsigned char *sl = slotlane - part * 16 + dst;
          wn_st_slot4(sl, kWinLong, (uint32_t)len, kWinLong, (uint32_t)rs, pol_keep);
          wn_st_slot4(sl + 16, kWinLong, (uint32_t)((uint64_t)rs >> 32), kWinLong, pw >> 31, pol_keep);
        }
        __syncwarp();
        {
          E e0, e1;
          range_of(ci, w, e0, e1);
          issue(s, ci, e0, e1);
          adv(ci);
        }
        adv(cc);
      }
      if (f1 > f0) {  // L2 prefetch of this warp's chunks two windows ahead
        const E q0 = f0 & ~(E)3;
        E q1 = (f1 + 3) & ~(E)3;
        if (q1 > nnz_al) q1 = nnz_al;
        if (q1 > q0) {
          wn_prefetch_l2(aix + q0, (uint32_t)(q1 - q0) * 4u, pol_stream);
          wn_prefetch_l2(av + q0, (uint32_t)(q1 - q0) * 4u, pol_stream);
        }
      }
      h0 = g0;
      h1 = g1;
      g0 = f0;
      g1 = f1;
      {
        // the last scatter warp of the CTA to finish the window publishes it
        __threadfence_block();
        __syncwarp();
        uint32_t last = 0;
        if (lane == 0) last = atomicAdd(&scat_cnt[w & 7], 1u) == kWinScat - 1;
        if (__shfl_sync(0xffffffffu, last, 0)) {
          if (lane == 0) {
            scat_cnt[w & 7] = 0;
            __threadfence();
            wn_red_release(p.scat_done + w);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------ accumulate
    const int aw = warp - kWinScat;
    const int dp = p.dp, d = p.d;
    const int64_t gaw = (int64_t)cta * kWinAcc + aw;
    const int64_t b0 = gaw * p.bpw;
    const int nb = (int)(b0 >= (int64_t)p.t ? 0 : ((int64_t)p.t - b0 < p.bpw ? (int64_t)p.t - b0 : p.bpw));
    double *accs = acc_all + (size_t)aw * p.bpw * dp;
    float *tile = tile_all + (size_t)aw * kWinTileRows * dp;
    for (int i = lane; i < p.bpw * dp; i += 32) accs[i] = 0.0;
    for (int i = lane; i < kWinTileRows * dp; i += 32) tile[i] = 0.f;
    __syncwarp();
    const uint32_t scat_want = (uint32_t)G;
    const int part = lane & 7, sub = lane >> 3;
    const uint64_t pol_keep = wn_policy_evict_last();
    int *offs = &acc_offs[aw][0];
    uint4 e[kWinTileRows / 4];
    auto load_wpi = [&](int w) -> int {
      return (nb > 0 && lane <= nb && w < nwin) ? __ldg(p.wpi + (size_t)w * (p.t + 1) + b0 + lane) : 0;
    };
    auto load_batch = [&](int w, int base, int hi) {
      const unsigned char *sb = p.slots + (size_t)(w % p.nbuf) * (size_t)W * 128;
      const int nr = hi - base < kWinTileRows ? hi - base : kWinTileRows;
#pragma unroll
      for (int i = 0; i < kWinTileRows / 4; ++i) {
        const int row = 4 * i + sub;
        e[i] = make_uint4(kWinEmpty, 0, kWinEmpty, 0);
        if (row < nr) e[i] = wn_ld_slot(sb + (size_t)(base + row) * 128 + part * 16, pol_keep);
      }
    };
    int off_next = load_wpi(0);
    bool pre = false;  // this window's first batch is already in flight
    for (int w = 0; w < nwin; ++w) {
      const int off = off_next;
      const int lo = __shfl_sync(0xffffffffu, off, 0), hi = __shfl_sync(0xffffffffu, off, nb);
      off_next = load_wpi(w + 1);  // in flight during this window
      __syncwarp();
      offs[lane] = off;
      __syncwarp();
      if (!pre) {
        wn_wait_count(p.scat_done + w, scat_want);
        if (lo < hi) load_batch(w, lo, hi);
      }
      pre = false;
      int k = 0;
      for (int base = lo; base < hi; base += kWinTileRows) {
        const int nrows = hi - base < kWinTileRows ? hi - base : kWinTileRows;
        // ---- scatter the batch into the tile
#pragma unroll
        for (int i = 0; i < kWinTileRows / 4; ++i) {
          const int row = 4 * i + sub;
          if (e[i].x < (uint32_t)d) tile[row * dp + e[i].x] = __uint_as_float(e[i].y);
          if (e[i].z < (uint32_t)d) tile[row * dp + e[i].z] = __uint_as_float(e[i].w);
        }
        bool any_long = false;
#pragma unroll
        for (int i = 0; i < kWinTileRows / 4; ++i) any_long |= (part == 0 && e[i].x == kWinLong);
        if (__any_sync(0xffffffffu, any_long)) {
#pragma unroll
          for (int i = 0; i < kWinTileRows / 4; ++i) {
            uint32_t m = __ballot_sync(0xffffffffu, part == 0 && e[i].x == kWinLong);
            while (m) {  // long rows straight from A, whole warp per row
              const int src = __ffs(m) - 1;
              m &= m - 1;
              const uint32_t len = __shfl_sync(0xffffffffu, e[i].y, src);
              const uint32_t rlo = __shfl_sync(0xffffffffu, e[i].w, src);
              const uint32_t rhi = __shfl_sync(0xffffffffu, e[i].y, src + 1);
              const uint32_t neg = __shfl_sync(0xffffffffu, e[i].w, src + 1);
              const int64_t rs = (int64_t)(((uint64_t)rhi << 32) | rlo);
              const int row = 4 * i + (src >> 3);
              for (uint32_t qq = lane; qq < len; qq += 32) {
                const float v = __ldg(av + rs + qq);
                tile[row * dp + __ldg(aix + rs + qq)] = neg ? -v : v;
              }
            }
          }
        }
        // ---- next batch in flight during the adds (the next window's first
        // batch when that window is already scattered)
        if (base + kWinTileRows < hi) {
          load_batch(w, base + kWinTileRows, hi);
        } else if (w + 1 < nwin) {
          const uint32_t seen = __shfl_sync(0xffffffffu, wn_ld_relaxed(p.scat_done + w + 1), 0);
          if (seen >= scat_want) {
            wn_fence_acquire();
            const int lo2 = __shfl_sync(0xffffffffu, off_next, 0), hi2 = __shfl_sync(0xffffffffu, off_next, nb);
            if (lo2 < hi2) load_batch(w + 1, lo2, hi2);
            pre = true;
          }
        }
        __syncwarp();
        // ---- add the rows bucket by bucket, ascending row order
        while (k < nb) {
          const int o0 = offs[k], o1 = offs[k + 1];
          const int s0 = (o0 > base ? o0 : base) - base;
          const int s1 = (o1 < base + nrows ? o1 : base + nrows) - base;
          if (s1 > s0) {
#pragma unroll
            for (int j = 0; j < kChunks; ++j) {
              const int c = 64 * j + 2 * lane;
              if (c < dp) {
                double2 a = *reinterpret_cast<double2 *>(accs + k * dp + c);
                for (int r = s0; r < s1; ++r) {
                  const float2 x = *reinterpret_cast<const float2 *>(tile + r * dp + c);
                  a.x += (double)x.x;
                  a.y += (double)x.y;
                }
                *reinterpret_cast<double2 *>(accs + k * dp + c) = a;
              }
            }
          }
          if (o1 > base + nrows) break;  // the bucket continues in the next batch
          ++k;
        }
        __syncwarp();
        {
          uint4 *z = reinterpret_cast<uint4 *>(tile);
          const int words = nrows * dp / 4;
          for (int i = lane; i < words; i += 32) z[i] = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }
      // the last accumulating warp of the CTA to finish the window releases its buffer
      __syncwarp();
      if (lane == 0 && atomicAdd(&acc_cnt[w & 7], 1u) == kWinAcc - 1) {
        acc_cnt[w & 7] = 0;
        wn_red_release(p.acc_done + w);
      }
    }
    // ---- write SA
    TOut *sa = (TOut *)p.sa;
    for (int kk = 0; kk < nb; ++kk)
      for (int c = lane; c < d; c += 32) sa[(b0 + kk) * p.ldsa + c] = (TOut)accs[kk * dp + c];
  }
}

// ---- window plan ---------------------------------------------------------
// From the per-bucket plan (rows of a bucket in ascending order): the rows of
// window w = row / W that fall in bucket b are one run of the bucket's list.
// Pass 0 writes the run lengths cnt[w][b]; after an exclusive scan over b per
// window, pass 1 writes pos[row] = wpi[w][b] + (rank inside the run) | sign.
template <int kPass>
__global__ void __launch_bounds__(256) win_plan_kernel(const int64_t *__restrict__ pindptr,
                                                       const uint32_t *__restrict__ prow, uint64_t t, int32_t W,
                                                       int32_t *__restrict__ wpi, uint32_t *__restrict__ pos) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= (int64_t)t) return;
  const int64_t beg = pindptr[b], end = pindptr[b + 1];
  int carry_w = -1, carry_cnt = 0;
  for (int64_t k0 = beg; k0 < end; k0 += 32) {
    const bool has = k0 + lane < end;
    const uint32_t wd = has ? __ldg(prow + k0 + lane) : 0u;
    const int w = has ? (int)((wd & 0x7fffffffu) / (uint32_t)W) : 0x7fffffff;
    const int wprev = __shfl_up_sync(0xffffffffu, w, 1);
    const bool head = lane == 0 ? (w != carry_w) : (w != wprev);
    const uint32_t hm = __ballot_sync(0xffffffffu, head);
    const uint32_t below = hm & (0xffffffffu >> (31 - lane));  // heads at or below this lane
    const int rank = below ? lane - (31 - __clz(below)) : carry_cnt + lane;
    if (kPass == 0) {
      // last element of a run (next lane starts a new run, or end of the chunk's valid part)
      const int wnext = __shfl_down_sync(0xffffffffu, w, 1);
      const bool last = has && (lane == 31 || wnext != w);
      // a run that continues into the next chunk is overwritten there with the larger count
      if (last) wpi[(size_t)w * (t + 1) + b] = rank + 1;
    } else if (has) {
      pos[wd & 0x7fffffffu] = (uint32_t)(wpi[(size_t)w * (t + 1) + b] + rank) | (wd & 0x80000000u);
    }
    carry_w = __shfl_sync(0xffffffffu, w, 31);
    carry_cnt = __shfl_sync(0xffffffffu, rank, 31) + 1;
  }
}

// exclusive scan over the t + 1 entries of every window (one CTA per window;
// entry t receives the window's row count)
__global__ void __launch_bounds__(1024) win_scan_kernel(int32_t *__restrict__ wpi, uint64_t t) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry_s, tot_s;
  int32_t *row = wpi + (size_t)blockIdx.x * (t + 1);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint64_t base = 0; base < t + 1; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const int32_t v = i < t ? row[i] : 0;
    int32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int32_t x = wsum[lane];
      int32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      wsum[lane] = xi - x;
      if (lane == 31) tot_s = xi;
    }
    __syncthreads();
    const int32_t c = carry_s;
    if (i <= t) row[i] = c + wsum[wid] + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = c + tot_s;
    __syncthreads();
  }
}

}  // namespace
}  // namespace skt
