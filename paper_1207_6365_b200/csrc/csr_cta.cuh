// csr_cta.cuh -- K4 "window gather" kernel for canonical CSR with narrow d
// (BASELINE config 4): every SM owns a contiguous bucket range with its fp64
// accumulators in shared memory and walks A window by window.
//
// The window plan (apply_csr_window.cu) sorts the rows of every W-row window
// stably by bucket: wrows[w*W + p] = row | sign << 31, wpi[w][b] = first rank
// of bucket b in window w.  CTA c owns buckets [c*B, (c+1)*B); its rows of a
// window are ONE contiguous range of wrows.  All CTAs walk the windows in the
// same order, so the rows being gathered at any moment lie in a narrow band
// of A: DRAM pages and the 128-byte lines shared by neighbouring rows are
// fetched once and hit in L2 for the other CTAs (the access pattern runs
// 0.16 ms on config 4 in this order vs 0.24 ms in bucket order,
// profiles/r01_gather_windows.txt), without any hand-off between CTAs.
//
// Inside a CTA the gather is decoupled from the ordered accumulation:
//  * loader warps copy each row's index / value entries straight into a
//    128-byte shared-memory slot with 4-byte cp.async (no registers held while
//    the data is in flight; completion is counted on an mbarrier by
//    cp.async.mbarrier.arrive), rounds of up to kCtaRing rows double-buffered,
//    row ids and indptr pairs loaded one round ahead;
//  * accumulating warps: each HALF warp owns buckets h, h + 2A, ... and adds
//    its buckets' rows in ascending row order, 16 lanes = the 16 entries of a
//    slot, acc[col] += v on the fp64 accumulators in shared memory (columns
//    are distinct inside a canonical row; the two halves of a warp work on
//    different buckets).  Per output element the additions run in ascending
//    row order from +0.0: bit-identical to the reference's bincount
//    (sketch.py:155-164).
// Rows longer than a slot are read from A by the accumulating half warp.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace skt {
namespace {

constexpr int kCtaLoad = 8;    // loader warps
constexpr int kCtaAcc = 16;    // accumulating warps (32 half warps)
constexpr int kCtaThreads = (kCtaLoad + kCtaAcc) * 32;
#ifndef SKT_CTA_RING
#define SKT_CTA_RING 288
#endif
#ifndef SKT_CTA_BUFS
#define SKT_CTA_BUFS 4
#endif
constexpr int kCtaRing = SKT_CTA_RING;  // rows per round (slots of one buffer), a multiple of 32
constexpr int kCtaBufs = SKT_CTA_BUFS;
constexpr int kCtaChunks = kCtaRing / 32;                            // chunks of 32 rows per round
constexpr int kCtaCpl = (kCtaChunks + kCtaLoad - 1) / kCtaLoad;      // chunks per loader warp and round
constexpr uint32_t kCtaLong = 0xffu;

struct CtaParams {
  const void *aip;
  const int32_t *aix;
  const float *av;
  int64_t n;
  int d, dp;
  uint64_t t;
  const uint32_t *wrows;  // [n]: rows of every window stably sorted by bucket, sign in bit 31
  const int32_t *wpi;     // [nwin][t + 1]
  int32_t W, nwin, bpc;   // rows per window, windows, buckets per CTA
  void *sa;
  int64_t ldsa;
};

__device__ __forceinline__ uint32_t ct_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ct_mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(ct_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void ct_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(ct_smem(bar)) : "memory");
}
__device__ __forceinline__ void ct_mbar_arrive_cpasync(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(ct_smem(bar)) : "memory");
}
__device__ __forceinline__ void ct_mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
          ct_smem(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void ct_cp4(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ uint32_t ct_lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 ct_lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double ct_ldsf64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
// acc[a] += v when on (one predicated load / add / store, no branch)
__device__ __forceinline__ void ct_acc_add(uint32_t a, double v, bool on) {
  asm volatile(
      "{ .reg .pred p; .reg .f64 t; setp.ne.u32 p, %2, 0; @p ld.shared.f64 t, [%0]; @p add.f64 t, t, %1; "
      "@p st.shared.f64 [%0], t; }" ::"r"(a),
      "d"(v), "r"((uint32_t)on)
      : "memory");
}
__device__ __forceinline__ void ct_stsf64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// The CTA's rounds: window w contributes its rank range [lo_w, hi_w) cut into
// pieces of <= kCtaRing rows.  Both roles step through the same sequence.
struct CtaRounds {
  const int32_t *wpi;
  uint64_t t;
  int64_t b_lo, b_hi;  // the CTA's buckets
  int nwin, w, r0, hi;
  int nlo, nhi;  // the next window's range, loaded one window ahead
  __device__ void range(int win, int &lo, int &h) const {
    lo = h = 0;
    if (win < nwin && b_lo < b_hi) {
      lo = __ldg(wpi + (size_t)win * (t + 1) + b_lo);
      h = __ldg(wpi + (size_t)win * (t + 1) + b_hi);
    }
  }
  __device__ void start() {
    w = 0;
    range(0, r0, hi);
    range(1, nlo, nhi);
    skip_empty();
  }
  __device__ void skip_empty() {
    while (w < nwin && r0 >= hi) {
      ++w;
      r0 = nlo;
      hi = nhi;
      range(w + 1, nlo, nhi);
    }
  }
  __device__ bool done() const { return w >= nwin; }
  __device__ int r1() const { return hi - r0 < kCtaRing ? hi : r0 + kCtaRing; }
  __device__ void next() {
    r0 = r1();
    skip_empty();
  }
};

template <typename IP, typename TOut>
__global__ void __launch_bounds__(kCtaThreads, 1) csr_cta_kernel(const CtaParams p) {
  extern __shared__ __align__(128) unsigned char ct_raw[];
  __shared__ __align__(8) uint64_t full[kCtaBufs], empty[kCtaBufs];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const IP *__restrict__ aip = (const IP *)p.aip;
  const int32_t *__restrict__ aix = p.aix;
  const float *__restrict__ av = p.av;
  // [buf][slot][16 x (col, val)] | [buf][slot] meta | acc [bpc][dp]
  unsigned char *slots = ct_raw;
  uint32_t *meta = (uint32_t *)(ct_raw + (size_t)kCtaBufs * kCtaRing * 128);
  double *acc = (double *)(meta + kCtaBufs * kCtaRing);
  const int dp = p.dp, d = p.d;

  for (int i = threadIdx.x; i < p.bpc * dp; i += kCtaThreads) acc[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kCtaBufs; ++b) {
      ct_mbar_init(&full[b], kCtaLoad * 32 + kCtaLoad);  // one copy-completion arrival per loader thread + one per warp
      ct_mbar_init(&empty[b], kCtaAcc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  CtaRounds it;
  it.wpi = p.wpi;
  it.t = p.t;
  it.b_lo = (int64_t)blockIdx.x * p.bpc;
  it.b_hi = it.b_lo + p.bpc < (int64_t)p.t ? it.b_lo + p.bpc : (int64_t)p.t;
  if (it.b_lo > it.b_hi) it.b_lo = it.b_hi;
  it.nwin = p.nwin;
  it.start();

  if (warp < kCtaLoad) {
    // ------------------------------------------------------------ loaders
    typedef typename std::conditional<sizeof(IP) == 4, int32_t, int64_t>::type E;
    const int g = lane >> 4, gl = lane & 15;
    // This warp's chunks of a round: chunk warp + kCtaLoad * k, lane = row.
    // Plan words are loaded two rounds ahead, indptr pairs one round ahead.
    constexpr uint32_t kNoRow = 0xffffffffu;
    auto load_rows = [&](const CtaRounds &r, uint32_t (&wr)[kCtaCpl]) {
#pragma unroll
      for (int k = 0; k < kCtaCpl; ++k) {
        wr[k] = kNoRow;
        if (!r.done()) {
          const int rank = r.r0 + 32 * (warp + kCtaLoad * k) + lane;
          if (rank < r.r1()) wr[k] = __ldg(p.wrows + (size_t)r.w * p.W + rank);
        }
      }
    };
    auto load_aip = [&](const uint32_t (&wr)[kCtaCpl], E (&rs)[kCtaCpl], int (&len)[kCtaCpl]) {
#pragma unroll
      for (int k = 0; k < kCtaCpl; ++k) {
        rs[k] = 0;
        len[k] = -1;  // no row
        if (wr[k] != kNoRow) {
          const int64_t row = wr[k] & 0x7fffffffu;
          rs[k] = (E)aip[row];
          len[k] = (int)((E)aip[row + 1] - rs[k]);
        }
      }
    };
    CtaRounds n1 = it;
    n1.next();
    CtaRounds n2 = n1;
    n2.next();
    uint32_t wr_c[kCtaCpl], wr_n[kCtaCpl];
    E rs_c[kCtaCpl];
    int len_c[kCtaCpl];
    load_rows(it, wr_c);
    load_rows(n1, wr_n);
    load_aip(wr_c, rs_c, len_c);
    uint32_t q = 0;
    while (!it.done()) {
      const int buf = q % kCtaBufs;
      const uint32_t ph = (q / kCtaBufs) & 1u;
      ct_mbar_wait(&empty[buf], ph ^ 1u);
      const uint32_t sbase = ct_smem(slots + (size_t)buf * kCtaRing * 128);
      uint32_t *mb = meta + buf * kCtaRing;
#pragma unroll
      for (int k = 0; k < kCtaCpl; ++k) {
        const int slot0 = 32 * (warp + kCtaLoad * k);
        if (slot0 < kCtaRing) {  // compile-time chunk bound for the last k
          // lane r: its row's meta word (entries | sign << 8), long rows: start in the slot
          if (len_c[k] >= 0) {
            const bool is_long = len_c[k] > 16;
            mb[slot0 + lane] = (is_long ? kCtaLong : (uint32_t)len_c[k]) | ((wr_c[k] >> 31) << 8);
            if (is_long) {
              uint32_t *sl = (uint32_t *)(slots + ((size_t)buf * kCtaRing + slot0 + lane) * 128);
              sl[0] = (uint32_t)rs_c[k];
              sl[1] = (uint32_t)((uint64_t)rs_c[k] >> 32);
              sl[2] = (uint32_t)len_c[k];
            }
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int r = 2 * i + g;
            const E rs_r = __shfl_sync(0xffffffffu, rs_c[k], r);
            const int len_r = __shfl_sync(0xffffffffu, len_c[k], r);
            if (gl < len_r && len_r <= 16) {
              const uint32_t dst = sbase + (uint32_t)(slot0 + r) * 128u + gl * 8;
              ct_cp4(dst, aix + rs_r + gl);
              ct_cp4(dst + 4, av + rs_r + gl);
            }
          }
        }
      }
      ct_mbar_arrive_cpasync(&full[buf]);  // fires when this thread's copies have landed
      __syncwarp();
      if (lane == 0) ct_mbar_arrive(&full[buf]);  // releases the meta words
      // rotate: next round's indptr pairs (its plan words arrived a round ago),
      // the round after's plan words
#pragma unroll
      for (int k = 0; k < kCtaCpl; ++k) wr_c[k] = wr_n[k];
      load_aip(wr_c, rs_c, len_c);
      load_rows(n2, wr_n);
      it = n1;
      n1 = n2;
      n2.next();
      ++q;
    }
  } else {
    // ------------------------------------------------------------ accumulate
    const int aw = warp - kCtaLoad;
    const int half = lane >> 4, j = lane & 15;
    const int h = aw * 2 + half;  // this half warp's buckets: h, h + 2A, ...
    constexpr int kHalves = 2 * kCtaAcc;
    const int nbk = (int)(it.b_hi - it.b_lo);
    const int kmax = (nbk + kHalves - 1) / kHalves;  // <= 8 (the host checks bpc)
    uint32_t q = 0;
    while (!it.done()) {
      const int buf = q % kCtaBufs;
      const uint32_t ph = (q / kCtaBufs) & 1u;
      const int r0 = it.r0, r1 = it.r1();
      const int32_t *wp = p.wpi + (size_t)it.w * (p.t + 1) + it.b_lo;
      // rank bounds of this half warp's buckets: lane 2k holds off[b_k], lane 2k+1 off[b_k + 1]
      int offv = 0;
      {
        const int kk = j >> 1, b = h + kHalves * kk;
        if (kk < kmax && b < nbk) offv = __ldg(wp + b + (j & 1));
      }
      ct_mbar_wait(&full[buf], ph);
      const unsigned char *sb = slots + (size_t)buf * kCtaRing * 128;
      const uint32_t sb_u = ct_smem(sb) + j * 8, mb_u = ct_smem(meta + buf * kCtaRing), acc_u = ct_smem(acc);
      for (int kk = 0; kk < kmax; ++kk) {
        const int b = h + kHalves * kk;
        const int o0 = __shfl_sync(0xffffffffu, offv, (lane & 16) + 2 * kk);
        const int o1 = __shfl_sync(0xffffffffu, offv, (lane & 16) + 2 * kk + 1);
        int s0 = 0, s1 = 0;
        if (b < nbk) {
          s0 = (o0 > r0 ? o0 : r0) - r0;
          s1 = (o1 < r1 ? o1 : r1) - r0;
          if (s1 < s0) s1 = s0;
        }
        const int mylen = s1 - s0;
        const int other = __shfl_xor_sync(0xffffffffu, mylen, 16);
        const int steps = mylen > other ? mylen : other;
        const uint32_t ab_u = acc_u + (uint32_t)(b < nbk ? b : 0) * (uint32_t)dp * 8u;
        uint32_t ma = mb_u + (uint32_t)s0 * 4u, sa_u = sb_u + (uint32_t)s0 * 128u;
        // the next row's meta word and entry are fetched one step ahead
        const int last = mylen > 0 ? mylen - 1 : 0;
        uint32_t m_n = ct_lds32(ma);
        uint2 e_n = ct_lds64(sa_u);
        for (int r = 0; r < steps; ++r) {
          const uint32_t m = m_n;
          const uint2 e = e_n;
          {  // unconditional (clamped) loads: no branch inside the step
            const uint32_t rn = (uint32_t)(r + 1 < mylen ? r + 1 : last);
            m_n = ct_lds32(ma + 4u * rn);
            e_n = ct_lds64(sa_u + 128u * rn);
          }
          const uint32_t len = m & 0xffu;
          const bool live = r < mylen;
          const bool is_long = live && len == kCtaLong;
          ct_acc_add(ab_u + e.x * 8u, (double)__uint_as_float(e.y ^ ((m >> 8) << 31)),
                     live && !is_long && (uint32_t)j < len);
          if (__any_sync(0xffffffffu, is_long)) {  // a row longer than a slot: straight from A, 16 entries per step
            if (is_long) {
              const uint32_t *sl = reinterpret_cast<const uint32_t *>(sb + (size_t)(s0 + r) * 128);
              const int64_t rs = (int64_t)(((uint64_t)sl[1] << 32) | sl[0]);
              const int rl = (int)sl[2];
              const bool neg = (m >> 8) != 0;
              for (int qq = j; qq < rl; qq += 16) {
                const float x = __ldg(av + rs + qq);
                const uint32_t a = ab_u + (uint32_t)__ldg(aix + rs + qq) * 8u;
                ct_stsf64(a, ct_ldsf64(a) + (double)(neg ? -x : x));
              }
            }
          }
          __syncwarp();
        }
      }
      __syncwarp();
      if (lane == 0) ct_mbar_arrive(&empty[buf]);
      it.next();
      ++q;
    }
  }
  __syncthreads();
  // ---- write SA
  TOut *sa = (TOut *)p.sa;
  const int nbk = (int)(it.b_hi - it.b_lo);
  for (int i = threadIdx.x; i < nbk * d; i += kCtaThreads) {
    const int b = i / d, c = i - b * d;
    sa[(it.b_lo + b) * p.ldsa + c] = (TOut)acc[(size_t)b * dp + c];
  }
}

// wrows[w * W + rank] = row | sign: the inverse of the window plan's pos[]
__global__ void __launch_bounds__(256) win_rows_kernel(const uint32_t *__restrict__ pos, int64_t n, int32_t W,
                                                       uint32_t *__restrict__ wrows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t pw = pos[i];
  wrows[(i / W) * W + (pw & 0x7fffffffu)] = (uint32_t)i | (pw & 0x80000000u);
}

}  // namespace
}  // namespace skt
