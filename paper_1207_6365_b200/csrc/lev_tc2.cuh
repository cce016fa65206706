// lev_tc2.cuh -- K5 v2: warp-specialised tcgen05 leverage contraction
// scores_i = || A_i . P ||^2 (reference leverage.py:90-91) for CSR A with fp32
// values and d <= 128, the CSR tiles streamed into shared memory by the
// bulk-copy engine and the products taken as scaled 2xFP16 on the tensor cores.
//
// Numerics.  Row i of a tile is scaled by 2^-e_i (e_i = frexp exponent of the
// row's largest |a|, so every scaled entry is < 1) and P by one 2^-f; both are
// split into fp16 hi + lo parts (hi = fp16(x), lo = fp16(x - hi): 22
// significant bits).  A row is stored with hi and lo INTERLEAVED along K
// (element 2c = hi(a_c), 2c+1 = lo(a_c): one 32-bit store per nonzero), and
// the B operand has two halves: rows 0..k-1 hold (P_hi[c], P_hi[c]) at
// (2c, 2c+1), rows k..2k-1 hold (P_lo[c], 0).  One N = 2k MMA per K step then
// yields A_hi P_hi + A_lo P_hi in columns 0..k-1 and A_hi P_lo in k..2k-1 (the
// dropped A_lo P_lo term is ~2^-22 relative), fp32 accumulation in TMEM.  The
// epilogue adds the halves, squares and sums in fp64 and rescales by the exact
// power of two 2^(2(e_i + f)).
//
// Producer warp (8).  A 128-row tile of CSR is one contiguous range of
// indices / values [indptr[row0], indptr[row0 + 128]) plus a 128-entry slice
// of indptr, so the tile is staged with three 1D bulk copies (cp.async.bulk
// global->shared, completion counted in bytes on the stage's "full" mbarrier)
// into a ring of stages; nst - 1 tiles stay in flight per SM without a
// register per nonzero.  The copies start at the 16-byte floor of each range;
// the <16-byte tail after the last whole chunk is loaded by the producer lane
// that prefetched the tile's bounds (32 tiles ahead) and stored beside it.
//
// MMA warp (9).  Waits for a densified A buffer ("a_full"), issues the tile's
// tcgen05.mma.kind::f16 chain into TMEM accumulator i&1, commits to mma_bar.
//
// Consumer warps (0-7).  Warp w densifies rows 16w..16w+15 of a landed tile,
// two rows at a time (a half-warp per row; the 8 row pairs in lock-step phases
// so their latencies overlap) into the 128B-swizzled K-major A buffer i&1,
// releases the stage and signals the MMA warp; then finishes tile i-1: warps
// 0-3 reduce its accumulator rows (tcgen05.ld 32x32b), warps 4-7 clear its A
// buffer.  Rows whose column indices are not strictly increasing (duplicates,
// unsorted) are rebuilt by their warp one lane per row in entry order, summing
// duplicates (scipy's a @ probe semantics).  Tiles whose range exceeds a stage
// are densified straight from global memory.
#pragma once

#include <cuda_fp16.h>

#include "lev_tc.cuh"

namespace skt {
namespace {

constexpr int kT2Consumers = 8;
constexpr int kT2ProducerWarp = kT2Consumers, kT2MmaWarp = kT2Consumers + 1;
constexpr int kT2Threads = (kT2Consumers + 2) * 32;
constexpr int kT2MaxStages = 4;
constexpr uint32_t kT2IpBytes = 1040;  // 129 x 8 B rounded up to 16 B

struct T2Layout {
  int dk;                // columns of A padded to a multiple of 32 (K of the MMA = 2 dk)
  int merged;            // one N = 2k MMA per K step (2k <= 256), else two N = k MMAs
  uint32_t a_bytes;      // one A buffer: 128 x 2dk fp16
  uint32_t p_bytes;      // the 2k-row B operand: 2k x 2dk fp16
  uint32_t stage_bytes, idx_off, val_off;
  uint32_t tm_cols;      // TMEM columns per accumulator buffer
  uint32_t tm_alloc;     // TMEM columns allocated
  int cap, nst;
  size_t smem;
};

__device__ __forceinline__ void t2_mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void t2_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(tc_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void t2_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void t2_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
          tc_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void t2_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void t2_consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kT2Consumers * 32) : "memory");
}
// fp16 x fp16 -> fp32, K-major A and B, N = n, M = 128
__host__ __device__ constexpr uint32_t t2_idesc(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void t2_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
// A tile: 128 rows x 2dk fp16, K-major, 128-byte swizzle (8-row x 64-element
// atoms of 1 KB, 16 atoms down the rows, one 16 KB atom column per 64 K).
// Word index of column pair c (fp16 elements 2c, 2c+1) of row r:
__device__ __forceinline__ uint32_t t2_a_word(int r, int c) {
  return (uint32_t)((c >> 5) * 4096 + (r >> 3) * 256 + (r & 7) * 32 + ((((c & 31) >> 2) ^ (r & 7)) << 2) + (c & 3));
}
// B operand (rows = N), fp16, K-major, no swizzle: core matrix 8 rows x 16 B
// (8 elements), LBO = R * 16 between K core matrices
__device__ __forceinline__ uint32_t t2_p_off(int r, int kk, int R) {
  return (uint32_t)((kk >> 3) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2);
}
// (hi, lo) fp16 split of x packed as one word, hi in the low half (element 2c)
__device__ __forceinline__ uint32_t t2_pack(float x) {
  const float hf = __half2float(__float2half_rn(x));
  const __half2 p = __floats2half2_rn(hf, x - hf);
  return *(const uint32_t *)&p;
}
__device__ __forceinline__ float t2_unpack(uint32_t w) {
  const __half2 p = *(const __half2 *)&w;
  return __low2float(p) + __high2float(p);
}
// frexp exponent of m (m in [2^(e-1), 2^e)) clamped so that 2^-e is a normal
// float; 0 for non-finite m (left unscaled)
__device__ __forceinline__ int t2_exp(float m) {
  const int be = (__float_as_int(m) >> 23) & 0xff;
  return be == 0xff ? 0 : (be - 126 > 126 ? 126 : be - 126);
}
// 8 TMEM columns of this warp's 32 lanes
#define T2_TMEM_LD8(taddr, v, o)                                                                   \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"           \
               : "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), \
                 "=r"(v[o + 5]), "=r"(v[o + 6]), "=r"(v[o + 7])                                    \
               : "r"(taddr))

// Densify this warp's 16 rows (two per step, a half-warp per row) of a tile
// into the interleaved A buffer.  idx / val point at the tile's first nonzero
// (shared-memory stage, or global memory when kGlobal); q0 / q1 are the rows'
// bounds relative to it.  Returns true when a row's columns are not strictly
// increasing.
template <bool kGlobal, typename IX>
__device__ __forceinline__ bool t2_densify(const IX *idx, const float *val, const int *q0, const int *q1,
                                           int r0, int lane, uint32_t *a, int *rexp_b, int rows) {
  const int half = lane >> 4, gl = lane & 15;
  int c[8];
  float v[8], m[8];
  bool dirty = false;
  uint32_t longm = 0;
#pragma unroll
  for (int pr = 0; pr < 8; ++pr) {  // the row's first 16 nonzeros (most rows: all of them)
    const int q = q0[pr] + gl;
    c[pr] = -1;
    v[pr] = 0.f;
    if (q < q1[pr]) {
      c[pr] = kGlobal ? (int)__ldg(idx + q) : (int)idx[q];
      v[pr] = kGlobal ? __ldg(val + q) : val[q];
    }
    if (q1[pr] - q0[pr] > 16) longm |= 1u << pr;
  }
#pragma unroll
  for (int pr = 0; pr < 8; ++pr) {
    const int cprev = __shfl_up_sync(0xffffffffu, c[pr], 1, 16);
    dirty |= gl > 0 && c[pr] >= 0 && c[pr] <= cprev;
    m[pr] = fabsf(v[pr]);
  }
  if (longm) {  // rest of the long rows: max and order
#pragma unroll
    for (int pr = 0; pr < 8; ++pr) {
      if (longm >> pr & 1) {
        for (int q = q0[pr] + gl + 16; q < q1[pr]; q += 16) {
          const int cc = kGlobal ? (int)__ldg(idx + q) : (int)idx[q];
          const int cp = kGlobal ? (int)__ldg(idx + q - 1) : (int)idx[q - 1];
          dirty |= cc <= cp;
          m[pr] = fmaxf(m[pr], fabsf(kGlobal ? __ldg(val + q) : val[q]));
        }
      }
    }
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
#pragma unroll
    for (int pr = 0; pr < 8; ++pr) m[pr] = fmaxf(m[pr], __shfl_xor_sync(0xffffffffu, m[pr], o, 16));
  }
#pragma unroll
  for (int pr = 0; pr < 8; ++pr) {
    const int r = r0 + pr * 2 + half;
    const int ex = t2_exp(m[pr]);
    const float sc = __int_as_float((127 - ex) << 23);
    if (gl == 0 && r < rows) rexp_b[r] = ex;
    if (c[pr] >= 0) a[t2_a_word(r, c[pr])] = t2_pack(v[pr] * sc);
    if (longm >> pr & 1) {
      for (int q = q0[pr] + gl + 16; q < q1[pr]; q += 16) {
        const int cc = kGlobal ? (int)__ldg(idx + q) : (int)idx[q];
        const float vv = kGlobal ? __ldg(val + q) : val[q];
        a[t2_a_word(r, cc)] = t2_pack(vv * sc);
      }
    }
  }
  return dirty;
}

// Phase timers for tools/lev_prof.cu (compiled out of the library).
#ifdef SKT_T2_PROF
__device__ unsigned long long g_t2_prof[16];
#define T2P_DECL long long t2p_last = clock64(), t2p_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define T2P(i)                                  \
  do {                                          \
    const long long t2p_now = clock64();        \
    t2p_acc[i] += t2p_now - t2p_last;           \
    t2p_last = t2p_now;                         \
  } while (0)
#define T2P_FLUSH(base, cond)                                                                          \
  do {                                                                                                 \
    if (cond)                                                                                          \
      for (int i_ = 0; i_ < 8; ++i_) atomicAdd(&g_t2_prof[(base) + i_], (unsigned long long)t2p_acc[i_]); \
  } while (0)
#else
#define T2P_DECL
#define T2P(i) \
  do {         \
  } while (0)
#define T2P_FLUSH(base, cond) \
  do {                        \
  } while (0)
#endif

template <typename IP, typename IX, typename TS>
__global__ void __launch_bounds__(kT2Threads, 1)
    lev_tc2_kernel(int64_t n, int d, const IP *__restrict__ aip, const IX *__restrict__ aix,
                   const float *__restrict__ av, const double *__restrict__ probe, int k,
                   TS *__restrict__ scores, T2Layout L) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[kT2MaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kT2MaxStages];
  __shared__ __align__(8) uint64_t afull_bar[2];
  __shared__ __align__(8) uint64_t mma_bar[2];
  __shared__ uint32_t tmem_base;
  __shared__ int rexp[2][kTcRows];  // per-row scale exponents of the two A buffers
  __shared__ float pmax_w[kT2Threads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int dk = L.dk;
  unsigned char *p_op = smem + 2 * L.a_bytes;  // A buffers 0, 1 first
  unsigned char *stages = p_op + L.p_bytes;
  constexpr int kCi = 16 / (int)sizeof(IX);  // index elements per 16-byte chunk
  constexpr int kCv = 4;                     // fp32 values per 16-byte chunk
  const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
  const int nst = L.nst;
  const int64_t cap = L.cap;

  // ---- one-time setup (all warps): zero both A buffers, stage the scaled B
  // operand, TMEM, barriers
  for (uint32_t i = tid; i < (2 * L.a_bytes + L.p_bytes) / 16; i += kT2Threads)
    ((uint4 *)smem)[i] = make_uint4(0, 0, 0, 0);
  float pm = 0.f;
  for (int i = tid; i < d * k; i += kT2Threads) pm = fmaxf(pm, (float)fabs(probe[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, o));
  if (lane == 0) pmax_w[warp] = pm;
  __syncthreads();
  pm = 0.f;
  for (int w = 0; w < kT2Threads / 32; ++w) pm = fmaxf(pm, pmax_w[w]);
  const int pe = t2_exp(pm);
  for (int i = tid; i < k * d; i += kT2Threads) {
    const int col = i / d, c = i % d;  // B row col <- P[c][col]
    const float x = (float)(probe[(int64_t)c * k + col] * __longlong_as_double((long long)(1023 - pe) << 52));
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    *(__half *)(p_op + t2_p_off(col, 2 * c, 2 * k)) = h;
    *(__half *)(p_op + t2_p_off(col, 2 * c + 1, 2 * k)) = h;
    *(__half *)(p_op + t2_p_off(k + col, 2 * c, 2 * k)) = l;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc_smem_u32(&tmem_base)),
                 "r"(L.tm_alloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      t2_mbar_init(&full_bar[s], 1);
      t2_mbar_init(&empty_bar[s], kT2Consumers);
    }
    for (int b = 0; b < 2; ++b) {
      t2_mbar_init(&afull_bar[b], kT2Consumers);
      t2_mbar_init(&mma_bar[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == kT2ProducerWarp) {
    // =================== producer warp ===================
    // lane j prefetches the bounds (and the <16-byte tails) of the tile 32
    // iterations ahead; the batch after next is requested at j == 0, its tails
    // at j == 16 once the bounds have landed.
    int64_t b_s = 0, b_e = 0, n_s = 0, n_e = 0;
    IX b_ti[kCi - 1], n_ti[kCi - 1];
    float b_tv[kCv - 1], n_tv[kCv - 1];
    auto bounds = [&](int64_t it, int64_t &s, int64_t &e) {
      const int64_t tile = blockIdx.x + it * (int64_t)gridDim.x;
      s = e = 0;
      if (tile < ntiles) {
        const int64_t row0 = tile * kTcRows;
        const int64_t rows = n - row0 < kTcRows ? n - row0 : kTcRows;
        s = (int64_t)aip[row0];
        e = (int64_t)aip[row0 + rows];
      }
    };
    auto tails = [&](int64_t e, IX *ti, float *tv) {
      const int64_t fi = e & ~(int64_t)(kCi - 1), fv = e & ~(int64_t)(kCv - 1);
#pragma unroll
      for (int q = 0; q < kCi - 1; ++q) ti[q] = fi + q < e ? aix[fi + q] : (IX)0;
#pragma unroll
      for (int q = 0; q < kCv - 1; ++q) tv[q] = fv + q < e ? av[fv + q] : 0.f;
    };
    T2P_DECL
    bounds(lane, b_s, b_e);
    tails(b_e, b_ti, b_tv);
    int st = 0;
    uint32_t ph = 1;  // empty barriers: the first pass over the ring does not wait
    for (int64_t it = 0;; ++it) {
      const int64_t tile = blockIdx.x + it * (int64_t)gridDim.x;
      if (tile >= ntiles) break;
      const int j = (int)(it & 31);
      if (j == 0 && it > 0) {
        b_s = n_s;
        b_e = n_e;
#pragma unroll
        for (int q = 0; q < kCi - 1; ++q) b_ti[q] = n_ti[q];
#pragma unroll
        for (int q = 0; q < kCv - 1; ++q) b_tv[q] = n_tv[q];
      }
      if (j == 0) bounds(it + 32 + lane, n_s, n_e);
      if (j == 16) tails(n_e, n_ti, n_tv);
      const int64_t s = __shfl_sync(0xffffffffu, b_s, j);
      const int64_t e = __shfl_sync(0xffffffffu, b_e, j);
      const int64_t row0 = tile * kTcRows;
      const int rows = (int)(n - row0 < kTcRows ? n - row0 : kTcRows);
      unsigned char *sb = stages + (size_t)st * L.stage_bytes;
      IP *sip = (IP *)sb;
      IX *six = (IX *)(sb + L.idx_off);
      float *sva = (float *)(sb + L.val_off);
      T2P(0);
      t2_wait(&empty_bar[st], ph);
      T2P(1);
      const int64_t fi0 = s & ~(int64_t)(kCi - 1), fv0 = s & ~(int64_t)(kCv - 1);
      const int64_t fi1 = e & ~(int64_t)(kCi - 1), fv1 = e & ~(int64_t)(kCv - 1);
      const bool over = e - fi0 > cap || e - fv0 > cap;
      if (rows < kTcRows) {  // last, partial tile: indptr by plain loads
        for (int r = lane; r <= rows; r += 32) sip[r] = aip[row0 + r];
      } else if (lane == j) {
        sip[kTcRows] = (IP)e;
      }
      if (!over && lane == j) {
#pragma unroll
        for (int q = 0; q < kCi - 1; ++q)
          if (fi1 + q < e) six[fi1 - fi0 + q] = b_ti[q];
#pragma unroll
        for (int q = 0; q < kCv - 1; ++q)
          if (fv1 + q < e) sva[fv1 - fv0 + q] = b_tv[q];
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t ib = rows == kTcRows ? (uint32_t)(kTcRows * sizeof(IP)) : 0u;
        const uint32_t xb = over ? 0u : (uint32_t)((fi1 - fi0) * (int64_t)sizeof(IX));
        const uint32_t vb = over ? 0u : (uint32_t)((fv1 - fv0) * 4);
        t2_arrive_tx(&full_bar[st], ib + xb + vb);
        if (ib) t2_bulk(sip, aip + row0, ib, &full_bar[st]);
        if (xb) t2_bulk(six, aix + fi0, xb, &full_bar[st]);
        if (vb) t2_bulk(sva, av + fv0, vb, &full_bar[st]);
      }
      __syncwarp();
      if (++st == nst) {
        st = 0;
        ph ^= 1u;
      }
      T2P(2);
    }
    T2P_FLUSH(8, lane == 0);
    return;
  }

  if (warp == kT2MmaWarp) {
    // =================== MMA warp ===================
    const uint32_t idesc = t2_idesc(L.merged ? 2 * k : k);
    const uint32_t lbo_p = (uint32_t)(2 * k) * 16;
    const uint32_t pb = tc_smem_u32(p_op);
    const uint32_t plo = pb + (uint32_t)(k / 8) * 128;  // rows k.. of the 2k-row operand
    const uint64_t sw128 = (uint64_t)2 << 61;
    for (int64_t it = 0;; ++it) {
      const int64_t tile = blockIdx.x + it * (int64_t)gridDim.x;
      if (tile >= ntiles) break;
      const int b = (int)(it & 1);
      t2_wait(&afull_bar[b], (uint32_t)((it >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t d_t = tmem + (uint32_t)b * L.tm_cols;
        const uint32_t ab = tc_smem_u32(smem + (size_t)b * L.a_bytes);
        for (int ks = 0; ks < dk / 8; ++ks) {  // K = 2 dk in steps of 16
          const uint64_t da = tc_desc(ab + (uint32_t)(ks >> 2) * 16384 + (uint32_t)(ks & 3) * 32, 16, 1024) | sw128;
          const uint32_t op = (uint32_t)ks * 2 * lbo_p;
          t2_mma(d_t, da, tc_desc(pb + op, lbo_p, 128), idesc, ks > 0);
          if (!L.merged) t2_mma(d_t, da, tc_desc(plo + op, lbo_p, 128), idesc, 1);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         tc_smem_u32(&mma_bar[b]))
                     : "memory");
      }
      __syncwarp();
    }
    return;
  }

  // =================== consumer warps 0..7 ===================
  const int half = lane >> 4;
  T2P_DECL
  int st = 0;
  uint32_t ph = 0;
  for (int64_t it = 0;; ++it) {
    const int64_t tile = blockIdx.x + it * (int64_t)gridDim.x;
    const bool have = tile < ntiles;
    const int b = (int)(it & 1);
    uint32_t *a = (uint32_t *)(smem + (size_t)b * L.a_bytes);
    T2P(7);
    if (have) {
      const int64_t row0 = tile * kTcRows;
      const int rows = (int)(n - row0 < kTcRows ? n - row0 : kTcRows);
      unsigned char *sb = stages + (size_t)st * L.stage_bytes;
      const IP *sip = (const IP *)sb;
      const IX *six = (const IX *)(sb + L.idx_off);
      const float *sva = (const float *)(sb + L.val_off);
      t2_wait(&full_bar[st], ph);
      T2P(0);
      const int64_t s = (int64_t)sip[0], e = (int64_t)sip[rows];
      const int pi = (int)(s & (kCi - 1)), pv = (int)(s & (kCv - 1));
      const bool over = e - (s - pi) > cap || e - (s - pv) > cap;
      const int r0 = warp * 16;
      int q0[8], q1[8];
#pragma unroll
      for (int pr = 0; pr < 8; ++pr) {
        const int r = r0 + pr * 2 + half;
        q0[pr] = q1[pr] = 0;
        if (r < rows) {
          q0[pr] = (int)((int64_t)sip[r] - s);
          q1[pr] = (int)((int64_t)sip[r + 1] - s);
        }
      }
      const bool dirty = over ? t2_densify<true>(aix + s, av + s, q0, q1, r0, lane, a, rexp[b], rows)
                              : t2_densify<false>(six + pi, sva + pv, q0, q1, r0, lane, a, rexp[b], rows);
      T2P(1);
      // the stage is consumed (a dirty rebuild re-reads global memory)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) t2_arrive(&empty_bar[st]);
      if (++st == nst) {
        st = 0;
        ph ^= 1u;
      }
      if (__any_sync(0xffffffffu, dirty)) {
        // rebuild the warp's 16 rows: clear them, then one lane per row,
        // entries in order, duplicates summed; scale from sum |a| (bounds any sum)
        for (int i = lane; i < 16 * (dk / 32) * 8; i += 32) {  // 16 rows x (dk/32 atoms) x 8 chunks
          const int rr = r0 + i / ((dk / 32) * 8), rest = i % ((dk / 32) * 8);
          const int ac = rest / 8, ch = rest % 8;
          *(uint4 *)(a + ac * 4096 + (rr >> 3) * 256 + (rr & 7) * 32 + ch * 4) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
        const int r = r0 + lane;
        if (lane < 16 && r < rows) {
          const int64_t rb = (int64_t)aip[row0 + r], re = (int64_t)aip[row0 + r + 1];
          float sum = 0.f;
          for (int64_t q = rb; q < re; ++q) sum += fabsf(av[q]);
          const int ex = t2_exp(sum);
          const float sc = __int_as_float((127 - ex) << 23);
          rexp[b][r] = ex;
          for (int64_t q = rb; q < re; ++q) {
            uint32_t *w = a + t2_a_word(r, (int)aix[q]);
            *w = t2_pack(av[q] * sc + t2_unpack(*w));
          }
        }
        __syncwarp();
      }
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) t2_arrive(&afull_bar[b]);
    }
    T2P(2);
    if (it > 0) {  // ---- finish tile it-1 (accumulator / A buffer b^1)
      const int pb = b ^ 1;
      const int64_t prow0 = (tile - gridDim.x) * kTcRows;
      t2_wait(&mma_bar[pb], (uint32_t)(((it - 1) >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      T2P(3);
      if (warp < 4) {  // TMEM lane = tile row = 32 * warp + lane
        double sc0 = 0.0, sc1 = 0.0, sc2 = 0.0, sc3 = 0.0;
        const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)pb * L.tm_cols;
        for (int c0 = 0; c0 < k; c0 += 32) {
          uint32_t u[32], w[32];
          const int g = (k - c0) >= 32 ? 4 : (k - c0) / 8;
#pragma unroll
          for (int gi = 0; gi < 4; ++gi) {
            if (gi < g) {
              T2_TMEM_LD8(base + (uint32_t)(c0 + 8 * gi), u, 8 * gi);
              if (L.merged) T2_TMEM_LD8(base + (uint32_t)(k + c0 + 8 * gi), w, 8 * gi);
            }
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int jj = 0; jj < 32; jj += 4) {
            if (jj < 8 * g) {
              float x0 = __uint_as_float(u[jj]), x1 = __uint_as_float(u[jj + 1]);
              float x2 = __uint_as_float(u[jj + 2]), x3 = __uint_as_float(u[jj + 3]);
              if (L.merged) {
                x0 += __uint_as_float(w[jj]);
                x1 += __uint_as_float(w[jj + 1]);
                x2 += __uint_as_float(w[jj + 2]);
                x3 += __uint_as_float(w[jj + 3]);
              }
              sc0 = fma((double)x0, (double)x0, sc0);
              sc1 = fma((double)x1, (double)x1, sc1);
              sc2 = fma((double)x2, (double)x2, sc2);
              sc3 = fma((double)x3, (double)x3, sc3);
            }
          }
        }
        const int row = warp * 32 + lane;
        const int64_t my_row = prow0 + row;
        // undo the scaling: x = x' 2^(e_i + f), an exact power of two in fp64
        const double unscale = __longlong_as_double((long long)(1023 + 2 * (rexp[pb][row] + pe)) << 52);
        if (my_row < n) scores[my_row] = (TS)(((sc0 + sc1) + (sc2 + sc3)) * unscale);
      } else {  // clear A buffer b^1 for tile it+1
        uint4 *z = (uint4 *)(smem + (size_t)pb * L.a_bytes);
        for (uint32_t i = tid - 128; i < L.a_bytes / 16; i += 128) z[i] = make_uint4(0, 0, 0, 0);
      }
      T2P(4);
    }
    if (!have) break;
    asm volatile("tcgen05.fence::before_thread_sync;");
    t2_consumer_sync();  // accumulator b^1 drained, A buffer b^1 clean, rexp[b^1] read
    T2P(5);
  }
  T2P_FLUSH(0, tid == 0);
  asm volatile("tcgen05.fence::before_thread_sync;");
  t2_consumer_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L.tm_alloc));
}

// Shared-memory / TMEM plan: two A buffers, the 2k-row B operand and the
// stage ring (cap nonzeros each).  nst = 0: does not fit (use lev_tc_kernel).
inline T2Layout lev_tc2_layout(int d, int k, int ix_bytes) {
  T2Layout L{};
  L.dk = (d + 31) & ~31;
  L.merged = 2 * k <= 256;
  L.a_bytes = (uint32_t)kTcRows * (2 * L.dk) * 2;
  L.p_bytes = (uint32_t)(2 * k) * (2 * L.dk) * 2;
  const uint32_t cols = (uint32_t)(L.merged ? 2 * k : k);
  L.tm_cols = (cols + 31) & ~31u;
  uint32_t alloc = 32;
  while (alloc < 2 * L.tm_cols) alloc <<= 1;
  L.tm_alloc = alloc;
  L.nst = 0;
  if (alloc > 512 || L.dk > 128) return L;
  const size_t budget = 232448 - 2048;  // opt-in max minus static smem / slack
  const size_t fixed = (size_t)2 * L.a_bytes + (size_t)L.p_bytes;
  if (fixed >= budget) return L;
  for (int nst = kT2MaxStages; nst >= 2; --nst) {
    const size_t per = (budget - fixed) / nst;
    if (per <= kT2IpBytes + 64) continue;
    int64_t cap = (int64_t)((per - kT2IpBytes - 32) / (size_t)(ix_bytes + 4));
    cap &= ~(int64_t)15;
    if (cap > 8192) cap = 8192;
    if (cap < 2048) continue;
    L.cap = (int)cap;
    L.nst = nst;
    L.idx_off = kT2IpBytes;
    L.val_off = kT2IpBytes + (uint32_t)(cap * ix_bytes + 16);
    L.stage_bytes = L.val_off + (uint32_t)(cap * 4 + 16);
    L.smem = fixed + (size_t)nst * L.stage_bytes;
    return L;
  }
  return L;
}

}  // namespace
}  // namespace skt
