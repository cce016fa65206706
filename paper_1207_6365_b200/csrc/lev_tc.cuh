// lev_tc.cuh -- K5 on the 5th-generation tensor cores: fused leverage-score
// contraction scores_i = || A_i . P ||^2 (reference leverage.py:90-91) for CSR
// A with fp32 values, d <= 256, probe width k a multiple of 8 up to 256.
//
// Per CTA tile of 128 rows:
//   1. densify: the rows' nonzeros are scattered into K-major fp32 tiles in
//      shared memory in the UMMA canonical no-swizzle layout -- A_hi = tf32(a)
//      and A_lo = tf32(a - A_hi) (3xTF32 split); the probe P^T (hi/lo) is
//      staged once per CTA in the same layout;
//   2. one thread issues tcgen05.mma.kind::tf32 (M=128, N=k, K=8 per
//      instruction): D = A_hi P_hi + A_hi P_lo + A_lo P_hi accumulated in TMEM
//      (128 lanes x k fp32 columns), completion via tcgen05.commit -> mbarrier;
//   3. epilogue: warp w reads TMEM lanes 32w..32w+31 (tcgen05.ld 32x32b, one
//      row per thread) and reduces the k products to the row's squared norm
//      in fp64; the written tile entries are re-zeroed.
// A is read once; the n x k product never leaves the SM.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

constexpr int kTcRows = 128;  // UMMA M
constexpr int kTcThreads = 128;

__device__ __forceinline__ uint32_t tc_smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major, no-swizzle canonical layout of an (R x K) fp32 operand tile:
// core matrix = 8 rows x 16 B (4 elements); element (r, c) at byte
//   (c / 4) * LBO + (r / 8) * 128 + (r % 8) * 16 + (c % 4) * 4,  LBO = R * 16.
__device__ __forceinline__ uint32_t tc_off(int r, int c, int R) {
  return (uint32_t)((c >> 2) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (c & 3) * 4);
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = n, M = 128
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// A tile offsets / descriptors (K-major, no swizzle).  The 128-byte-swizzled
// layout was measured: faster MMAs in isolation (tools/lev_prof.cu), but 4%
// slower in this kernel (the scatter's extra address math), so not used.
__device__ __forceinline__ uint32_t tc_a_off(int r, int c) { return tc_off(r, c, kTcRows); }
__device__ __forceinline__ uint64_t tc_a_desc(uint32_t base, int ks) {  // K step ks (8 elements)
  return tc_desc(base + (uint32_t)ks * 2 * (kTcRows * 16), kTcRows * 16, 128);
}
// Merged probe operand (k % 32 == 0, 2k <= 256): P staged as one 2k-row
// operand [P_hi; P_lo], A_hi.[P_hi | P_lo] is one N = 2k MMA and A_lo.P_hi
// accumulates into columns 0..k-1 -- 16 instead of 24 MMAs per 128 x 64 tile
// (-6% on config 4); the epilogue adds columns c and k + c.
__host__ __device__ inline bool tc_merged(int k) { return k % 32 == 0 && 2 * k <= 256; }

// 32 TMEM columns of this warp's 32 lanes
#define TC_TMEM_LD32(taddr, v)                                                                            \
  asm volatile(                                                                                           \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"   \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                         \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),  \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),         \
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),       \
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),       \
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                            \
      : "r"(taddr))

// TMEM columns a CTA allocates for a k-wide accumulator
__host__ __device__ inline uint32_t lev_tc_cols(int k) {
  const int c = tc_merged(k) ? 2 * k : k;
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : 256;
}

template <typename IP, typename IX, typename TS, bool kMerged>
__global__ void __launch_bounds__(kTcThreads) lev_tc_kernel(int64_t n, int d, int dk,
                                                            const IP *__restrict__ aip,
                                                            const IX *__restrict__ aix,
                                                            const float *__restrict__ av,
                                                            const double *__restrict__ probe,
                                                            int k, TS *__restrict__ scores) {
  // dk = d rounded up to a multiple of 8 (K of the MMA chain)
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t a_bytes = (uint32_t)kTcRows * dk * 4;
  const uint32_t p_bytes = (uint32_t)k * dk * 4;
  float *a_hi = (float *)smem;
  float *a_lo = (float *)(smem + a_bytes);
  float *p_hi = (float *)(smem + 2 * a_bytes);
  float *p_lo = (float *)(smem + 2 * a_bytes + p_bytes);
  constexpr bool merged = kMerged;  // host selects tc_merged(k)

  // ---- one-time setup: zero A tiles, stage P^T (K-major: row = probe column)
  for (uint32_t i = tid; i < 2 * a_bytes / 16; i += kTcThreads) ((uint4 *)smem)[i] = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < k * dk; i += kTcThreads) {
    const int col = i / dk, kk = i % dk;  // P^T[col][kk] = P[kk][col]
    const double p = kk < d ? probe[(int64_t)kk * k + col] : 0.0;
    const float hi = tf32_hi((float)p);
    const float lo = tf32_hi((float)(p - (double)hi));
    if (merged) {  // one 2k-row operand at p_hi
      *(float *)((unsigned char *)p_hi + tc_off(col, kk, 2 * k)) = hi;
      *(float *)((unsigned char *)p_hi + tc_off(k + col, kk, 2 * k)) = lo;
    } else {
      const uint32_t off = tc_off(col, kk, k);
      *(float *)((unsigned char *)p_hi + off) = hi;
      *(float *)((unsigned char *)p_lo + off) = lo;
    }
  }
  if (warp == 0) {
    const uint32_t ncols = lev_tc_cols(k);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc_smem_u32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(tc_smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = tc_idesc(k);
  uint32_t phase = 0;

  const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
  constexpr int G = 8, S = 32 / G, E = 16;  // 8 lanes per row, <= 16 staged nonzeros per lane
  const int g = lane / G, gl = lane % G;
  // row descriptor of this lane's row (lane-per-row) for a tile
  auto load_desc = [&](int64_t tile, int64_t &rs, int &len) {
    const int64_t row = tile * kTcRows + warp * 32 + lane;
    rs = 0;
    len = 0;
    if (tile < ntiles && row < n) {
      rs = (int64_t)aip[row];
      len = (int)((int64_t)aip[row + 1] - rs);
    }
  };
  // nonzeros of a tile into registers: iteration i covers rows 4i + g, lanes
  // gl and gl + 8 of each row (rows of <= 16 nonzeros complete here)
  int pc[E];
  float pv[E];
  // the tail (nonzeros 16..79) of the warp's first long row also goes in
  // flight with the tile, so a dense row does not put a dependent load round
  // trip inside the densify phase (the whole CTA would wait on it)
  int lr = -1, lc[2];
  float lv[2];
  auto load_data = [&](int64_t rs, int len) {
    {
      const uint32_t lm = __ballot_sync(0xffffffffu, len > 2 * G);
      lr = lm ? __ffs(lm) - 1 : -1;
      lc[0] = lc[1] = -1;
      if (lm) {
        const int64_t rs_r = __shfl_sync(0xffffffffu, rs, lr);
        const int len_r = __shfl_sync(0xffffffffu, len, lr);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = 2 * G + lane + 32 * j;
          if (q < len_r) {
            lc[j] = (int)__ldg(aix + rs_r + q);
            lv[j] = __ldg(av + rs_r + q);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      const int r = i * S + g;
      const int64_t rs_r = __shfl_sync(0xffffffffu, rs, r);
      const int len_r = __shfl_sync(0xffffffffu, len, r);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = gl + G * j;
        pc[2 * i + j] = -1;
        if (q < len_r) {
          pc[2 * i + j] = (int)__ldg(aix + rs_r + q);
          pv[2 * i + j] = __ldg(av + rs_r + q);
        }
      }
    }
  };
  auto put = [&](int trow, int c, float v) {
    const float hi = tf32_hi(v);
    const float lo = tf32_hi(v - hi);
    const uint32_t off = tc_a_off(trow, c);
    *(float *)((unsigned char *)a_hi + off) = hi;
    *(float *)((unsigned char *)a_lo + off) = lo;
  };

  int64_t tile = blockIdx.x;
  int64_t rs_c, rs_n;
  int len_c, len_n;
  load_desc(tile, rs_c, len_c);
  if (tile < ntiles) load_data(rs_c, len_c);
  load_desc(tile + gridDim.x, rs_n, len_n);
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTcRows;
    // ---- densify the staged nonzeros (3xTF32 split)
    // column order check: a non-increasing pair (duplicate / unsorted row)
    // marks the tile dirty -> rebuilt below one thread per row
    bool dirty = false;
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      const int p0 = __shfl_up_sync(0xffffffffu, pc[2 * i], 1, G);      // entry gl - 1
      const int p7 = __shfl_sync(0xffffffffu, pc[2 * i], G - 1, G);     // entry 7
      const int p1 = __shfl_up_sync(0xffffffffu, pc[2 * i + 1], 1, G);  // entry gl + 7
      if (gl > 0 && pc[2 * i] >= 0) dirty |= pc[2 * i] <= p0;
      if (pc[2 * i + 1] >= 0) dirty |= pc[2 * i + 1] <= (gl > 0 ? p1 : p7);
    }
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (pc[i] >= 0) put(warp * 32 + (i / 2) * S + g, pc[i], pv[i]);
    if (lr >= 0) {
      const int64_t rs_r = __shfl_sync(0xffffffffu, rs_c, lr);
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (lc[j] >= 0) {
          dirty |= lc[j] <= (int)__ldg(aix + rs_r + 2 * G + lane + 32 * j - 1);
          put(warp * 32 + lr, lc[j], lv[j]);
        }
    }
    const uint32_t longm = __ballot_sync(0xffffffffu, len_c > 2 * G);
    for (uint32_t m = longm; m; m &= m - 1) {  // rest of the rows with > 16 nonzeros (whole warp)
      const int r = __ffs(m) - 1;
      const int64_t rs_r = __shfl_sync(0xffffffffu, rs_c, r);
      const int len_r = __shfl_sync(0xffffffffu, len_c, r);
      for (int q = (r == lr ? 2 * G + 64 : 2 * G) + lane; q < len_r; q += 32) {
        const int c = (int)__ldg(aix + rs_r + q);
        dirty |= c <= (int)__ldg(aix + rs_r + q - 1);
        put(warp * 32 + r, c, __ldg(av + rs_r + q));
      }
    }
    if (__syncthreads_or(dirty)) {
      // rebuild: clear, then one thread per row in entry order, summing
      // duplicates before the split (scipy's a @ probe semantics)
      for (uint32_t i = tid; i < 2 * a_bytes / 16; i += kTcThreads) ((uint4 *)smem)[i] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      const int64_t r = row0 + tid;
      if (r < n) {
        const int64_t rb = (int64_t)aip[r], re = (int64_t)aip[r + 1];
        for (int64_t q = rb; q < re; ++q) {
          const uint32_t off = tc_a_off(tid, (int)aix[q]);
          float *h = (float *)((unsigned char *)a_hi + off);
          float *l = (float *)((unsigned char *)a_lo + off);
          const float v = av[q] + (*h + *l);
          const float hv = tf32_hi(v);
          *h = hv;
          *l = tf32_hi(v - hv);
        }
      }
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- MMA chain: 3xTF32 over K = dk in steps of 8 (one thread issues)
    if (tid == 0) {
      const uint32_t lbo_a = kTcRows * 16, lbo_p = (uint32_t)k * 16;
      const uint32_t ah = tc_smem_u32(a_hi), al = tc_smem_u32(a_lo);
      const uint32_t ph = tc_smem_u32(p_hi), pl = tc_smem_u32(p_lo);
      for (int ks = 0; ks < dk / 8; ++ks) {
        const uint32_t oa = (uint32_t)ks * 2 * lbo_a, op = (uint32_t)ks * 2 * lbo_p;
        if (merged) {
          const uint32_t lbo_p2 = 2 * lbo_p, op2 = (uint32_t)ks * 2 * lbo_p2;
          tc_mma(tmem, tc_a_desc(ah, ks), tc_desc(ph + op2, lbo_p2, 128), tc_idesc(2 * k), ks > 0);
          tc_mma(tmem, tc_a_desc(al, ks), tc_desc(ph + op2, lbo_p2, 128), idesc, 1);
        } else {
          tc_mma(tmem, tc_a_desc(ah, ks), tc_desc(ph + op, lbo_p, 128), idesc, ks > 0);
          tc_mma(tmem, tc_a_desc(ah, ks), tc_desc(pl + op, lbo_p, 128), idesc, 1);
          tc_mma(tmem, tc_a_desc(al, ks), tc_desc(ph + op, lbo_p, 128), idesc, 1);
        }
        (void)oa;
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       tc_smem_u32(&mbar))
                   : "memory");
    }
    // ---- overlap: the next tile's nonzeros and descriptors go in flight now
    int cur_c[E];
#pragma unroll
    for (int i = 0; i < E; ++i) cur_c[i] = pc[i];
    const int len_cur = len_c;
    const int64_t rs_cur = rs_c;
    if (tile + gridDim.x < ntiles) load_data(rs_n, len_n);
    rs_c = rs_n;
    len_c = len_n;
    load_desc(tile + 2 * (int64_t)gridDim.x, rs_n, len_n);
    // ---- wait for the accumulator
    asm volatile(
        "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
            tc_smem_u32(&mbar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- epilogue: row = TMEM lane = 32 * warp + lane; k columns, 32 at a time
    double sc = 0.0;
    for (int c0 = 0; c0 < k; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      uint32_t w2[kMerged ? 32 : 1];
      TC_TMEM_LD32(taddr, v);
      if constexpr (kMerged) TC_TMEM_LD32(taddr + (uint32_t)k, w2);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int cn = k - c0 < 32 ? k - c0 : 32;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < cn) {
          double x;
          if constexpr (kMerged)
            x = (double)(__uint_as_float(v[j]) + __uint_as_float(w2[j]));
          else
            x = (double)__uint_as_float(v[j]);
          sc = fma(x, x, sc);
        }
      }
    }
    const int64_t my_row = row0 + warp * 32 + lane;
    if (my_row < n) scores[my_row] = (TS)sc;
    // ---- re-zero what this tile wrote
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (cur_c[i] >= 0) {
        const uint32_t off = tc_a_off(warp * 32 + (i / 2) * S + g, cur_c[i]);
        *(float *)((unsigned char *)a_hi + off) = 0.f;
        *(float *)((unsigned char *)a_lo + off) = 0.f;
      }
    }
    const uint32_t longz = __ballot_sync(0xffffffffu, len_cur > 2 * G);
    (void)rs_cur;
    for (uint32_t m = longz; m; m &= m - 1) {
      const int r = __ffs(m) - 1;
      for (int c = lane; c < dk; c += 32) {
        const uint32_t off = tc_a_off(warp * 32 + r, c);
        *(float *)((unsigned char *)a_hi + off) = 0.f;
        *(float *)((unsigned char *)a_lo + off) = 0.f;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM drained and tile clean before the next MMA
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t ncols = lev_tc_cols(k);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
  }
}

inline size_t lev_tc_smem(int dk, int k) { return (size_t)2 * kTcRows * dk * 4 + (size_t)2 * k * dk * 4; }

}  // namespace
}  // namespace skt
