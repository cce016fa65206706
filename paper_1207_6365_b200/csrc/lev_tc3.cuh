// lev_tc3.cuh -- K5 default kernel for fp32 CSR: the register-staged tile
// pipeline of lev_tc.cuh with the scaled 2xFP16 operands of lev_tc2.cuh.
//
// Numerics (as lev_tc2.cuh): row i of a tile is scaled by 2^-e_i (frexp
// exponent of its largest |a|) and the probe by one 2^-f; each scaled value is
// split into fp16 hi + lo (22 significant bits) stored INTERLEAVED along K
// (element 2c = hi, 2c+1 = lo: one 32-bit store per nonzero, at the tf32
// layout's word position of column c), and the B operand holds rows
// [P_hi, P_hi] / [P_lo, 0] interleaved the same way, so ONE
// tcgen05.mma.kind::f16 with N = 2k per 16-element K step gives A_hi P_hi +
// A_lo P_hi in TMEM columns 0..k-1 and A_hi P_lo in k..2k-1 (A_lo P_lo,
// ~2^-22 relative, dropped).  The epilogue adds the halves, squares and sums
// in fp64 and rescales by the exact 2^(2(e_i + f)).
//
// Against the 3xTF32 kernel (lev_tc.cuh): 8 instead of 16 MMAs per 128 x 64
// tile, one store instead of two per nonzero, and half the A tile (32 KB), so
// four CTAs share an SM instead of two -- their MMA chains, densify phases and
// epilogues overlap.  Tile flow per CTA: densify from registers (nonzeros of
// the tile prefetched during the previous tile, first long row's tail too),
// order check (duplicates / unsorted rows -> serial rebuild), one thread
// issues the MMA chain, the next tile's loads go in flight, epilogue, re-zero.
#pragma once

#include "lev_tc2.cuh"

namespace skt {
namespace {

__host__ __device__ inline bool tc3_ok(int k) { return k % 32 == 0 && 2 * k <= 256; }
__host__ __device__ inline uint32_t tc3_cols(int k) {
  const int c = 2 * k;
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : 256;
}
inline size_t lev_tc3_smem(int dk, int k) {  // A: 128 x dk words; B: 2k x 2dk fp16
  return (size_t)kTcRows * dk * 4 + (size_t)(2 * k) * (2 * dk) * 2;
}

#ifndef SKT_TC3_BLOCKCLEAR
#define SKT_TC3_BLOCKCLEAR 1
#endif
#ifndef SKT_TC3_L2PF
#define SKT_TC3_L2PF 1
#endif

template <typename IP, typename IX, typename TS>
__global__ void __launch_bounds__(kTcThreads, 4) lev_tc3_kernel(int64_t n, int d, int dk,
                                                             const IP *__restrict__ aip,
                                                             const IX *__restrict__ aix,
                                                             const float *__restrict__ av,
                                                             const double *__restrict__ probe, int k,
                                                             TS *__restrict__ scores) {
  // dk = d rounded up to a multiple of 8 (column pairs; K of the chain = 2 dk)
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  __shared__ int rexp[kTcRows];
  __shared__ float pmax_w[kTcThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t a_bytes = (uint32_t)kTcRows * dk * 4;
  uint32_t *aw = (uint32_t *)smem;  // word (r, c) at tc_off(r, c, 128) / 4
  unsigned char *p_op = smem + a_bytes;
  const uint32_t p_bytes = (uint32_t)(2 * k) * (2 * dk) * 2;

  // ---- one-time setup: zero A and B, scaled probe operand, TMEM, barrier
  for (uint32_t i = tid; i < (a_bytes + p_bytes) / 16; i += kTcThreads) ((uint4 *)smem)[i] = make_uint4(0, 0, 0, 0);
  float pm = 0.f;
  for (int i = tid; i < d * k; i += kTcThreads) pm = fmaxf(pm, (float)fabs(probe[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, o));
  if (lane == 0) pmax_w[warp] = pm;
  __syncthreads();
  pm = 0.f;
  for (int w = 0; w < kTcThreads / 32; ++w) pm = fmaxf(pm, pmax_w[w]);
  const int pe = t2_exp(pm);
  const double pscale = __longlong_as_double((long long)(1023 - pe) << 52);
  for (int i = tid; i < k * d; i += kTcThreads) {
    const int col = i / d, c = i % d;  // B row col <- P[c][col]
    const float x = (float)(probe[(int64_t)c * k + col] * pscale);
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    *(__half *)(p_op + t2_p_off(col, 2 * c, 2 * k)) = h;
    *(__half *)(p_op + t2_p_off(col, 2 * c + 1, 2 * k)) = h;
    *(__half *)(p_op + t2_p_off(k + col, 2 * c, 2 * k)) = l;
  }
  const uint32_t ncols = tc3_cols(k);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc_smem_u32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(tc_smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = t2_idesc(2 * k);
  uint32_t phase = 0;

  const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
#ifndef SKT_TC3_G
#define SKT_TC3_G 8
#endif
  // G lanes per row, S = 32/G rows per warp instruction, NI = G row iterations
  // per warp, JP = 16/G staged nonzeros per lane and row: the first NR = 16
  // nonzeros of every row are staged (E = 16 registers per lane).  G = 4 (8
  // rows of distinct row mod 8 per store: no bank conflicts) measured 5%
  // slower than G = 8 on config 4 (less coalesced loads, more shuffles).
  constexpr int G = SKT_TC3_G, S = 32 / G, NI = G, JP = 16 / G, E = 16, NR = 16;
  const int g = lane / G, gl = lane % G;
  auto load_desc = [&](int64_t tile, int64_t &rs, int &len) {
    const int64_t row = tile * kTcRows + warp * 32 + lane;
    rs = 0;
    len = 0;
    if (tile < ntiles && row < n) {
      rs = (int64_t)aip[row];
      len = (int)((int64_t)aip[row + 1] - rs);
    }
  };
  // raw indptr pair of a tile two ahead: converted one iteration later, so
  // the loads stay in flight instead of stalling the warp right after issue
  auto load_desc_raw = [&](int64_t tile, IP &b, IP &e) {
    const int64_t row = tile * kTcRows + warp * 32 + lane;
    b = e = (IP)0;
    if (tile < ntiles && row < n) {
      b = __ldg(aip + row);
      e = __ldg(aip + row + 1);
    }
  };
  // nonzeros of a tile into registers: iteration i covers rows 4i + g, lanes
  // gl and gl + 8 of each row; the tail (nonzeros 16..79) of the warp's first
  // long row goes in flight too
  int pc[E];
  float pv[E];
  int lr = -1, lc[2];
  float lv[2];
  auto load_data = [&](int64_t rs, int len) {
    {
      const uint32_t lm = __ballot_sync(0xffffffffu, len > NR);
      lr = lm ? __ffs(lm) - 1 : -1;
      lc[0] = lc[1] = -1;
      if (lm) {
        const int64_t rs_r = __shfl_sync(0xffffffffu, rs, lr);
        const int len_r = __shfl_sync(0xffffffffu, len, lr);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = NR + lane + 32 * j;
          if (q < len_r) {
            lc[j] = (int)__ldg(aix + rs_r + q);
            lv[j] = __ldg(av + rs_r + q);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int r = i * S + g;
      const int64_t rs_r = __shfl_sync(0xffffffffu, rs, r);
      const int len_r = __shfl_sync(0xffffffffu, len, r);
#pragma unroll
      for (int j = 0; j < JP; ++j) {
        const int q = gl + G * j;
        pc[i * JP + j] = -1;
        if (q < len_r) {
          pc[i * JP + j] = (int)__ldg(aix + rs_r + q);
          pv[i * JP + j] = __ldg(av + rs_r + q);
        }
      }
    }
  };

  int64_t tile = blockIdx.x;
  int64_t rs_c, rs_n;
  int len_c, len_n;
  load_desc(tile, rs_c, len_c);
  if (tile < ntiles) load_data(rs_c, len_c);
  load_desc(tile + gridDim.x, rs_n, len_n);
  IP rb_2, re_2;
  load_desc_raw(tile + 2 * (int64_t)gridDim.x, rb_2, re_2);
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTcRows;
    const uint32_t longm = __ballot_sync(0xffffffffu, len_c > NR);
    // ---- per-row max |a| (registers, then the long rows' tails) -> scale
    float m[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      m[i] = 0.f;
#pragma unroll
      for (int j = 0; j < JP; ++j)
        if (pc[i * JP + j] >= 0) m[i] = fmaxf(m[i], fabsf(pv[i * JP + j]));
    }
    if (longm) {
      for (uint32_t mm = longm; mm; mm &= mm - 1) {  // max over each long row's tail (whole warp)
        const int r = __ffs(mm) - 1;
        const int64_t rs_r = __shfl_sync(0xffffffffu, rs_c, r);
        const int len_r = __shfl_sync(0xffffffffu, len_c, r);
        float t = 0.f;
        if (r == lr) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (lc[j] >= 0) t = fmaxf(t, fabsf(lv[j]));
        }
        for (int q = (r == lr ? NR + 64 : NR) + lane; q < len_r; q += 32) t = fmaxf(t, fabsf(__ldg(av + rs_r + q)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, o));
        // fold into the row's group: row r = 4i + g
#pragma unroll
        for (int i = 0; i < NI; ++i)
          if (i * S + g == r) m[i] = fmaxf(m[i], t);
      }
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], o, G));
      if (gl == 0) rexp[warp * 32 + i * S + g] = t2_exp(m[i]);
    }
    __syncwarp();
    // ---- column order check (duplicates / unsorted rows -> rebuild below)
    bool dirty = false;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
#pragma unroll
      for (int j = 0; j < JP; ++j) {  // predecessor of entry gl + G j: lane gl - 1 (same j) or lane G - 1 (j - 1)
        const int c = pc[i * JP + j];
        const int ps = __shfl_up_sync(0xffffffffu, c, 1, G);
        const int pw = j > 0 ? __shfl_sync(0xffffffffu, pc[i * JP + j - 1], G - 1, G) : -1;
        if (c >= 0 && (gl > 0 || j > 0)) dirty |= c <= (gl > 0 ? ps : pw);
      }
    }
    // ---- densify: one packed (hi, lo) word per nonzero
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int r = warp * 32 + i * S + g;
      const float sc = __int_as_float((127 - rexp[r]) << 23);
#pragma unroll
      for (int j = 0; j < JP; ++j)
        if (pc[i * JP + j] >= 0) aw[tc_off(r, pc[i * JP + j], kTcRows) >> 2] = t2_pack(pv[i * JP + j] * sc);
    }
    if (lr >= 0) {
      const int64_t rs_r = __shfl_sync(0xffffffffu, rs_c, lr);
      const float sc = __int_as_float((127 - rexp[warp * 32 + lr]) << 23);
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (lc[j] >= 0) {
          dirty |= lc[j] <= (int)__ldg(aix + rs_r + NR + lane + 32 * j - 1);
          aw[tc_off(warp * 32 + lr, lc[j], kTcRows) >> 2] = t2_pack(lv[j] * sc);
        }
    }
    for (uint32_t mm = longm; mm; mm &= mm - 1) {  // rest of the long rows (whole warp)
      const int r = __ffs(mm) - 1;
      const int64_t rs_r = __shfl_sync(0xffffffffu, rs_c, r);
      const int len_r = __shfl_sync(0xffffffffu, len_c, r);
      const float sc = __int_as_float((127 - rexp[warp * 32 + r]) << 23);
      for (int q = (r == lr ? NR + 64 : NR) + lane; q < len_r; q += 32) {
        const int c = (int)__ldg(aix + rs_r + q);
        dirty |= c <= (int)__ldg(aix + rs_r + q - 1);
        aw[tc_off(warp * 32 + r, c, kTcRows) >> 2] = t2_pack(__ldg(av + rs_r + q) * sc);
      }
    }
    if (__syncthreads_or(dirty)) {
      // rebuild: clear, then one thread per row in entry order, duplicates
      // summed before the split; scale from sum |a| (bounds any partial sum)
      for (uint32_t i = tid; i < a_bytes / 16; i += kTcThreads) ((uint4 *)smem)[i] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      const int64_t r = row0 + tid;
      if (r < n) {
        const int64_t rb = (int64_t)aip[r], re = (int64_t)aip[r + 1];
        float sum = 0.f;
        for (int64_t q = rb; q < re; ++q) sum += fabsf(av[q]);
        const int ex = t2_exp(sum);
        const float sc = __int_as_float((127 - ex) << 23);
        rexp[tid] = ex;
        for (int64_t q = rb; q < re; ++q) {
          uint32_t *w = aw + (tc_off(tid, (int)aix[q], kTcRows) >> 2);
          *w = t2_pack(av[q] * sc + t2_unpack(*w));
        }
      }
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- MMA chain: K = 2 dk fp16 in steps of 16, one N = 2k MMA per step
    if (tid == 0) {
      const uint32_t lbo_a = kTcRows * 16, lbo_p = (uint32_t)(2 * k) * 16;
      const uint32_t ab = tc_smem_u32(aw), pb = tc_smem_u32(p_op);
      for (int ks = 0; ks < dk / 8; ++ks)
        t2_mma(tmem, tc_desc(ab + (uint32_t)ks * 2 * lbo_a, lbo_a, 128),
               tc_desc(pb + (uint32_t)ks * 2 * lbo_p, lbo_p, 128), idesc, ks > 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       tc_smem_u32(&mbar))
                   : "memory");
    }
    // ---- overlap: the next tile's nonzeros and descriptors go in flight now
#if !SKT_TC3_BLOCKCLEAR
    int cur_c[E];
#pragma unroll
    for (int i = 0; i < E; ++i) cur_c[i] = pc[i];
    const uint32_t longz = longm;
#endif
    if (tile + gridDim.x < ntiles) load_data(rs_n, len_n);
    rs_c = rs_n;
    len_c = len_n;
    rs_n = (int64_t)rb_2;
    len_n = (int)((int64_t)re_2 - (int64_t)rb_2);
#if SKT_TC3_L2PF
    // tile + 2's rows into L2 now: its register loads (issued one iteration
    // from here, consumed right after this tile's epilogue) then hit L2
    if (len_n > 0) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(aix + rs_n));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(av + rs_n));
    }
    if (len_n > 24) {  // long rows: their next 128 bytes too
      asm volatile("prefetch.global.L2 [%0];" ::"l"(aix + rs_n + 32));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(av + rs_n + 32));
    }
#endif
    load_desc_raw(tile + 3 * (int64_t)gridDim.x, rb_2, re_2);
    // ---- wait for the accumulator
    asm volatile(
        "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
            tc_smem_u32(&mbar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- epilogue: row = TMEM lane = 32 warp + lane; x_c = D[c] + D[k + c]
    double sc0 = 0.0, sc1 = 0.0;
    const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < k; c0 += 32) {
      uint32_t v[32], w2[32];
      TC_TMEM_LD32(tbase + (uint32_t)c0, v);
      TC_TMEM_LD32(tbase + (uint32_t)(k + c0), w2);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const double x0 = (double)(__uint_as_float(v[j]) + __uint_as_float(w2[j]));
        const double x1 = (double)(__uint_as_float(v[j + 1]) + __uint_as_float(w2[j + 1]));
        sc0 = fma(x0, x0, sc0);
        sc1 = fma(x1, x1, sc1);
      }
    }
    const int myr = warp * 32 + lane;
    const int64_t my_row = row0 + myr;
    const double unscale = __longlong_as_double((long long)(1023 + 2 * (rexp[myr] + pe)) << 52);
    if (my_row < n) scores[my_row] = (TS)((sc0 + sc1) * unscale);
#if SKT_TC3_BLOCKCLEAR
    // ---- clear this warp's 32 rows of the A tile: in every 16-byte K column
    // they are one contiguous 512-byte block (16 r + 2048 (c / 4)), one
    // 16-byte store per lane -- fewer instructions than re-zeroing the
    // scattered entries, and no registers held across the MMA wait
    {
      unsigned char *blk = (unsigned char *)aw + warp * 512 + lane * 16;
      for (int kc = 0; kc < dk / 4; ++kc) *(uint4 *)(blk + kc * (kTcRows * 16)) = make_uint4(0, 0, 0, 0);
    }
#else
    // ---- re-zero what this tile wrote
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (cur_c[i] >= 0) aw[tc_off(warp * 32 + (i / JP) * S + g, cur_c[i], kTcRows) >> 2] = 0u;
    for (uint32_t mm = longz; mm; mm &= mm - 1) {
      const int r = __ffs(mm) - 1;
      for (int c = lane; c < dk; c += 32) aw[tc_off(warp * 32 + r, c, kTcRows) >> 2] = 0u;
    }
#endif
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM drained, tile clean, rexp read before the next densify
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

}  // namespace
}  // namespace skt
