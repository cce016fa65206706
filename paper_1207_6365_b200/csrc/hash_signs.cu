// hash_signs.cu -- K1: bit-exact bucket hash h and sign s of SparseEmbedding
// (reference sketch.py:147-148) generated on the GPU.
//
// numpy semantics restated (numpy 2.3.5, see oracle/skt_oracle.c):
//   * PCG64 XSL-RR: step the 128-bit LCG, output rotr64(hi ^ lo, state >> 122)
//   * next_uint32: 64-bit output k feeds 32-bit draws 2k (low half), 2k+1 (high)
//   * integers(0, t): Lemire  m = u * t;  accept iff (uint32)m >= (2^32 - t) % t;
//     value m >> 32.  t == 1 consumes nothing; t == 2^32 returns u.
//   * choice([-1, 1]) == integers(0, 2): +1 iff the top bit of the draw is set.
//
// Layout: a warp owns 32 * kJ consecutive 64-bit outputs; lane l computes
// outputs o0 + l + 32 j, so each warp-iteration writes 64 consecutive h values
// (coalesced).  Each lane jumps ahead once (O(log o) 128-bit mults) and then
// advances by 32 outputs per iteration with one precomputed affine step.
// When the rejection threshold is non-zero (t not a power of two) the draws
// are stream-compacted: pass 1 counts accepted draws per warp, a device scan
// gives each warp its first accepted-draw rank, pass 2 regenerates and writes.
#include "common.cuh"
#include "scan.cuh"

namespace skt {
namespace {

constexpr int kJ = 64;                       // outputs per lane per warp
constexpr int64_t kOutPerWarp = 32LL * kJ;  // 2048 outputs = 4096 draws
constexpr int kThreads = 256;

struct GenParams {
  uint64_t s_hi, s_lo, inc_hi, inc_lo;   // seeded state, increment
  uint64_t m32_hi, m32_lo, p32_hi, p32_lo;  // affine step of 32 outputs
};

__device__ __forceinline__ u128 lane_state(const GenParams &g, uint64_t out_index) {
  const u128 inc = mk128(g.inc_hi, g.inc_lo);
  const Affine128 a = lcg_power(out_index, inc);
  return a.mult * mk128(g.s_hi, g.s_lo) + a.plus;
}

__device__ __forceinline__ uint32_t bounded(uint32_t u, uint64_t t) {
  return t == (1ull << 32) ? u : (uint32_t)(((uint64_t)u * t) >> 32);
}

// Direct mode: no rejection possible, draw index == row index.
// kind 0 = bucket (writes h), kind 1 = sign (writes s).
template <int kKind>
__global__ void __launch_bounds__(kThreads) gen_direct_kernel(GenParams g, int64_t row_begin,
                                                              int64_t row_end, uint64_t t,
                                                              uint32_t *__restrict__ h,
                                                              int8_t *__restrict__ s) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t o_first = row_begin >> 1, o_last = (row_end - 1) >> 1;
  const int64_t o_w = o_first + warp * kOutPerWarp;
  if (o_w > o_last) return;
  const u128 inc = mk128(g.inc_hi, g.inc_lo), mult = pcg_mult();
  const u128 m32 = mk128(g.m32_hi, g.m32_lo), p32 = mk128(g.p32_hi, g.p32_lo);
  u128 st = lane_state(g, (uint64_t)(o_w + lane));
  for (int j = 0; j < kJ; ++j) {
    const int64_t o = o_w + lane + 32LL * j;
    if (o_w + 32LL * j > o_last) break;  // warp-uniform
    const uint64_t v = pcg_output(st * mult + inc);
    st = m32 * st + p32;
    const uint32_t u[2] = {(uint32_t)v, (uint32_t)(v >> 32)};
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t r = 2 * o + half;
      if (r >= row_begin && r < row_end) {
        if (kKind == 0)
          h[r - row_begin] = bounded(u[half], t);
        else
          s[r - row_begin] = (u[half] >> 31) ? (int8_t)1 : (int8_t)-1;
      }
    }
  }
}

// Rejection mode, pass 1: accepted draws per warp over outputs [0, n_out).
__global__ void __launch_bounds__(kThreads) count_accept_kernel(GenParams g, int64_t n_out,
                                                                uint64_t t, uint32_t thr,
                                                                uint32_t *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t o_w = warp * kOutPerWarp;
  if (o_w >= n_out) return;
  const u128 inc = mk128(g.inc_hi, g.inc_lo), mult = pcg_mult();
  const u128 m32 = mk128(g.m32_hi, g.m32_lo), p32 = mk128(g.p32_hi, g.p32_lo);
  u128 st = lane_state(g, (uint64_t)(o_w + lane));
  uint32_t c = 0;
  for (int j = 0; j < kJ; ++j) {
    const int64_t o = o_w + lane + 32LL * j;
    if (o >= n_out) break;
    const uint64_t v = pcg_output(st * mult + inc);
    st = m32 * st + p32;
    c += ((uint32_t)((uint64_t)(uint32_t)v * t) >= thr);
    c += ((uint32_t)((v >> 32) * t) >= thr);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) counts[warp] = c;
}

// Rejection mode, pass 2: regenerate; accepted draw of global rank r -> row r.
__global__ void __launch_bounds__(kThreads) write_accept_kernel(GenParams g, int64_t n_out,
                                                                uint64_t t, uint32_t thr,
                                                                const uint32_t *__restrict__ offs,
                                                                int64_t row_begin, int64_t row_end,
                                                                uint32_t *__restrict__ h) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t o_w = warp * kOutPerWarp;
  if (o_w >= n_out) return;
  int64_t running = offs[warp];
  if (running >= row_end) return;
  const u128 inc = mk128(g.inc_hi, g.inc_lo), mult = pcg_mult();
  const u128 m32 = mk128(g.m32_hi, g.m32_lo), p32 = mk128(g.p32_hi, g.p32_lo);
  u128 st = lane_state(g, (uint64_t)(o_w + lane));
  for (int j = 0; j < kJ; ++j) {
    if (o_w + 32LL * j >= n_out || running >= row_end) break;  // warp-uniform
    const int64_t o = o_w + lane + 32LL * j;
    const bool live = o < n_out;
    const uint64_t v = pcg_output(st * mult + inc);
    st = m32 * st + p32;
    const uint64_t m0 = (uint64_t)(uint32_t)v * t, m1 = (v >> 32) * t;
    const uint32_t a0 = live && (uint32_t)m0 >= thr, a1 = live && (uint32_t)m1 >= thr;
    const uint32_t c = a0 + a1;
    const uint32_t incl = warp_incl_scan(c);
    const int64_t r0 = running + incl - c;  // rank of this lane's first accepted draw
    if (a0 && r0 >= row_begin && r0 < row_end) h[r0 - row_begin] = (uint32_t)(m0 >> 32);
    const int64_t r1 = r0 + a0;
    if (a1 && r1 >= row_begin && r1 < row_end) h[r1 - row_begin] = (uint32_t)(m1 >> 32);
    running += __shfl_sync(0xffffffffu, incl, 31);
  }
}

GenParams make_params(const skt_pcg64 &p) {
  GenParams g;
  g.s_hi = p.state_hi;
  g.s_lo = p.state_lo;
  g.inc_hi = p.inc_hi;
  g.inc_lo = p.inc_lo;
  const Affine128 a = lcg_power(32, mk128(p.inc_hi, p.inc_lo));
  g.m32_hi = (uint64_t)(a.mult >> 64);
  g.m32_lo = (uint64_t)a.mult;
  g.p32_hi = (uint64_t)(a.plus >> 64);
  g.p32_lo = (uint64_t)a.plus;
  return g;
}

inline uint32_t lemire_threshold(uint64_t t) {
  return t >= (1ull << 32) ? 0u : (uint32_t)(((1ull << 32) - t) % t);
}

// Draws to generate so that >= row_end are accepted with overwhelming
// probability (verified after the count pass; grown on the rare shortfall).
int64_t draws_needed(int64_t row_end, uint32_t thr, int attempt) {
  const double p = (double)thr / 4294967296.0;
  const double mean = (double)row_end / (1.0 - p);
  const double sd = sqrt((double)row_end * p) / (1.0 - p);
  double d = mean + 16.0 * sd + 4096.0;
  for (int i = 0; i < attempt; ++i) d *= 1.5;
  return (int64_t)d;
}

size_t ws_bytes_for(int64_t row_end, uint64_t t) {
  const uint32_t thr = lemire_threshold(t);
  if (t <= 1 || thr == 0) return 0;
  // sized for attempt 2 (two retries) -- enough in practice; else EWORKSPACE
  const int64_t n_out = (draws_needed(row_end, thr, 2) + 1) / 2;
  const int64_t warps = (n_out + kOutPerWarp - 1) / kOutPerWarp;
  return sizeof(uint32_t) * (size_t)(warps + scan_partials_len(warps) + 1);
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_hash_signs_workspace(int64_t row_end, uint64_t t, size_t *bytes) {
  if (!bytes || row_end < 0 || t < 1 || t > (1ull << 32))
    return fail(SKT_EINVAL, "skt_hash_signs_workspace", "bad arguments");
  *bytes = ws_bytes_for(row_end, t);
  return SKT_OK;
}

extern "C" skt_status skt_hash_signs(const skt_pcg64 *bucket_stream, const skt_pcg64 *sign_stream,
                                     int64_t row_begin, int64_t row_end, uint64_t t, uint32_t *h,
                                     int8_t *s, void *ws, size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_hash_signs";
  if (!bucket_stream || row_begin < 0 || row_end < row_begin || t < 1 || t > (1ull << 32))
    return fail(SKT_EINVAL, fn, "bad arguments (need 0 <= row_begin <= row_end, 1 <= t <= 2^32)");
  if (s && !sign_stream) return fail(SKT_EINVAL, fn, "sign output without a sign stream");
  const int64_t rows = row_end - row_begin;
  if (rows == 0) return SKT_OK;
  if (!h) return fail(SKT_EINVAL, fn, "h is NULL");
  cudaStream_t stream = as_stream(stream_);

  // ---- signs: integers(0, 2) never rejects -> direct
  if (s) {
    const GenParams g = make_params(*sign_stream);
    const int64_t n_out = ((row_end - 1) >> 1) - (row_begin >> 1) + 1;
    const int64_t warps = (n_out + kOutPerWarp - 1) / kOutPerWarp;
    const int64_t blocks = (warps * 32 + kThreads - 1) / kThreads;
    SKT_LAUNCH(gen_direct_kernel<1>, (unsigned)blocks, kThreads, 0, stream, g, row_begin, row_end,
               2ull, (uint32_t *)nullptr, s);
  }

  // ---- buckets
  if (t == 1) {  // numpy: rng == 0 -> fill with the offset, no draws consumed
    SKT_CUDA_TRY(cudaMemsetAsync(h, 0, sizeof(uint32_t) * rows, stream), fn);
    return check_launch(fn);
  }
  const GenParams g = make_params(*bucket_stream);
  const uint32_t thr = lemire_threshold(t);
  if (thr == 0) {
    const int64_t n_out = ((row_end - 1) >> 1) - (row_begin >> 1) + 1;
    const int64_t warps = (n_out + kOutPerWarp - 1) / kOutPerWarp;
    const int64_t blocks = (warps * 32 + kThreads - 1) / kThreads;
    SKT_LAUNCH(gen_direct_kernel<0>, (unsigned)blocks, kThreads, 0, stream, g, row_begin, row_end,
               t, h, (int8_t *)nullptr);
    return check_launch(fn);
  }

  // rejection possible: count -> scan -> verify -> write
  for (int attempt = 0; attempt < 3; ++attempt) {
    const int64_t n_out = (draws_needed(row_end, thr, attempt) + 1) / 2;
    const int64_t warps = (n_out + kOutPerWarp - 1) / kOutPerWarp;
    const size_t need = sizeof(uint32_t) * (size_t)(warps + scan_partials_len(warps) + 1);
    if (!ws || ws_bytes < need) return fail(SKT_EWORKSPACE, fn, "workspace too small");
    uint32_t *counts = (uint32_t *)ws;
    uint32_t *partials = counts + warps;
    const int64_t blocks = (warps * 32 + kThreads - 1) / kThreads;
    SKT_LAUNCH(count_accept_kernel, (unsigned)blocks, kThreads, 0, stream, g, n_out, t, thr, counts);
    skt_status st = exclusive_scan_u32(counts, warps, partials, stream, fn);
    if (st != SKT_OK) return st;
    uint32_t total = 0;
    const int64_t nb = scan_partials_len(warps) - 1;
    SKT_CUDA_TRY(cudaMemcpyAsync(&total, partials + nb, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                 stream), fn);
    SKT_CUDA_TRY(cudaStreamSynchronize(stream), fn);
    if ((int64_t)total < row_end) continue;  // astronomically rare: generate more draws
    SKT_LAUNCH(write_accept_kernel, (unsigned)blocks, kThreads, 0, stream, g, n_out, t, thr, counts,
               row_begin, row_end, h);
    return check_launch(fn);
  }
  return fail(SKT_ECUDA, fn, "could not generate enough accepted draws");
}
