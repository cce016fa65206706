// plan.cu -- K2: the sketch plan = S as a t x n CSR (reference sketch.py:149-151,
// scipy COO->CSR, a stable counting sort of row ids by bucket).  With shift > 0
// the rows are stably sorted by bucket group (h >> shift) instead -- the row
// order the grouped apply kernels sweep -- and blo[] holds each row's bucket
// inside its group.
//
// GPU form: a stable LSD radix sort of (key = h[i], value = i | sign<<31) with
// 8-bit digits (ceil(log2 t / 8) passes), then indptr[b] = lower_bound(keys, b).
// Stability inside a tile comes from warp-ordered ranking with __match_any_sync
// (no atomics on positions), so the plan is deterministic run to run.
//   tile = 8 warps x 16 rounds x 32 lanes = 4096 keys, warp w owns keys
//   [w*512, (w+1)*512) of the tile, round j = 32 consecutive keys.
#include "common.cuh"
#include "scan.cuh"

namespace skt {
namespace {

constexpr int kBits = 8;
constexpr int kBins = 1 << kBits;
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kRounds = 16;
constexpr int kTile = kThreads * kRounds;  // 4096
constexpr uint32_t kInvalid = 0xffffffffu;

__global__ void __launch_bounds__(kThreads) upsweep_kernel(const uint32_t *__restrict__ keys,
                                                           int64_t n, int shift, int64_t n_tiles,
                                                           uint32_t *__restrict__ tile_hist) {
  __shared__ uint32_t hist[kBins];
  for (int i = threadIdx.x; i < kBins; i += kThreads) hist[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 4
  for (int k = 0; k < kRounds; ++k) {
    const int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
    if (i < n) atomicAdd(&hist[(keys[i] >> shift) & (kBins - 1)], 1u);
  }
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < kBins; dgt += kThreads)
    tile_hist[(int64_t)dgt * n_tiles + blockIdx.x] = hist[dgt];
}

// kFirst: values are generated (row id | sign bit) instead of loaded.
template <bool kFirst>
__global__ void __launch_bounds__(kThreads) downsweep_kernel(
    const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
    const int8_t *__restrict__ sgn, uint32_t *__restrict__ keys_out,
    uint32_t *__restrict__ vals_out, int64_t n, int shift, int64_t n_tiles,
    const uint32_t *__restrict__ tile_offsets) {
  __shared__ uint32_t wcnt[kWarps][kBins];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kBins; i += kThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();

  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)w * (kRounds * 32);
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t key[kRounds], val[kRounds], loc[kRounds];
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    const int64_t i = base + j * 32 + lane;
    const bool valid = i < n;
    key[j] = valid ? keys_in[i] : 0u;
    if (kFirst)
      val[j] = valid ? ((uint32_t)i | (sgn && sgn[i] < 0 ? 0x80000000u : 0u)) : 0u;
    else
      val[j] = valid ? vals_in[i] : 0u;
    const uint32_t dgt = valid ? ((key[j] >> shift) & (kBins - 1)) : kInvalid;
    const uint32_t peers = __match_any_sync(0xffffffffu, dgt);
    const uint32_t old = valid ? wcnt[w][dgt] : 0u;
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[w][dgt] = old + __popc(peers);
    __syncwarp();
    loc[j] = valid ? old + __popc(peers & lt_mask) : kInvalid;
  }
  __syncthreads();
  // per-warp base of each digit: global tile offset + counts of earlier warps
  for (int dgt = threadIdx.x; dgt < kBins; dgt += kThreads) {
    uint32_t run = tile_offsets[(int64_t)dgt * n_tiles + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
      const uint32_t c = wcnt[ww][dgt];
      wcnt[ww][dgt] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    if (loc[j] != kInvalid) {
      const uint32_t pos = wcnt[w][(key[j] >> shift) & (kBins - 1)] + loc[j];
      keys_out[pos] = key[j];
      vals_out[pos] = val[j];
    }
  }
}

// t == 1 (no bits to sort): the plan is the identity with signs.
__global__ void identity_vals_kernel(const int8_t *__restrict__ sgn, int64_t n,
                                     uint32_t *__restrict__ rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    rows[i] = (uint32_t)i | (sgn && sgn[i] < 0 ? 0x80000000u : 0u);
}

// indptr[g] = first position whose group (key >> shift) is >= g, g in [0, ngroups];
// blo[i] = key & (2^shift - 1): the bucket inside its group.
__global__ void indptr_kernel(const uint32_t *__restrict__ keys, int64_t n, uint64_t ngroups,
                              int shift, int64_t *__restrict__ indptr) {
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= ngroups;
       b += (uint64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((uint64_t)(keys[mid] >> shift) < b)
        lo = mid + 1;
      else
        hi = mid;
    }
    indptr[b] = lo;
  }
}

__global__ void blo_kernel(const uint32_t *__restrict__ keys, int64_t n, uint32_t mask,
                           uint8_t *__restrict__ blo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    blo[i] = (uint8_t)(keys[i] & mask);
}

int num_passes(uint64_t t, int shift) {
  if (t <= 1) return 0;
  const int bits = 64 - __builtin_clzll(t - 1) - shift;
  return bits <= 0 ? 0 : (bits + kBits - 1) / kBits;
}

struct PlanWs {
  uint32_t *keys_a, *keys_b, *vals_b, *tile_hist, *partials;
  size_t bytes;
};

PlanWs carve(void *ws, int64_t n, uint64_t t, int shift) {
  PlanWs p{};
  const int64_t n_tiles = (n + kTile - 1) / kTile;
  const int64_t hist_len = (int64_t)kBins * n_tiles;
  auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t off = 0;
  char *base = (char *)ws;
  auto take = [&](size_t bytes) {
    char *ptr = base ? base + off : nullptr;
    off += align(bytes);
    return (uint32_t *)ptr;
  };
  if (num_passes(t, shift) > 0) {
    p.keys_a = take(sizeof(uint32_t) * n);
    p.keys_b = take(sizeof(uint32_t) * n);
    p.vals_b = take(sizeof(uint32_t) * n);
    p.tile_hist = take(sizeof(uint32_t) * hist_len);
    p.partials = take(sizeof(uint32_t) * scan_partials_len(hist_len));
  }
  p.bytes = off;
  return p;
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_plan_workspace(int64_t n, uint64_t t, int32_t shift, size_t *bytes) {
  if (!bytes || n < 0 || n >= (1LL << 31) || t < 1 || t > (1ull << 32) || shift < 0 || shift > 8)
    return fail(SKT_EINVAL, "skt_plan_workspace",
                "bad arguments (0 <= n < 2^31, 1 <= t <= 2^32, 0 <= shift <= 8)");
  *bytes = carve(nullptr, n, t, shift).bytes;
  return SKT_OK;
}

extern "C" skt_status skt_plan_build(const uint32_t *h, const int8_t *s, int64_t n, uint64_t t,
                                     int32_t shift, int64_t *indptr, uint32_t *rows, uint8_t *blo,
                                     void *ws, size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_plan_build";
  if (n < 0 || n >= (1LL << 31) || t < 1 || t > (1ull << 32) || shift < 0 || shift > 8 || !indptr ||
      (n > 0 && (!h || !rows)) || (shift > 0 && n > 0 && !blo))
    return fail(SKT_EINVAL, fn, "bad arguments (0 <= n < 2^31, 1 <= t <= 2^32, 0 <= shift <= 8)");
  cudaStream_t stream = as_stream(stream_);
  const PlanWs p = carve(ws, n, t, shift);
  if (p.bytes > 0 && (!ws || ws_bytes < p.bytes)) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  const int passes = num_passes(t, shift);
  const uint64_t ngroups = ((t - 1) >> shift) + 1;
  const uint32_t *sorted_keys = h;
  if (n > 0 && passes == 0) {
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    SKT_LAUNCH(identity_vals_kernel, (unsigned)blocks, 256, 0, stream, s, n, rows);
  } else if (n > 0) {
    const int64_t n_tiles = (n + kTile - 1) / kTile;
    const int64_t hist_len = (int64_t)kBins * n_tiles;
    const uint32_t *kin = h;
    const uint32_t *vin = nullptr;
    for (int pass = 0; pass < passes; ++pass) {
      uint32_t *kout = (pass & 1) ? p.keys_b : p.keys_a;
      uint32_t *vout = ((passes - 1 - pass) & 1) ? p.vals_b : rows;
      const int bit = shift + pass * kBits;
      SKT_LAUNCH(upsweep_kernel, (unsigned)n_tiles, kThreads, 0, stream, kin, n, bit, n_tiles,
                 p.tile_hist);
      skt_status st = exclusive_scan_u32(p.tile_hist, hist_len, p.partials, stream, fn);
      if (st != SKT_OK) return st;
      if (pass == 0)
        SKT_LAUNCH(downsweep_kernel<true>, (unsigned)n_tiles, kThreads, 0, stream, kin, nullptr, s,
                   kout, vout, n, bit, n_tiles, p.tile_hist);
      else
        SKT_LAUNCH(downsweep_kernel<false>, (unsigned)n_tiles, kThreads, 0, stream, kin, vin,
                   nullptr, kout, vout, n, bit, n_tiles, p.tile_hist);
      kin = kout;
      vin = vout;
    }
    sorted_keys = kin;
  }
  {
    const uint64_t work = ngroups + 1;
    const uint64_t blocks = std::min<uint64_t>((work + 255) / 256, 148ull * 16);
    SKT_LAUNCH(indptr_kernel, (unsigned)blocks, 256, 0, stream, sorted_keys, n, ngroups, shift, indptr);
  }
  if (shift > 0 && n > 0) {
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    SKT_LAUNCH(blo_kernel, (unsigned)blocks, 256, 0, stream, sorted_keys, n, (1u << shift) - 1u, blo);
  }
  return check_launch(fn);
}
