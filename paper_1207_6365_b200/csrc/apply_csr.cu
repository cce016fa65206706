// apply_csr.cu -- K4: SA = S.A for CSR A (reference sketch.py:155-164: repeat
// + np.bincount, i.e. out[h(i)*d + j] += s(i) * v over the stored nonzeros in
// row-major order, fp64 from +0.0).
//
// One warp owns one bucket and keeps its SA row as d fp64 accumulators in
// shared memory.  The bucket's rows are taken 32 at a time from the plan
// (ascending row id); their nonzeros are first staged into shared memory with
// coalesced, flattened loads (every lane has many loads in flight), then
// accumulated row by row in plan order.  Inside a row the columns are distinct
// (canonical CSR), so one warp step adds up to 32 of them without conflicts;
// successive rows are ordered by __syncwarp.  Per output element the additions
// therefore happen in ascending row order, exactly as the bincount does --
// bit-identical fp64.  Non-canonical rows (duplicate columns) are serialised
// in stored order with __match_any_sync.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "csr_group.cuh"
#include "csr_lane.cuh"
#include "csr_sweep.cuh"
#include "csr_quad.cuh"
#include "csr_tile.cuh"
#include "csr_wide.cuh"

namespace skt {
namespace {

constexpr int kStage = 256;  // staged nonzeros per warp per window
constexpr int kMaxWarps = 8;

struct WarpSmem {
  // byte offsets inside one warp's slice
  static __host__ __device__ size_t acc_bytes(int64_t d) { return ((size_t)d * 8 + 15) & ~(size_t)15; }
  static __host__ __device__ size_t bytes(int64_t d) {
    return acc_bytes(d) + kStage * 8 + kStage * 4 + 34 * 4 + 32 * 8;
  }
};

template <typename I>
__device__ __forceinline__ int64_t ld_idx(const I *p) {
  return (int64_t)__ldg(p);
}

template <typename IP, typename IX, typename TV, typename TOut, bool kCanon>
__global__ void __launch_bounds__(kMaxWarps * 32) apply_csr_kernel(
    const int64_t *__restrict__ pindptr, const uint32_t *__restrict__ prow, uint64_t t,
    const IP *__restrict__ aip, const IX *__restrict__ aix, const TV *__restrict__ av, int64_t d,
    TOut *__restrict__ sa, int64_t ldsa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t bucket = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (bucket >= (int64_t)t) return;  // whole warp exits together

  unsigned char *base = smem_raw + (size_t)w * WarpSmem::bytes(d);
  double *acc = (double *)base;
  double *sval = (double *)(base + WarpSmem::acc_bytes(d));
  int32_t *scol = (int32_t *)(sval + kStage);
  int32_t *soff = scol + kStage;             // 33 used
  int64_t *srs = (int64_t *)(soff + 34);     // 32 row starts, sign in bit 63

  for (int64_t c = lane; c < d; c += 32) acc[c] = 0.0;
  const int64_t beg = pindptr[bucket], end = pindptr[bucket + 1];
  const uint32_t lt_mask = (1u << lane) - 1u;

  for (int64_t k0 = beg; k0 < end; k0 += 32) {
    const int nrows = (int)((end - k0) < 32 ? (end - k0) : 32);
    const bool valid = lane < nrows;
    const uint32_t wrd = valid ? __ldg(prow + k0 + lane) : 0u;
    const int64_t row = wrd & 0x7fffffffu;
    const int64_t rs = valid ? ld_idx(aip + row) : 0;
    const int64_t re = valid ? ld_idx(aip + row + 1) : 0;
    const int32_t len = (int32_t)(re - rs);
    // exclusive scan of row lengths
    int32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int32_t off = incl - len;
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    soff[lane] = off;
    if (lane == 31) soff[32] = total;
    srs[lane] = rs | ((int64_t)(wrd >> 31) << 63);
    __syncwarp();

    for (int32_t w0 = 0; w0 < total; w0 += kStage) {
      const int32_t wend = min(total, w0 + kStage);
      // ---- stage: flattened, coalesced loads of this window's nonzeros
      for (int32_t f = w0 + lane; f < wend; f += 32) {
        int lo = 0, hi = nrows;  // find r: soff[r] <= f < soff[r+1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (soff[mid] <= f) lo = mid; else hi = mid;
        }
        const int64_t rsw = srs[lo];
        const int64_t p = (rsw & 0x7fffffffffffffffLL) + (f - soff[lo]);
        const double v = (double)av[p];
        scol[f - w0] = (int32_t)aix[p];
        sval[f - w0] = rsw < 0 ? -v : v;
      }
      __syncwarp();
      // ---- accumulate in plan (= ascending row) order
      for (int r = 0; r < nrows; ++r) {
        const int32_t pb = max(soff[r], w0), pe = min(soff[r + 1], wend);
        for (int32_t p0 = pb; p0 < pe; p0 += 32) {
          const int32_t p = p0 + lane;
          const bool has = p < pe;
          const int32_t c = has ? scol[p - w0] : -1;
          const double v = has ? sval[p - w0] : 0.0;
          if (kCanon) {
            if (has) acc[c] += v;
          } else {
            const uint32_t peers = __match_any_sync(0xffffffffu, c);
            const int rank = __popc(peers & lt_mask);
            const int rounds = __reduce_max_sync(0xffffffffu, has ? rank + 1 : 0);
            for (int rr = 0; rr < rounds; ++rr) {
              if (has && rank == rr) acc[c] += v;
              __syncwarp();
            }
          }
          __syncwarp();
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
  TOut *o = sa + bucket * ldsa;
  for (int64_t c = lane; c < d; c += 32) o[c] = (TOut)acc[c];
}

// SKT_CSR_KERNEL=lane selects the bucket-lane kernel over the tile kernel (A/B).
inline bool force_lane() {
  static const bool on = [] {
    const char *e = getenv("SKT_CSR_KERNEL");
    return e && e[0] == 'l';
  }();
  return on;
}

// SKT_CSR_KERNEL=tile keeps the tile kernel where the 128-bit-load kernel (csr_quad.cuh) would run (A/B).
inline bool force_tile() {
  static const bool on = [] {
    const char *e = getenv("SKT_CSR_KERNEL");
    return e && e[0] == 't';
  }();
  return on;
}

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch(const int64_t *pindptr, const uint32_t *prow, const uint8_t *blo, int shift,
                  uint64_t t, int64_t n, const void *aip, const void *aix, const void *av,
                  int64_t nnz, int64_t d, void *sa, int64_t ldsa, uint32_t flags, cudaStream_t stream) {
  static const char *fn = "skt_apply_csr";
  const bool canon = (flags & SKT_CSR_CANONICAL) != 0;
  if (flags & SKT_CSR_FAST) {  // unordered atomics into a zeroed SA (any d)
    if (shift != 0) return fail(SKT_EINVAL, fn, "fast mode needs the per-bucket plan (shift 0)");
    SKT_CUDA_TRY(cudaMemset2DAsync(sa, ldsa * sizeof(TOut), 0, d * sizeof(TOut), t, stream), fn);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)kNumSMs * 16));
    SKT_LAUNCH((csr_atomic_kernel<IP, IX, TV, TOut>), (unsigned)blocks, 256, 0, stream, pindptr, prow, t, n,
               (const IP *)aip, (const IX *)aix, (const TV *)av, (TOut *)sa, ldsa);
    return check_launch(fn);
  }
  const int64_t gb = 1LL << shift;
  const bool short_rows = n > 0 && nnz <= 8 * n;  // mean row length <= 8
  // (1a) tiled sweep over a bucket-group plan (rows of ~8+ nonzeros, narrow d,
  // groups of 2 or 4 buckets)
  static const bool sweep_short = getenv("SKT_SWEEP_SHORT") != nullptr;  // A/B: sweep short rows too
  if (canon && (shift == 1 || shift == 2) && (!short_rows || sweep_short) && d <= kTileMaxD) {
    const int dp = (int)((d + 1) & ~1LL);
    const int rmax = (int)std::min<int64_t>(32, tile_bytes<TV>() / ((int64_t)dp * sizeof(TV)));
    int R = 16;
    if (const char *e = getenv("SKT_SWEEP_R")) R = atoi(e) <= 16 ? 16 : 32;
    if (R > rmax) R = 16;
    const int64_t ngroups = (int64_t)((t - 1) >> shift) + 1;
    const size_t smem = sweep_slice_bytes(R, dp, (int)sizeof(TV)) * kSweepWarps;
    if (R <= rmax) {
      const int64_t blocks = (ngroups + kSweepWarps - 1) / kSweepWarps;
      const int chunks = (int)((d + 63) / 64);
      typedef void (*KFn)(const int64_t *, const uint32_t *, const uint8_t *, int64_t, uint64_t, const IP *,
                          const IX *, const TV *, int, int, TOut *, int64_t);
#define SKT_SWEEP_PICK(RT, SH)                                                                    \
  (chunks <= 1 ? (KFn)csr_sweep_kernel<IP, IX, TV, TOut, 1, RT, SH>                               \
               : chunks <= 2 ? (KFn)csr_sweep_kernel<IP, IX, TV, TOut, 2, RT, SH>                 \
                             : (KFn)csr_sweep_kernel<IP, IX, TV, TOut, 4, RT, SH>)
      const KFn k = R == 16 ? (shift == 1 ? SKT_SWEEP_PICK(16, 1) : SKT_SWEEP_PICK(16, 2))
                            : (shift == 1 ? SKT_SWEEP_PICK(32, 1) : SKT_SWEEP_PICK(32, 2));
#undef SKT_SWEEP_PICK
      SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
      SKT_LAUNCH(k, (unsigned)blocks, kSweepWarps * 32, smem, stream, pindptr, prow, blo, ngroups, t,
                 (const IP *)aip, (const IX *)aix, (const TV *)av, (int)d, dp, (TOut *)sa, ldsa);
      return check_launch(fn);
    }
  }
  // (1) grouped sweep over a bucket-group plan (short rows)
  const size_t group_acc = (size_t)gb * d * sizeof(double);
  if (canon && shift > 0 && group_acc <= 24 * 1024) {
    const int64_t ngroups = (int64_t)((t - 1) >> shift) + 1;
    const size_t smem = group_acc * kGroupWarps;
    const int64_t blocks = (ngroups + kGroupWarps - 1) / kGroupWarps;
    auto k = short_rows ? csr_group_kernel<IP, IX, TV, TOut, 8> : csr_group_kernel<IP, IX, TV, TOut, 16>;
    SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
    SKT_LAUNCH(k, (unsigned)blocks, kGroupWarps * 32, smem, stream, pindptr, prow, blo, ngroups,
               shift, t, (const IP *)aip, (const IX *)aix, (const TV *)av, (int)d, (TOut *)sa, ldsa);
    return check_launch(fn);
  }
  // (2a) densify tiles with 128-bit loads: fp32 values, int32 columns, d <= 64, rows of ~8-20
  // nonzeros, index / value arrays on 16-byte boundaries
  if constexpr (std::is_same<TV, float>::value && std::is_same<IX, int32_t>::value) {
    if (canon && shift == 0 && d <= kQuadD && !short_rows && nnz <= 20 * n && !force_lane() && !force_tile() &&
        ((reinterpret_cast<uintptr_t>(aix) | reinterpret_cast<uintptr_t>(av)) & 15) == 0) {
      const size_t smem = (size_t)kQuadTileBytes * kQuadWarps;
      const int64_t blocks = ((int64_t)t + kQuadWarps - 1) / kQuadWarps;
      auto k = csr_quad_kernel<IP, TOut>;
      SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
      SKT_LAUNCH(k, (unsigned)blocks, kQuadWarps * 32, smem, stream, pindptr, prow, t, (const IP *)aip,
                 (const int32_t *)aix, (const float *)av, (int)d, (TOut *)sa, ldsa);
      return check_launch(fn);
    }
  }
  // (2) densify-in-shared-memory tiles, warp per bucket (longer rows)
  if (canon && shift == 0 && d <= kTileMaxD && !force_lane()) {
    const int dp = (int)((d + 1) & ~1LL);
    const int R = (int)std::min<int64_t>(32, tile_bytes<TV>() / ((int64_t)dp * sizeof(TV)));
    const size_t smem = (size_t)tile_slice_bytes<TV>() * kTileWarps;
    const int64_t blocks = ((int64_t)t + kTileWarps - 1) / kTileWarps;
    const int chunks = (int)((d + 63) / 64);
    auto k = chunks <= 1 ? csr_tile_kernel<IP, IX, TV, TOut, 1>
                         : chunks <= 2 ? csr_tile_kernel<IP, IX, TV, TOut, 2> : csr_tile_kernel<IP, IX, TV, TOut, 4>;
    SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
    SKT_LAUNCH(k, (unsigned)blocks, kTileWarps * 32, smem, stream, pindptr, prow, t, (const IP *)aip,
               (const IX *)aix, (const TV *)av, (int)d, dp, R, (TOut *)sa, ldsa);
    return check_launch(fn);
  }
  // (3) bucket-lane kernel: BPW buckets per warp, CS lanes (column ranges) per bucket
  if (canon && shift == 0) {
    // about 16 warps per SM resident at once: CS = 32 * 2368 / t, power of two in [1, 8]
    int cs = 1;
    while (cs < 8 && cs < d && (double)t * cs / 32.0 < 148.0 * 12) cs <<= 1;
    size_t lane_smem = 0;
    void (*k)(const int64_t *, const uint32_t *, uint64_t, const IP *, const IX *, const TV *, int, TOut *,
              int64_t) = nullptr;
    switch (cs) {  // 16 (or 32) rows per round: RPB = 16 / buckets-per-warp
      case 1: k = csr_lane_kernel<IP, IX, TV, TOut, 1, 1>; lane_smem = LaneSmem<IX, TV, 32, 1>::bytes((int)d); break;
      case 2: k = csr_lane_kernel<IP, IX, TV, TOut, 2, 1>; lane_smem = LaneSmem<IX, TV, 16, 1>::bytes((int)d); break;
      case 4: k = csr_lane_kernel<IP, IX, TV, TOut, 4, 2>; lane_smem = LaneSmem<IX, TV, 8, 2>::bytes((int)d); break;
      default: k = csr_lane_kernel<IP, IX, TV, TOut, 8, 4>; lane_smem = LaneSmem<IX, TV, 4, 4>::bytes((int)d); break;
    }
    if (lane_smem <= 200 * 1024) {
      const int64_t bpw = 32 / cs;
      const int64_t blocks = ((int64_t)t + bpw - 1) / bpw;
      SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lane_smem), fn);
      SKT_LAUNCH(k, (unsigned)blocks, 32, lane_smem, stream, pindptr, prow, t, (const IP *)aip,
                 (const IX *)aix, (const TV *)av, (int)d, (TOut *)sa, ldsa);
      return check_launch(fn);
    }
  }
  if (shift != 0)
    return fail(SKT_EINVAL, fn, "non-canonical or wide-d CSR needs the per-bucket plan (shift 0)");
  const size_t per_warp = WarpSmem::bytes(d);
  const size_t kSmemMax = 200 * 1024;
  int warps = (int)std::min<size_t>(kMaxWarps, kSmemMax / per_warp);
  if (warps < 1) {
    // (5) too wide for shared memory: fp64 accumulation in the output row, a
    // block per bucket (few buckets) or a warp per bucket (SKT_CSR_ROWSEQ=warp)
    if (!canon) return fail(SKT_ENOTSUP, fn, "non-canonical CSR this wide is not supported");
    if (!std::is_same<TOut, double>::value)
      return fail(SKT_ENOTSUP, fn, "deterministic wide-d CSR writes fp64 SA (round on the host side)");
    const char *rq = getenv("SKT_CSR_ROWSEQ");
    if (!(rq && rq[0] == 'w')) {
      SKT_LAUNCH((csr_rowseq_block_kernel<IP, IX, TV>), (unsigned)t, kRowseqThreads, 0, stream, pindptr, prow, t,
                 (const IP *)aip, (const IX *)aix, (const TV *)av, d, (double *)sa, ldsa);
      return check_launch(fn);
    }
    const int64_t blocks = ((int64_t)t + 3) / 4;
    SKT_LAUNCH((csr_rowseq_kernel<IP, IX, TV, TOut>), (unsigned)blocks, 128, 0, stream, pindptr, prow, t,
               (const IP *)aip, (const IX *)aix, (const TV *)av, d, (double *)nullptr, (TOut *)sa, ldsa);
    return check_launch(fn);
  }
  const size_t smem = per_warp * warps;
  const int64_t blocks = ((int64_t)t + warps - 1) / warps;
  auto k = canon ? apply_csr_kernel<IP, IX, TV, TOut, true> : apply_csr_kernel<IP, IX, TV, TOut, false>;
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
  SKT_LAUNCH(k, (unsigned)blocks, warps * 32, smem, stream, pindptr, prow, t, (const IP *)aip,
             (const IX *)aix, (const TV *)av, d, (TOut *)sa, ldsa);
  return check_launch(fn);
}

template <typename IP, typename IX>
skt_status by_vals(const int64_t *pindptr, const uint32_t *prow, const uint8_t *blo, int shift,
                   uint64_t t, int64_t n, const void *aip, const void *aix, const void *av,
                   skt_dtype vt, int64_t nnz, int64_t d, void *sa, skt_dtype ot, int64_t ldsa,
                   uint32_t flags, cudaStream_t s) {
  if (vt == SKT_F32)
    return ot == SKT_F64 ? launch<IP, IX, float, double>(pindptr, prow, blo, shift, t, n, aip, aix, av, nnz, d, sa, ldsa, flags, s)
                         : launch<IP, IX, float, float>(pindptr, prow, blo, shift, t, n, aip, aix, av, nnz, d, sa, ldsa, flags, s);
  return ot == SKT_F64 ? launch<IP, IX, double, double>(pindptr, prow, blo, shift, t, n, aip, aix, av, nnz, d, sa, ldsa, flags, s)
                       : launch<IP, IX, double, float>(pindptr, prow, blo, shift, t, n, aip, aix, av, nnz, d, sa, ldsa, flags, s);
}


}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_apply_csr(const int64_t *indptr, const uint32_t *rows,
                                    const uint8_t *blo, int32_t shift, uint64_t t, int64_t n,
                                    const void *a_indptr, skt_itype indptr_type,
                                    const void *a_indices, skt_itype index_type,
                                    const void *a_vals, skt_dtype val_dtype, int64_t nnz,
                                    int64_t d, void *sa, skt_dtype sa_dtype, int64_t ldsa,
                                    uint32_t flags, void *stream_) {
  static const char *fn = "skt_apply_csr";
  if (!indptr || t < 1 || t > (1ull << 32) || n < 0 || d < 0 || ldsa < d || !a_indptr ||
      shift < 0 || shift > 8 || (shift > 0 && n > 0 && !blo) ||
      (indptr_type != SKT_I32 && indptr_type != SKT_I64) ||
      (index_type != SKT_I32 && index_type != SKT_I64) ||
      (val_dtype != SKT_F32 && val_dtype != SKT_F64) ||
      (sa_dtype != SKT_F32 && sa_dtype != SKT_F64) || d >= (1LL << 31) || nnz < 0)
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (d == 0) return SKT_OK;
  if (!sa || (n > 0 && !rows)) return fail(SKT_EINVAL, fn, "NULL buffer");
  cudaStream_t s = as_stream(stream_);
  if (indptr_type == SKT_I32)
    return index_type == SKT_I32
               ? by_vals<int32_t, int32_t>(indptr, rows, blo, shift, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, flags, s)
               : by_vals<int32_t, int64_t>(indptr, rows, blo, shift, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, flags, s);
  return index_type == SKT_I32
             ? by_vals<int64_t, int32_t>(indptr, rows, blo, shift, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, flags, s)
             : by_vals<int64_t, int64_t>(indptr, rows, blo, shift, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, flags, s);
}

