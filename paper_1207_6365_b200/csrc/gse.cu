// gse.cu -- generalized sparse embedding (reference GeneralizedSparseEmbedding,
// sketch.py:176-238): every input row j lands in k_blocks output rows
//   h_b(j) = outer(j) * (k v) + b v + inner_b(j),  weight sign_b(j) / sqrt(k),
// one per block b.  Its S is a t x n CSR with k entries per column; per output
// row the entries come from a single block and are in ascending j.
//
// The plan machinery of the CountSketch is reused on n' = k n "virtual rows"
// (vid = b n + j, the draw order of the reference's (k, n)-shaped streams):
// K1 draws outer buckets / inner buckets / inner signs from the reference's
// streams (1, 0) / (1, 1) / (1, 2), gse_buckets_kernel combines them into
// h(vid), K2 sorts the virtual rows by bucket (stable: ascending vid = ascending
// j inside an output row) and gse_fold_kernel rewrites the plan words to the
// input row j (sign bit kept).
//
// Apply: the reference computes self._mat @ a with scipy's csr_matvecs (dense)
// or csr_matmat (CSR): per output element, the fp64 sum over the row's entries
// in order of round(w_p * a_jc), starting from 0, without FMA contraction
// (verified bit-exact against the reference).  The weighted kernels below do
// exactly that (__dmul_rn + __dadd_rn), so the result is bit-identical.
#include <type_traits>

#include <cstdlib>

#include "common.cuh"
#include "dense_g4.cuh"

namespace skt {
namespace {

constexpr int kGseWarps = 4;

__global__ void gse_buckets_kernel(const uint32_t *__restrict__ outer, const uint32_t *__restrict__ inner,
                                   int64_t n, int k, uint32_t v, uint32_t *__restrict__ h) {
  const int64_t total = (int64_t)k * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / n, j = e - b * n;
    h[e] = outer[j] * ((uint32_t)k * v) + (uint32_t)b * v + inner[e];
  }
}

__global__ void gse_fold_kernel(uint32_t *__restrict__ rows, int64_t count, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = rows[e];
    rows[e] = (uint32_t)((int64_t)(w & 0x7fffffffu) % n) | (w & 0x80000000u);
  }
}

// dense A: warp per output row, lanes over 32-column chunks, entries in plan order
template <typename TA>
__global__ void __launch_bounds__(kGseWarps * 32) gse_dense_kernel(const int64_t *__restrict__ indptr,
                                                                   const uint32_t *__restrict__ rows, uint64_t t,
                                                                   const TA *__restrict__ a, int64_t d, int64_t lda,
                                                                   double w, double *__restrict__ sa, int64_t ldsa,
                                                                   int32_t *__restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * kGseWarps + (threadIdx.x >> 5);
  if (o >= (int64_t)t) return;
  const int64_t beg = indptr[o], end = indptr[o + 1];
  bool bad = false;
  for (int64_t c0 = 0; c0 < d; c0 += 32) {
    const int64_t c = c0 + lane;
    double acc = 0.0;
    if (c < d) {
      for (int64_t p = beg; p < end; ++p) {
        const uint32_t wd = __ldg(rows + p);
        const double x = (double)a[(int64_t)(wd & 0x7fffffffu) * lda + c];
        bad |= !isfinite(x);
        acc = __dadd_rn(acc, __dmul_rn((wd >> 31) ? -w : w, x));
      }
      sa[o * ldsa + c] = acc;
    }
  }
  if (flag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

// CSR A: warp per output row, the row's d accumulators in shared memory (or in
// the fp64 output row when too wide); the entries of each plan row are added
// in stored order (duplicate columns serialised in that order).
template <typename IP, typename IX, typename TV, bool kSmem>
__global__ void __launch_bounds__(kGseWarps * 32) gse_csr_kernel(const int64_t *__restrict__ indptr,
                                                                 const uint32_t *__restrict__ rows, uint64_t t,
                                                                 const IP *__restrict__ aip, const IX *__restrict__ aix,
                                                                 const TV *__restrict__ av, int64_t d, double w,
                                                                 double *__restrict__ sa, int64_t ldsa) {
  extern __shared__ double sacc[];
  const int lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * kGseWarps + (threadIdx.x >> 5);
  if (o >= (int64_t)t) return;
  double *acc = kSmem ? sacc + (size_t)(threadIdx.x >> 5) * d : sa + o * ldsa;
  for (int64_t c = lane; c < d; c += 32) acc[c] = 0.0;
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t beg = indptr[o], end = indptr[o + 1];
  for (int64_t p = beg; p < end; ++p) {
    const uint32_t wd = __ldg(rows + p);
    const double ws = (wd >> 31) ? -w : w;
    const int64_t j = wd & 0x7fffffffu;
    const int64_t rs = (int64_t)aip[j], re = (int64_t)aip[j + 1];
    for (int64_t q0 = rs; q0 < re; q0 += 32) {
      const int64_t q = q0 + lane;
      const bool has = q < re;
      const int64_t c = has ? (int64_t)__ldg(aix + q) : -1;
      const double v = has ? (double)__ldg(av + q) : 0.0;
      // same-column lanes add in stored (lane) order
      const unsigned peers = __match_any_sync(0xffffffffu, c);
      const int rank = __popc(peers & lt);
      const int rounds = __reduce_max_sync(0xffffffffu, has ? rank + 1 : 0);
      for (int r = 0; r < rounds; ++r) {
        if (has && rank == r) acc[c] = __dadd_rn(acc[c], __dmul_rn(ws, v));
        __syncwarp();
      }
    }
  }
  if (kSmem) {
    __syncwarp();
    for (int64_t c = lane; c < d; c += 32) sa[o * ldsa + c] = acc[c];
  }
}

template <typename IP, typename IX, typename TV>
skt_status gse_csr_launch(const int64_t *indptr, const uint32_t *rows, uint64_t t, const void *aip,
                          const void *aix, const void *av, int64_t d, double w, double *sa, int64_t ldsa,
                          cudaStream_t st) {
  static const char *fn = "skt_gse_apply_csr";
  const int64_t blocks = ((int64_t)t + kGseWarps - 1) / kGseWarps;
  const size_t smem = (size_t)kGseWarps * d * sizeof(double);
  if (smem <= 200 * 1024) {
    auto k = gse_csr_kernel<IP, IX, TV, true>;
    SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
    SKT_LAUNCH(k, (unsigned)blocks, kGseWarps * 32, smem, st, indptr, rows, t, (const IP *)aip, (const IX *)aix,
               (const TV *)av, d, w, sa, ldsa);
  } else {
    SKT_LAUNCH((gse_csr_kernel<IP, IX, TV, false>), (unsigned)blocks, kGseWarps * 32, 0, st, indptr, rows, t,
               (const IP *)aip, (const IX *)aix, (const TV *)av, d, w, sa, ldsa);
  }
  return check_launch(fn);
}

template <typename IP, typename IX>
skt_status gse_csr_v(const int64_t *indptr, const uint32_t *rows, uint64_t t, const void *aip, const void *aix,
                     const void *av, skt_dtype vt, int64_t d, double w, double *sa, int64_t ldsa, cudaStream_t st) {
  return vt == SKT_F32 ? gse_csr_launch<IP, IX, float>(indptr, rows, t, aip, aix, av, d, w, sa, ldsa, st)
                       : gse_csr_launch<IP, IX, double>(indptr, rows, t, aip, aix, av, d, w, sa, ldsa, st);
}

inline unsigned grid_elems(int64_t total) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)kNumSMs * 16));
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_gse_buckets(const uint32_t *outer, const uint32_t *inner, int64_t n, int32_t k,
                                      uint32_t v, uint64_t q, uint32_t *h, void *stream_) {
  static const char *fn = "skt_gse_buckets";
  if (n < 0 || k < 1 || v < 1 || q < 1 || (double)q * k * v > 4294967295.0 || (n > 0 && (!outer || !inner || !h)))
    return fail(SKT_EINVAL, fn, "bad arguments (t = q k v must fit in 32 bits)");
  if (n == 0) return SKT_OK;
  SKT_LAUNCH(gse_buckets_kernel, grid_elems((int64_t)k * n), 256, 0, as_stream(stream_), outer, inner, n, (int)k, v, h);
  return check_launch(fn);
}

extern "C" skt_status skt_gse_fold_rows(uint32_t *rows, int64_t count, int64_t n, void *stream_) {
  static const char *fn = "skt_gse_fold_rows";
  if (count < 0 || n < 1 || (count > 0 && !rows)) return fail(SKT_EINVAL, fn, "bad arguments");
  if (count == 0) return SKT_OK;
  SKT_LAUNCH(gse_fold_kernel, grid_elems(count), 256, 0, as_stream(stream_), rows, count, n);
  return check_launch(fn);
}

extern "C" skt_status skt_gse_apply_dense(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                                          const void *a, skt_dtype a_dtype, int64_t d, int64_t lda, double weight,
                                          double *sa, int64_t ldsa, int32_t *nonfinite_flag, void *stream_) {
  static const char *fn = "skt_gse_apply_dense";
  if (!indptr || t < 1 || n < 0 || d < 0 || lda < d || ldsa < d || (a_dtype != SKT_F32 && a_dtype != SKT_F64) ||
      !(fabs(weight) <= 1.0))
    return fail(SKT_EINVAL, fn, "bad arguments");
  cudaStream_t st = as_stream(stream_);
  if (nonfinite_flag) SKT_CUDA_TRY(cudaMemsetAsync(nonfinite_flag, 0, sizeof(int32_t), st), fn);
  if (d == 0) return SKT_OK;
  if (!sa) return fail(SKT_EINVAL, fn, "NULL output");
  // rows of 512 B .. 2 KB: the K3 TMA gather4 kernel with weighted terms
  {
    const int64_t esz = a_dtype == SKT_F32 ? 4 : 8, row_bytes = d * esz, lda_bytes = lda * esz;
    const int nbox = g4_boxes(d, esz);
    const char *g4e = getenv("SKT_DENSE_G4");
    CUtensorMap map;
    if (!(g4e && g4e[0] == '0') && nbox > 0 && lda_bytes % 16 == 0 && (uintptr_t)a % 16 == 0 && n > 0 &&
        n < (1LL << 31) && make_row_map(&map, a, a_dtype == SKT_F64, n, d, lda_bytes, d / nbox)) {
      const size_t smem = dense_g4_smem((int)row_bytes);
      const int64_t gblocks = ((int64_t)t + kG4Warps - 1) / kG4Warps;
      typedef void (*KFn)(const CUtensorMap, const int64_t *, const uint32_t *, uint64_t, int, int, double *, int64_t,
                          int32_t *, const unsigned char *, int64_t, double, int, const PushTable);
#define SKT_G4W(TIN)                                                                \
  (row_bytes == 512    ? (KFn)dense_g4_kernel<TIN, double, 1, true, true>           \
   : row_bytes == 1024 ? (KFn)dense_g4_kernel<TIN, double, 2, true, true>           \
   : row_bytes == 2048 ? (KFn)dense_g4_kernel<TIN, double, 4, true, true>           \
   : row_bytes < 1024  ? (KFn)dense_g4_kernel<TIN, double, 2, false, true>          \
                       : (KFn)dense_g4_kernel<TIN, double, 4, false, true>)
      const KFn k = a_dtype == SKT_F32 ? SKT_G4W(float) : SKT_G4W(double);
#undef SKT_G4W
      SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
      SKT_LAUNCH(k, (unsigned)gblocks, kG4Warps * 32, smem, st, map, indptr, rows, t, (int)row_bytes, (int)d, sa,
                 ldsa, nonfinite_flag, (const unsigned char *)a, lda_bytes, weight, nbox, PushTable{});
      return check_launch(fn);
    }
  }
  const int64_t blocks = ((int64_t)t + kGseWarps - 1) / kGseWarps;
  if (a_dtype == SKT_F32)
    SKT_LAUNCH(gse_dense_kernel<float>, (unsigned)blocks, kGseWarps * 32, 0, st, indptr, rows, t, (const float *)a,
               d, lda, weight, sa, ldsa, nonfinite_flag);
  else
    SKT_LAUNCH(gse_dense_kernel<double>, (unsigned)blocks, kGseWarps * 32, 0, st, indptr, rows, t,
               (const double *)a, d, lda, weight, sa, ldsa, nonfinite_flag);
  return check_launch(fn);
}

extern "C" skt_status skt_gse_apply_csr(const int64_t *indptr, const uint32_t *rows, uint64_t t,
                                        const void *a_indptr, skt_itype indptr_type, const void *a_indices,
                                        skt_itype index_type, const void *a_vals, skt_dtype val_dtype, int64_t d,
                                        double weight, double *sa, int64_t ldsa, void *stream_) {
  static const char *fn = "skt_gse_apply_csr";
  if (!indptr || t < 1 || d < 0 || ldsa < d || !a_indptr || (indptr_type != SKT_I32 && indptr_type != SKT_I64) ||
      (index_type != SKT_I32 && index_type != SKT_I64) || (val_dtype != SKT_F32 && val_dtype != SKT_F64))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (d == 0) return SKT_OK;
  if (!sa) return fail(SKT_EINVAL, fn, "NULL output");
  cudaStream_t st = as_stream(stream_);
  if (indptr_type == SKT_I32)
    return index_type == SKT_I32
               ? gse_csr_v<int32_t, int32_t>(indptr, rows, t, a_indptr, a_indices, a_vals, val_dtype, d, weight, sa, ldsa, st)
               : gse_csr_v<int32_t, int64_t>(indptr, rows, t, a_indptr, a_indices, a_vals, val_dtype, d, weight, sa, ldsa, st);
  return index_type == SKT_I32
             ? gse_csr_v<int64_t, int32_t>(indptr, rows, t, a_indptr, a_indices, a_vals, val_dtype, d, weight, sa, ldsa, st)
             : gse_csr_v<int64_t, int64_t>(indptr, rows, t, a_indptr, a_indices, a_vals, val_dtype, d, weight, sa, ldsa, st);
}
