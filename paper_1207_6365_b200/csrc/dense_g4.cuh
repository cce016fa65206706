// dense_g4.cuh -- K3 on TMA gather4: SA = S.A for dense row-major A whose rows
// are 16-byte multiples of 128 B .. 1 KB (BASELINE config 3: 512 B rows).
//
// One warp per bucket.  Lane 0 issues cp.async.bulk.tensor.2d ... tile::gather4:
// four rows at arbitrary row coordinates of A (the next four plan rows of the
// bucket) land in one shared-memory stage per instruction, completion counted
// in bytes on the stage's mbarrier.  A kG4Stages-deep ring per warp keeps 16
// rows (8 KB at 512 B) in flight without holding registers, and the TMA engine
// is issued once per 2 KB -- a 1D bulk copy per row is TMA-issue bound at
// ~46 SM cycles per copy (3.8 TB/s on 512 B rows), gather4 is not
// (tools/gather4_bench.cu: 7.15 TB/s for config 3's random rows incl. the fp64
// accumulate, the streaming-read ceiling).
//
// The plan words (row | sign << 31) are read 32 at a time, coalesced, one
// chunk ahead; the quad's rows and signs are broadcast with shuffles.  The
// lanes consume a landed stage row by row: lane l owns the 16-byte column
// chunks l, l + 32 of a row and adds s_i * A[i, cols] into fp64 accumulators in
// ascending row order from +0.0 -- the reference's csr_matvecs order, so the
// fp64 result is bit-identical.  The non-finite scan of as_dense is fused.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "dense_tma.cuh"

namespace skt {
namespace {

#ifndef SKT_G4_WARPS
#define SKT_G4_WARPS 4
#endif
#ifndef SKT_G4_STAGES
#define SKT_G4_STAGES 6
#endif
constexpr int kG4Warps = SKT_G4_WARPS;
constexpr int kG4Stages = SKT_G4_STAGES;  // quads in flight per warp (<= 8: issues stay within the next word chunk)

__device__ __forceinline__ void g4_load(void *dst, const CUtensorMap *map, uint64_t *bar, int col, int r0, int r1,
                                        int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}

// s_i * A[i, cols of one 16-byte chunk] into fp64: the sign is an XOR of the
// sign bits (exact), then (fp32) convert and add -- acc + (double)(s x), the
// reference's value
template <typename TIn>
struct G4;
template <>
struct G4<float> {
  static constexpr int E = 4;
  __device__ static __forceinline__ void add(const uint4 &u, uint32_t m, double (&acc)[4]) {
    acc[0] += (double)__uint_as_float(u.x ^ m);
    acc[1] += (double)__uint_as_float(u.y ^ m);
    acc[2] += (double)__uint_as_float(u.z ^ m);
    acc[3] += (double)__uint_as_float(u.w ^ m);
  }
  // weighted (generalized embedding): acc + fl(w (s x)), no fused multiply-add
  __device__ static __forceinline__ void add_w(const uint4 &u, uint32_t m, double w, double (&acc)[4]) {
    acc[0] = __dadd_rn(acc[0], __dmul_rn(w, (double)__uint_as_float(u.x ^ m)));
    acc[1] = __dadd_rn(acc[1], __dmul_rn(w, (double)__uint_as_float(u.y ^ m)));
    acc[2] = __dadd_rn(acc[2], __dmul_rn(w, (double)__uint_as_float(u.z ^ m)));
    acc[3] = __dadd_rn(acc[3], __dmul_rn(w, (double)__uint_as_float(u.w ^ m)));
  }
};
template <>
struct G4<double> {
  static constexpr int E = 2;
  __device__ static __forceinline__ void add(const uint4 &u, uint32_t m, double (&acc)[2]) {
    acc[0] += __longlong_as_double((long long)(((uint64_t)(u.y ^ m) << 32) | u.x));
    acc[1] += __longlong_as_double((long long)(((uint64_t)(u.w ^ m) << 32) | u.z));
  }
  __device__ static __forceinline__ void add_w(const uint4 &u, uint32_t m, double w, double (&acc)[2]) {
    acc[0] = __dadd_rn(acc[0], __dmul_rn(w, __longlong_as_double((long long)(((uint64_t)(u.y ^ m) << 32) | u.x))));
    acc[1] = __dadd_rn(acc[1], __dmul_rn(w, __longlong_as_double((long long)(((uint64_t)(u.w ^ m) << 32) | u.z))));
  }
};

template <typename TIn, bool kW>
__device__ __forceinline__ void g4_term(const uint4 &u, uint32_t m, double w, double (&acc)[G4<TIn>::E]) {
  if (kW)
    G4<TIn>::add_w(u, m, w, acc);
  else
    G4<TIn>::add(u, m, acc);
}

// Finiteness of the bucket's rows (as_dense's scan, _validation.py:25-26).
// A non-finite input makes its column's fp64 sum non-finite (inf stays inf,
// inf - inf and NaN give NaN; a weight |w| <= 1 keeps finite terms finite), so
// only a bucket whose sums are not all finite can hold one.  fp32 inputs cannot overflow an fp64 sum of < 2^31 rows, so
// for them the test of the sums is exact; fp64 sums of finite values can
// overflow, so such a bucket's rows are re-scanned element by element (rare).
template <typename TIn>
__device__ bool g4_rescan(const unsigned char *a, int64_t lda_bytes, const int64_t beg, int nrows,
                          const uint32_t *__restrict__ rows, int row_bytes, int lane) {
  bool bad = false;
  for (int p = 0; p < nrows; ++p) {
    const unsigned char *r = a + (int64_t)(__ldg(rows + beg + p) & 0x7fffffffu) * lda_bytes;
    for (int off = 4 * lane; off < row_bytes; off += 128) {
      const uint32_t w = *reinterpret_cast<const uint32_t *>(r + off);
      if (sizeof(TIn) == 4) bad |= (w & 0x7f800000u) == 0x7f800000u;
      else if (off & 4) bad |= (w & 0x7ff00000u) == 0x7ff00000u;  // the high word of each double
    }
  }
  return __any_sync(0xffffffffu, bad);
}

// Fused exchange (row-sharded multi-GPU S.A): instead of writing its partial
// bucket row into its own SA, the kernel stores it straight into the owner
// rank's receive buffer -- a peer pointer over NVLink (symmetric memory) --
// slot [my_rank][bucket - bounds[owner]], so the transfer overlaps the
// remaining buckets' compute; the owner then sums its N slots in rank order.
constexpr int kPushMaxRanks = 8;
struct PushTable {
  void *peer[kPushMaxRanks];           // receive buffer base of each rank (device / peer pointers)
  int64_t bounds[kPushMaxRanks + 1];   // owner g holds buckets [bounds[g], bounds[g + 1])
  int64_t cap;                         // bucket rows per source slot (>= max owner range)
  int64_t ldr;                         // row stride of a slot (elements)
  int nranks, me;
  int64_t b0;                          // global bucket id of local bucket 0 (bucket-range launches)
};

// K = 16-byte chunks per lane per row (row_bytes <= K * 512).  A row is fetched
// as nbox (1 or 2) column boxes of row_bytes / nbox (a box is <= 256 elements,
// 1 KB); a stage holds box b's four rows at b * 4 * box_bytes.
// kW: every term weighted by w (the generalized embedding's 1/sqrt(k), with
// the reference's separate rounding of the product), otherwise w is unused.
template <typename TIn, typename TOut, int K, bool kFull, bool kW = false, bool kPush = false>
__global__ void __launch_bounds__(kG4Warps * 32) dense_g4_kernel(const __grid_constant__ CUtensorMap map,
                                                                 const int64_t *__restrict__ indptr,
                                                                 const uint32_t *__restrict__ rows, uint64_t t,
                                                                 int row_bytes, int d, TOut *__restrict__ sa,
                                                                 int64_t ldsa, int32_t *__restrict__ flag,
                                                                 const unsigned char *__restrict__ a_raw,
                                                                 int64_t lda_bytes, double wgt, int nbox,
                                                                 const __grid_constant__ PushTable push) {
  constexpr int E = G4<TIn>::E;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[kG4Warps][kG4Stages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t bucket = (int64_t)blockIdx.x * kG4Warps + w;
  if (bucket >= (int64_t)t) return;
  const int stage_bytes = 4 * row_bytes;                // the four rows, packed
  const int stage_stride = (stage_bytes + 127) & ~127;  // TMA tensor destinations are 128-byte aligned
  unsigned char *ring = smem_raw + (size_t)w * kG4Stages * stage_stride;
  // two column boxes only for rows > 1 KB (K = 4); otherwise one box = the row
  const int box_bytes = K > 2 ? row_bytes / nbox : row_bytes, box_elems = K > 2 ? d / nbox : d;
  // this lane's 16-byte column chunks: offset inside a stage (row 0) per k,
  // the lane's own offset folded into the ring base when there is one box
  const uint32_t ring_s = smem_u32(ring) + (K > 2 ? 0u : 16u * lane);
  uint32_t loff[K];
  bool lval[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int o = k * 512 + 16 * lane;
    lval[k] = kFull || o < row_bytes;
    if (K > 2) {
      const int b = o >= box_bytes ? 1 : 0;
      loff[k] = (uint32_t)(b * 4 * box_bytes + (o - b * box_bytes));
    } else {
      loff[k] = (uint32_t)(k * 512);
    }
  }
  if (lane == 0)
    for (int s = 0; s < kG4Stages; ++s) mbar_init(&bars[w][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();

  const int64_t beg = indptr[bucket], end = indptr[bucket + 1];
  const int nrows = (int)(end - beg);
  const int nq = (nrows + 3) >> 2;
  // plan words: lane j <-> position 32 c + j of the bucket (chunk c)
  auto words = [&](int c) -> uint32_t {
    const int p = 32 * c + lane;
    return p < nrows ? __ldg(rows + beg + p) : 0u;
  };
  // chunk c (being consumed), c + 1 (issues run up to 4 quads ahead) and
  // c + 2 (in flight: 12 quads of consumption to arrive)
  uint32_t wc = words(0), wn = words(1), wn2 = words(2);
  uint32_t sgn = __ballot_sync(0xffffffffu, (wc >> 31) != 0);  // sign bits of chunk c's rows
  // issue quad q (its chunk is c0 = the chunk of the quad being consumed, or the next one)
  auto issue = [&](int q, int c0) {
    const uint32_t src = (q >> 3) == c0 ? wc : wn;
    const int l0 = (4 * q) & 31;
    int r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t wd = __shfl_sync(0xffffffffu, src, l0 + j);
      // the last quad's padding slots fetch its first row again (never added)
      r[j] = 4 * q + j < nrows ? (int)(wd & 0x7fffffffu) : r[0];
    }
    if (lane == 0) {
      const int s = q % kG4Stages;
      mbar_arrive_tx(&bars[w][s], (uint32_t)stage_bytes);
      g4_load(ring + s * stage_stride, &map, &bars[w][s], 0, r[0], r[1], r[2], r[3]);
      if (K > 2 && nbox > 1)
        g4_load(ring + s * stage_stride + 4 * box_bytes, &map, &bars[w][s], box_elems, r[0], r[1], r[2], r[3]);
    }
  };
  for (int q = 0; q < kG4Stages && q < nq; ++q) issue(q, 0);

  double acc[K][E];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int e = 0; e < E; ++e) acc[k][e] = 0.0;
  for (int q = 0; q < nq; ++q) {
    const int c = q >> 3;
    if (q > 0 && (q & 7) == 0) {  // consumption enters chunk c: shift the word window
      wc = wn;
      wn = wn2;
      wn2 = words(c + 2);
      sgn = __ballot_sync(0xffffffffu, (wc >> 31) != 0);
    }
    const int s = q % kG4Stages;
    mbar_wait(&bars[w][s], (uint32_t)((q / kG4Stages) & 1));
    const uint32_t st = ring_s + (uint32_t)(s * stage_stride);
    const uint32_t qs = sgn >> ((4 * q) & 31);  // bit j = sign of row 4q + j
    const int cnt = nrows - 4 * q < 4 ? nrows - 4 * q : 4;
    if (cnt == 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t m = ((qs >> j) & 1u) << 31;
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (lval[k]) g4_term<TIn, kW>(lds128(st + loff[k] + j * box_bytes), m, wgt, acc[k]);
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        const uint32_t m = ((qs >> j) & 1u) << 31;
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (lval[k]) g4_term<TIn, kW>(lds128(st + loff[k] + j * box_bytes), m, wgt, acc[k]);
      }
    }
    __syncwarp();  // every lane is done with stage s before it is refilled
    if (q + kG4Stages < nq) issue(q + kG4Stages, c);
  }
  bool bad = false;
  TOut *o = sa + bucket * ldsa;
  if (kPush) {  // the owner rank's receive slot (warp-uniform owner search, <= 8 ranks)
    const int64_t gb = push.b0 + bucket;
    int g = 0;
    while (g + 1 < push.nranks && gb >= push.bounds[g + 1]) ++g;
    o = (TOut *)push.peer[g] + ((int64_t)push.me * push.cap + (gb - push.bounds[g])) * push.ldr;
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int col = (k * 32 + lane) * E;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      bad |= !isfinite(acc[k][e]);
      if (col + e < d) o[col + e] = (TOut)acc[k][e];
    }
  }
  if (flag && __any_sync(0xffffffffu, bad)) {
    const bool real = sizeof(TIn) == 4 || g4_rescan<TIn>(a_raw, lda_bytes, beg, nrows, rows, row_bytes, lane);
    if (real && lane == 0) atomicOr(flag, 1);
  }
}

// out[r][c] = sum over src = 0 .. nslots-1 (in that order) of recv[src][r][c]:
// the owner's fixed-order reduction of the pushed partials (deterministic)
template <typename T>
__global__ void __launch_bounds__(256) slot_sum_kernel(const T *__restrict__ recv, int nslots, int64_t rows, int64_t d,
                                                       int64_t slot_stride, int64_t ldr, T *__restrict__ out,
                                                       int64_t ldo) {
  const int64_t total = rows * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d, c = i % d;
    double acc = (double)recv[r * ldr + c];
    for (int s = 1; s < nslots; ++s) acc += (double)recv[s * slot_stride + r * ldr + c];
    out[r * ldo + c] = (T)acc;
  }
}

// rows the gather4 kernels take: 512 B .. 2 KB, 16-byte multiples, as one box
// (<= 1 KB) or two equal boxes (each a 16-byte multiple); returns nbox or 0
inline int g4_boxes(int64_t d, int64_t esz) {
  const int64_t rb = d * esz;
  if (rb < 512 || rb > 2048 || rb % 16) return 0;
  if (rb <= 1024) return 1;
  return (d % 2 == 0 && (rb / 2) % 16 == 0) ? 2 : 0;
}

inline size_t dense_g4_smem(int row_bytes) {
  return (size_t)kG4Warps * kG4Stages * (((size_t)4 * row_bytes + 127) & ~(size_t)127);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// 2D map over A (n rows x d elements, row stride lda_bytes), box = one row's
// box_elems columns; gather4 fetches four such boxes at arbitrary row coordinates
inline bool make_row_map(CUtensorMap *map, const void *a, bool f64, int64_t n, int64_t d, int64_t lda_bytes,
                         int64_t box_elems) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)d, (cuuint64_t)n};
  const cuuint64_t gstride[1] = {(cuuint64_t)lda_bytes};
  const cuuint32_t box[2] = {(cuuint32_t)box_elems, 1};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(a),
            gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace
}  // namespace skt
