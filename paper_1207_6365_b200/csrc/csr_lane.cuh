// csr_lane.cuh -- K4 "bucket-lane" kernel: S.A for canonical CSR A with
// narrow d (reference sketch.py:155-164, repeat + np.bincount).
//
// A warp owns BPW = 32 / CS consecutive buckets; lane (b, q) owns columns
// [q*W, (q+1)*W) of bucket b's SA row (W = ceil(d / CS)) as fp64 accumulators
// in shared memory.  The warp walks round by round: round r = the r-th row of
// each of its buckets (plan order = ascending row id inside a bucket).  Every
// lane scans its bucket's row of the round and adds the entries that fall in
// its column range.  No two lanes ever share an accumulator, and each lane
// adds its bucket's rows in ascending order, so per SA element the additions
// run in ascending row order from +0.0 -- bit-identical to the bincount.
//
// Rows are copied global->shared with cp.async (G lanes per row, first G
// nonzeros; longer rows finish with a direct read), kStages rounds ahead of the
// accumulation, descriptors (plan word, indptr pair) one further round ahead.
// With BPW buckets per warp the whole problem is resident at once (one wave)
// and every bucket's rows are spread uniformly over A, so all warps sweep A
// from low to high rows together: sectors shared by adjacent rows and DRAM
// pages are fetched once and hit in L2 for the other warps.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

constexpr int kLaneStages = 4;  // rounds of rows in flight per warp
constexpr int kLaneG = 16;      // staged nonzeros per row (and lanes per row when copying)

__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T>
__device__ __forceinline__ void cp_async_elem(T *dst, const T *src) {
  if (sizeof(T) == 8)
    cp_async8(dst, src);
  else
    cp_async4(dst, src);
}

// Shared memory of one warp: acc [BPW][dp] doubles (dp = d | 1: odd stride,
// bank spread), kStages x { desc [BPW] int4, idx [BPW][G+1], val [BPW][G+1] }.
template <typename IX, typename TV, int BPW>
struct LaneSmem {
  static __host__ __device__ int dp(int d) { return d | 1; }
  static __host__ __device__ size_t acc_bytes(int d) { return (size_t)BPW * dp(d) * sizeof(double); }
  static __host__ __device__ size_t stage_bytes() {
    const size_t raw = (size_t)BPW * 16 + (size_t)BPW * (kLaneG + 1) * (sizeof(IX) + sizeof(TV));
    return (raw + 15) & ~(size_t)15;
  }
  static __host__ __device__ size_t bytes(int d) {
    return ((acc_bytes(d) + 15) & ~(size_t)15) + kLaneStages * stage_bytes();
  }
};

template <typename IP, typename IX, typename TV, typename TOut, int CS>
__global__ void __launch_bounds__(32) csr_lane_kernel(const int64_t *__restrict__ pindptr,
                                                      const uint32_t *__restrict__ prow,
                                                      uint64_t t, const IP *__restrict__ aip,
                                                      const IX *__restrict__ aix,
                                                      const TV *__restrict__ av, int d,
                                                      TOut *__restrict__ sa, int64_t ldsa) {
  constexpr int BPW = 32 / CS;    // buckets per warp
  constexpr int RPI = 32 / kLaneG;  // rows copied per cp.async iteration
  using L = LaneSmem<IX, TV, BPW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int dp = L::dp(d);
  double *acc = (double *)smem_raw;
  unsigned char *stg = smem_raw + ((L::acc_bytes(d) + 15) & ~(size_t)15);
  for (int i = lane; i < BPW * dp; i += 32) acc[i] = 0.0;

  // this lane's bucket / column range (bucket-major: lanes b*CS .. b*CS+CS-1)
  const int mb = lane / CS, mq = lane % CS;
  const int W = (d + CS - 1) / CS;
  const int c_lo = mq * W, c_hi = min(d, c_lo + W);
  const uint64_t b0 = (uint64_t)blockIdx.x * BPW;
  // descriptor streams: lane j < BPW walks bucket b0 + j's plan slice
  const bool dlive = lane < BPW && b0 + lane < t;
  const int64_t kb = dlive ? pindptr[b0 + lane] : 0, ke = dlive ? pindptr[b0 + lane + 1] : 0;
  const int64_t cnt = ke - kb;
  const int64_t rounds = (int64_t)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
  double *my_acc = acc + mb * dp;

  auto stage_ptr = [&](int64_t q) { return stg + (q % kLaneStages) * L::stage_bytes(); };
  auto load_desc = [&](int64_t q, uint32_t wrd) -> int4 {
    if (!dlive || q >= cnt) return make_int4(0, 0, 0, 0);
    const int64_t row = wrd & 0x7fffffffu;
    const int64_t rs = (int64_t)aip[row];
    const int len = (int)((int64_t)aip[row + 1] - rs);
    return make_int4((int)(uint32_t)rs, (int)(rs >> 32), len, (int)(wrd >> 31));
  };
  auto word = [&](int64_t q) -> uint32_t { return (dlive && q < cnt) ? __ldg(prow + kb + q) : 0u; };
  // publish round q's descriptors and cp.async the first G nonzeros of its rows
  auto stage = [&](int64_t q, int4 ds) {
    unsigned char *sp = stage_ptr(q);
    int4 *sdesc = (int4 *)sp;
    IX *sidx = (IX *)(sp + BPW * 16);
    TV *sval = (TV *)(sidx + BPW * (kLaneG + 1));
    if (lane < BPW) sdesc[lane] = ds;
    __syncwarp();
    const int g = lane / kLaneG, gl = lane % kLaneG;
#pragma unroll
    for (int i = 0; i < (BPW + RPI - 1) / RPI; ++i) {
      const int r = i * RPI + g;
      if (r < BPW) {
        const int4 dr = sdesc[r];
        if (gl < dr.z) {
          const int64_t rs = (int64_t)(uint32_t)dr.x | ((int64_t)dr.y << 32);
          cp_async_elem(sidx + r * (kLaneG + 1) + gl, aix + rs + gl);
          cp_async_elem(sval + r * (kLaneG + 1) + gl, av + rs + gl);
        }
      }
    }
  };

  // ---- prologue: rounds 0 .. kStages-2 in flight, descriptor of the next one loaded
#pragma unroll
  for (int s = 0; s < kLaneStages - 1; ++s) {
    if (s < rounds) stage(s, load_desc(s, word(s)));
    cp_async_commit();
  }
  int4 d_next = load_desc(kLaneStages - 1, word(kLaneStages - 1));
  uint32_t w_next = word(kLaneStages);

  for (int64_t q = 0; q < rounds; ++q) {
    const int64_t qn = q + kLaneStages - 1;
    if (qn < rounds) stage(qn, d_next);
    cp_async_commit();
    d_next = load_desc(qn + 1, w_next);  // in flight during this round
    w_next = word(qn + 2);
    cp_async_wait<kLaneStages - 1>();  // round q has landed
    __syncwarp();
    // ---- accumulate: lane (b, q) adds the entries of bucket b's row in its column range
    const unsigned char *sp = stage_ptr(q);
    const int4 ds = ((const int4 *)sp)[mb];
    const int len = ds.z;
    const double sg = ds.w ? -1.0 : 1.0;
    const IX *sidx = (const IX *)(sp + BPW * 16) + mb * (kLaneG + 1);
    const TV *sval = (const TV *)((const IX *)(sp + BPW * 16) + BPW * (kLaneG + 1)) + mb * (kLaneG + 1);
    const int lh = len < kLaneG ? len : kLaneG;
    for (int e = 0; e < lh; ++e) {
      const int c = (int)sidx[e];
      if (c >= c_lo && c < c_hi) my_acc[c] += sg * (double)sval[e];
    }
    if (len > kLaneG) {  // tail of a long row, straight from global memory
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      for (int e = kLaneG; e < len; ++e) {
        const int c = (int)__ldg(aix + rs + e);
        if (c >= c_lo && c < c_hi) my_acc[c] += sg * (double)__ldg(av + rs + e);
      }
    }
    __syncwarp();  // stage q is rewritten kStages - 1 rounds later
  }
  __syncwarp();
  for (int r = 0; r < BPW; ++r) {
    const uint64_t br = b0 + r;
    if (br >= t) break;
    TOut *o = sa + br * ldsa;
    for (int c = lane; c < d; c += 32) o[c] = (TOut)acc[r * dp + c];
  }
}

}  // namespace
}  // namespace skt
