// csr_lane.cuh -- K4 "bucket-lane" kernel: S.A for canonical CSR A with
// narrow d (reference sketch.py:155-164, repeat + np.bincount).
//
// A warp owns BPW = 32 / CS consecutive buckets and keeps their SA rows as
// fp64 accumulators in shared memory; CS lanes serve each bucket.  The warp
// walks round by round: round q = rows q*RPB .. q*RPB+RPB-1 of each of its
// buckets (plan order = ascending row id inside a bucket).  The CS lanes of a
// bucket split a row's entries round-robin; a canonical row has distinct
// columns, so they never touch the same accumulator, and a __syncwarp orders
// successive rows -- per SA element the additions run in ascending row order
// from +0.0, bit-identical to the bincount.
//
// Rows are copied global->shared with cp.async (G lanes per row, first G
// nonzeros; longer rows finish with a direct read), kStages rounds ahead of the
// accumulation, descriptors (plan word, indptr pair) one further round ahead.
// With BPW buckets per warp the whole problem is resident at once (one wave)
// and every bucket's rows are spread uniformly over A, so all warps sweep A
// from low to high rows together: sectors shared by adjacent rows and DRAM
// pages are fetched once and hit in L2 for the other warps (ncu: DRAM traffic
// ~1.2x algorithmic vs ~1.9x for per-bucket warps).
#pragma once

#include "common.cuh"

namespace skt {
namespace {

constexpr int kLaneStages = 4;  // rounds of rows in flight per warp (power of two)
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
// bank spread), kStages x { desc [RPR] int4, idx [RPR][G+1], val [RPR][G+1] }
// with RPR = BPW * RPB rows per round.
template <typename IX, typename TV, int BPW, int RPB>
struct LaneSmem {
  static constexpr int RPR = BPW * RPB;
  static __host__ __device__ int dp(int d) { return d | 1; }
  static __host__ __device__ size_t acc_bytes(int d) {
    return ((size_t)BPW * dp(d) * sizeof(double) + 15) & ~(size_t)15;
  }
  static __host__ __device__ size_t stage_bytes() {
    const size_t raw = (size_t)RPR * 16 + (size_t)RPR * (kLaneG + 1) * (sizeof(IX) + sizeof(TV));
    return (raw + 15) & ~(size_t)15;
  }
  static __host__ __device__ size_t bytes(int d) { return acc_bytes(d) + kLaneStages * stage_bytes(); }
};

template <typename IP, typename IX, typename TV, typename TOut, int CS, int RPB>
__global__ void __launch_bounds__(32) csr_lane_kernel(const int64_t *__restrict__ pindptr,
                                                      const uint32_t *__restrict__ prow,
                                                      uint64_t t, const IP *__restrict__ aip,
                                                      const IX *__restrict__ aix,
                                                      const TV *__restrict__ av, int d,
                                                      TOut *__restrict__ sa, int64_t ldsa) {
  constexpr int BPW = 32 / CS;       // buckets per warp
  constexpr int RPR = BPW * RPB;     // rows per round (<= 32)
  constexpr int RPI = 32 / kLaneG;   // rows copied per cp.async iteration
  static_assert(RPR <= 32, "one descriptor lane per row of a round");
  using L = LaneSmem<IX, TV, BPW, RPB>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int dp = L::dp(d);
  double *acc = (double *)smem_raw;
  unsigned char *stg = smem_raw + L::acc_bytes(d);
  for (int i = lane; i < BPW * dp; i += 32) acc[i] = 0.0;

  const int mb = lane / CS, mq = lane % CS;  // accumulating role: bucket, lane in bucket
  const uint64_t b0 = (uint64_t)blockIdx.x * BPW;
  // descriptor role: lane j < RPR streams row (q * RPB + j % RPB) of bucket j / RPB
  const int db = lane / RPB, dsub = lane % RPB;
  const bool dlive = lane < RPR && b0 + db < t;
  const int64_t kb = dlive ? pindptr[b0 + db] : 0, ke = dlive ? pindptr[b0 + db + 1] : 0;
  const int64_t cnt = ke - kb;
  const int64_t rounds = ((int64_t)__reduce_max_sync(0xffffffffu, (unsigned)cnt) + RPB - 1) / RPB;
  double *my_acc = acc + mb * dp;

  auto stage_ptr = [&](int64_t q) { return stg + (size_t)((int)q & (kLaneStages - 1)) * L::stage_bytes(); };
  auto word = [&](int64_t q) -> uint32_t {
    const int64_t k = q * RPB + dsub;
    return (dlive && k < cnt) ? __ldg(prow + kb + k) : 0xffffffffu;
  };
  auto load_desc = [&](uint32_t wrd) -> int4 {
    if (wrd == 0xffffffffu) return make_int4(0, 0, 0, 0);
    const int64_t row = wrd & 0x7fffffffu;
    const int64_t rs = (int64_t)aip[row];
    const int len = (int)((int64_t)aip[row + 1] - rs);
    return make_int4((int)(uint32_t)rs, (int)(rs >> 32), len, (int)(wrd >> 31));
  };
  // publish round q's descriptors and cp.async the first G nonzeros of its rows
  auto stage = [&](int64_t q, int4 ds) {
    unsigned char *sp = stage_ptr(q);
    int4 *sdesc = (int4 *)sp;
    IX *sidx = (IX *)(sp + RPR * 16);
    TV *sval = (TV *)(sidx + RPR * (kLaneG + 1));
    if (lane < RPR) sdesc[lane] = ds;
    __syncwarp();
    const int g = lane / kLaneG, gl = lane % kLaneG;
    constexpr int kIt = (RPR + RPI - 1) / RPI;
    // read every descriptor first: the cp.async asm statements are compiler
    // memory barriers, so interleaving would serialise the shared loads
    int4 dr[kIt];
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
      const int r = i * RPI + g;
      dr[i] = r < RPR ? sdesc[r] : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
      const int r = i * RPI + g;
      if (gl < dr[i].z) {
        const int64_t rs = (int64_t)(uint32_t)dr[i].x | ((int64_t)dr[i].y << 32);
        cp_async_elem(sidx + r * (kLaneG + 1) + gl, aix + rs + gl);
        cp_async_elem(sval + r * (kLaneG + 1) + gl, av + rs + gl);
      }
    }
  };

  // ---- prologue: rounds 0 .. kStages-2 in flight; descriptors of the next
  // kDescAhead rounds in flight in a register pipeline (rotated each round)
  constexpr int kDescAhead = 4;
#pragma unroll
  for (int s = 0; s < kLaneStages - 1; ++s) {
    if (s < rounds) stage(s, load_desc(word(s)));
    cp_async_commit();
  }
  int4 dpipe[kDescAhead];
#pragma unroll
  for (int i = 0; i < kDescAhead; ++i) dpipe[i] = load_desc(word(kLaneStages - 1 + i));
  uint32_t w_next = word(kLaneStages - 1 + kDescAhead);

  for (int64_t q = 0; q < rounds; ++q) {
    const int64_t qn = q + kLaneStages - 1;
    if (qn < rounds) stage(qn, dpipe[0]);
    cp_async_commit();
#pragma unroll
    for (int i = 0; i + 1 < kDescAhead; ++i) dpipe[i] = dpipe[i + 1];
    dpipe[kDescAhead - 1] = load_desc(w_next);  // round qn + kDescAhead, in flight
    w_next = word(qn + kDescAhead + 1);
    cp_async_wait<kLaneStages - 1>();  // round q has landed
    __syncwarp();
    // ---- accumulate: bucket mb's rows of round q, in order
    const unsigned char *sp = stage_ptr(q);
    const IX *sidx0 = (const IX *)(sp + RPR * 16);
    const TV *sval0 = (const TV *)(sidx0 + RPR * (kLaneG + 1));
#pragma unroll
    for (int sub = 0; sub < RPB; ++sub) {
      const int r = mb * RPB + sub;
      const int4 ds = ((const int4 *)sp)[r];
      const int len = ds.z;
      const double sg = ds.w ? -1.0 : 1.0;
      const IX *sidx = sidx0 + r * (kLaneG + 1);
      const TV *sval = sval0 + r * (kLaneG + 1);
      // this lane's share of the staged entries: gather all, add, scatter back
      // (distinct columns inside a row: no load-after-store chain needed)
      constexpr int kE = (kLaneG + CS - 1) / CS;
      int col[kE];
      double upd[kE];
#pragma unroll
      for (int j = 0; j < kE; ++j) {
        const int e = mq + j * CS;
        const bool ok = e < kLaneG && e < len;
        col[j] = ok ? (int)sidx[e] : -1;
        upd[j] = ok ? sg * (double)sval[e] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kE; ++j)
        if (col[j] >= 0) upd[j] += my_acc[col[j]];
#pragma unroll
      for (int j = 0; j < kE; ++j)
        if (col[j] >= 0) my_acc[col[j]] = upd[j];
      if (len > kLaneG) {  // tail of a long row, straight from global memory
        const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
        for (int e = kLaneG + mq; e < len; e += CS)
          my_acc[(int)__ldg(aix + rs + e)] += sg * (double)__ldg(av + rs + e);
      }
      __syncwarp();  // orders successive rows of a bucket; frees the stage
    }
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
