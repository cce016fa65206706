// csr_sweep.cuh -- K4 "bucket-lane" kernel: S.A for canonical CSR A with
// narrow d (reference sketch.py:155-164, repeat + np.bincount).
//
// A warp owns 32 consecutive buckets and LANE l owns bucket b0 + l: it keeps
// that bucket's SA row as d fp64 accumulators in shared memory and adds the
// bucket's rows one after the other in plan (= ascending row) order.  Lanes
// never share an accumulator, so there are no conflicts and no serialisation;
// per SA element the additions run in ascending row order from +0.0 --
// bit-identical to the reference's bincount.
//
// Round q of a warp = the q-th row of each of its 32 buckets.  The rows'
// nonzeros are copied global -> shared with cp.async, G lanes per row
// (coalesced), kStages rounds ahead of the accumulation, with the row
// descriptors (plan word, indptr pair) prefetched one further round ahead.
// Every bucket's rows are spread uniformly over A and taken in ascending
// order, so all warps sweep A from low to high rows together: sectors shared by
// adjacent rows and DRAM pages are fetched once and hit in L2 for the others.
// Nonzeros of a row beyond the first G are read by the owning lane directly.
#pragma once

#include "common.cuh"

namespace skt {
namespace {

constexpr int kLaneStages = 8;  // rounds in flight per warp (~1 us of DRAM latency)

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

// Shared memory of one warp: acc [32][dp] doubles (dp odd: bank spread), then
// kStages x { idx [32][G+1], val [32][G+1] } (+1 pad: conflict-free per-lane
// reads of a row).
template <typename IX, typename TV, int G>
struct LaneSmem {
  static __host__ __device__ int dp(int d) { return d | 1; }
  static __host__ __device__ size_t acc_bytes(int d) { return (size_t)32 * dp(d) * sizeof(double); }
  static __host__ __device__ size_t stage_bytes() {
    return (size_t)32 * (G + 1) * (sizeof(IX) + sizeof(TV));
  }
  static __host__ __device__ size_t bytes(int d) {
    return acc_bytes(d) + kLaneStages * stage_bytes() + kLaneStages * 32 * sizeof(int4);
  }
};

template <typename IP, typename IX, typename TV, typename TOut, int G>
__global__ void __launch_bounds__(32) csr_lane_kernel(const int64_t *__restrict__ pindptr,
                                                      const uint32_t *__restrict__ prow,
                                                      uint64_t t, const IP *__restrict__ aip,
                                                      const IX *__restrict__ aix,
                                                      const TV *__restrict__ av, int d,
                                                      TOut *__restrict__ sa, int64_t ldsa) {
  using L = LaneSmem<IX, TV, G>;
  constexpr int S = 32 / G;  // rows copied per iteration
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int dp = L::dp(d);
  double *acc = (double *)smem_raw;
  unsigned char *stg = smem_raw + L::acc_bytes(d);
  int4 *sdesc = (int4 *)(stg + kLaneStages * L::stage_bytes());  // [kStages][32]
  for (int i = lane; i < 32 * dp; i += 32) acc[i] = 0.0;

  const uint64_t b = (uint64_t)blockIdx.x * 32 + lane;
  const bool live = b < t;
  const int64_t kb = live ? pindptr[b] : 0, ke = live ? pindptr[b + 1] : 0;
  const int64_t cnt = ke - kb;
  const int64_t rounds = (int64_t)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
  const int g = lane / G, gl = lane % G;
  double *my_acc = acc + lane * dp;

  // descriptor of this lane's row of round q: (row start lo, hi, length, neg)
  auto load_desc = [&](int64_t q, uint32_t wrd) -> int4 {
    if (q >= cnt) return make_int4(0, 0, 0, 0);
    const int64_t row = wrd & 0x7fffffffu;
    const int64_t rs = (int64_t)aip[row];
    const int len = (int)((int64_t)aip[row + 1] - rs);
    return make_int4((int)(uint32_t)rs, (int)(rs >> 32), len, (int)(wrd >> 31));
  };
  auto word = [&](int64_t q) -> uint32_t { return q < cnt ? __ldg(prow + kb + q) : 0u; };
  // publish the descriptor of round q and cp.async the first G nonzeros of
  // every lane's row of round q into stage q % kStages
  auto stage = [&](int64_t q, int4 ds) {
    const int sq = (int)(q % kLaneStages);
    sdesc[sq * 32 + lane] = ds;
    __syncwarp();
    IX *sidx = (IX *)(stg + sq * L::stage_bytes());
    TV *sval = (TV *)(sidx + 32 * (G + 1));
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int r = i * S + g;
      const int4 dr = sdesc[sq * 32 + r];
      if (gl < dr.z) {
        const int64_t rs = (int64_t)(uint32_t)dr.x | ((int64_t)dr.y << 32);
        cp_async_elem(sidx + r * (G + 1) + gl, aix + rs + gl);
        cp_async_elem(sval + r * (G + 1) + gl, av + rs + gl);
      }
    }
  };

  // ---- prologue: stage rounds 0 .. kStages-2; descriptor of the next round in flight
#pragma unroll
  for (int s = 0; s < kLaneStages - 1; ++s) {
    if (s < rounds) stage(s, load_desc(s, word(s)));
    cp_async_commit();
  }
  int4 d_next = load_desc(kLaneStages - 1, word(kLaneStages - 1));
  uint32_t w_next = word(kLaneStages);

  for (int64_t q = 0; q < rounds; ++q) {
    // issue round q + kStages - 1 (its descriptor arrived during the last round)
    const int64_t qn = q + kLaneStages - 1;
    if (qn < rounds) stage(qn, d_next);
    cp_async_commit();
    d_next = load_desc(qn + 1, w_next);  // in flight during this round
    w_next = word(qn + 2);
    cp_async_wait<kLaneStages - 1>();  // round q has landed
    __syncwarp();
    // ---- accumulate: lane l adds its own row of round q into its bucket
    const int sq = (int)(q % kLaneStages);
    const int4 ds = sdesc[sq * 32 + lane];
    const int len = ds.z;
    const double sg = ds.w ? -1.0 : 1.0;
    const IX *sidx = (const IX *)(stg + sq * L::stage_bytes()) + lane * (G + 1);
    const TV *sval = (const TV *)(stg + sq * L::stage_bytes() + 32 * (G + 1) * sizeof(IX)) + lane * (G + 1);
    // columns inside a canonical row are distinct: gather all G accumulators,
    // add, scatter back (no false load-after-store chain between elements)
    int col[G];
    double upd[G];
#pragma unroll
    for (int e = 0; e < G; ++e) {
      col[e] = e < len ? (int)sidx[e] : -1;
      upd[e] = e < len ? sg * (double)sval[e] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < G; ++e)
      if (col[e] >= 0) upd[e] += my_acc[col[e]];
#pragma unroll
    for (int e = 0; e < G; ++e)
      if (col[e] >= 0) my_acc[col[e]] = upd[e];
    if (len > G) {  // tail of a long row, straight from global memory
      const int64_t rs = (int64_t)(uint32_t)ds.x | ((int64_t)ds.y << 32);
      for (int e = G; e < len; ++e) my_acc[(int)__ldg(aix + rs + e)] += sg * (double)__ldg(av + rs + e);
    }
    __syncwarp();  // stage sq and sdesc[sq] are rewritten kStages - 1 rounds later
  }
  __syncwarp();
  // ---- write the 32 SA rows (coalesced along d)
  for (int r = 0; r < 32; ++r) {
    const uint64_t br = (uint64_t)blockIdx.x * 32 + r;
    if (br >= t) break;
    TOut *o = sa + br * ldsa;
    for (int c = lane; c < d; c += 32) o[c] = (TOut)acc[r * dp + c];
  }
}

}  // namespace
}  // namespace skt
