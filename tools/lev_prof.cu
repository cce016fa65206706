// lev_prof.cu -- phase timing of the K5 v2 kernel (lev_tc2.cuh) on a
// config-4-shaped CSR (16 nnz/row + 1% dense rows, d = 64, k = 32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSKT_T2_PROF \
//        -I include tools/lev_prof.cu -o tools/lev_prof && tools/lev_prof
// Prints kernel times (v1, v2) and the per-tile cycles of each v2 phase
// (thread 0 of every CTA, producer lane 0), averaged over all tiles.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <vector>

#include "../paper_1207_6365_b200/csrc/lev_tc2.cuh"

using namespace skt;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

// tcgen05 MMA chain latency, nothing else running on the SM: mode 0 = 24 x
// (N=32) unmerged 3xTF32 chain, mode 1 = 8 x (N=64) + 8 x (N=32) merged chain
__global__ void mma_chain_kernel(int mode, int reps, long long *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  const int dk = 64, k = 32;
  for (int i = threadIdx.x; i < (4 * 128 * dk * 4 + 2 * k * dk * 4) / 16; i += blockDim.x) ((uint4 *)sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&tb)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(tc_smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t a_bytes = 128 * dk * 4;
    const uint32_t ah = tc_smem_u32(sm), al = ah + a_bytes, pb = ah + 4 * a_bytes;
    const uint32_t lbo_a = 128 * 16, lbo_p = 2 * k * 16, plo = pb + (k / 8) * 128;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int ks = 0; ks < dk / 8; ++ks) {
        const uint32_t oa = ks * 2 * lbo_a, op = ks * 2 * lbo_p;
        if (mode >= 2) {  // A in the 128B-swizzled K-major layout (16 KB per 32-element atom column)
          const uint32_t sa = (uint32_t)(ks / 4) * 16384 + (uint32_t)(ks % 4) * 32;
          const uint64_t sw = (uint64_t)2 << 61;
          // mode 3: even / odd K-steps into two independent accumulators (cols 0 / 64)
          const uint32_t dt = tb + (mode == 3 ? (uint32_t)(ks & 1) * 64 : 0u);
          const uint32_t acc = mode == 3 ? (ks > 1) : (ks > 0);
          tc_mma(dt, tc_desc(ah + sa, 16, 1024) | sw, tc_desc(pb + op, lbo_p, 128), tc_idesc(64), acc);
          tc_mma(dt, tc_desc(al + sa, 16, 1024) | sw, tc_desc(pb + op, lbo_p, 128), tc_idesc(32), 1);
          continue;
        }
        if (mode == 1) {
          tc_mma(tb, tc_desc(ah + oa, lbo_a, 128), tc_desc(pb + op, lbo_p, 128), tc_idesc(64), ks > 0);
        } else {
          tc_mma(tb, tc_desc(ah + oa, lbo_a, 128), tc_desc(pb + op, lbo_p, 128), tc_idesc(32), ks > 0);
          tc_mma(tb, tc_desc(ah + oa, lbo_a, 128), tc_desc(plo + op, lbo_p, 128), tc_idesc(32), 1);
        }
        tc_mma(tb, tc_desc(al + oa, lbo_a, 128), tc_desc(pb + op, lbo_p, 128), tc_idesc(32), 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tc_smem_u32(&bar)) : "memory");
      asm volatile("{ .reg .pred P; W_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W_%=; }" ::"r"(tc_smem_u32(&bar)), "r"(r & 1) : "memory");
    }
    out[mode] = (clock64() - t0) / reps;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(128));
}

int main(int argc, char **argv) {
  {
    long long *dout, hout[4];
    cudaMalloc(&dout, 32);
    const int sm_bytes = 4 * 128 * 64 * 4 + 2 * 32 * 64 * 4;
    cudaFuncSetAttribute(mma_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes);
    for (int mode = 0; mode < 4; ++mode) mma_chain_kernel<<<1, 128, sm_bytes>>>(mode, 200, dout);
    cudaMemcpy(hout, dout, 32, cudaMemcpyDeviceToHost);
    printf("MMA chain (quiet SM): unmerged 24 MMAs %lld cycles, merged 16 MMAs %lld cycles, merged SW128 A %lld, 2 accumulators %lld (%s)\n", hout[0], hout[1], hout[2], hout[3],
           cudaGetErrorString(cudaGetLastError()));
  }
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 22);
  const int d = 64, k = 32, per = 16;
  uint64_t x = 88172645463325252ull;
  auto rnd = [&]() {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
  };
  std::vector<int> ip(n + 1);
  std::vector<int> ix;
  std::vector<float> v;
  ix.reserve(n * 17);
  v.reserve(n * 17);
  ip[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    uint64_t mask = 0;
    if (rnd() % 100 == 0) {
      mask = ~0ull;
    } else {
      int c = 0;
      while (c < per) {
        const int j = (int)(rnd() % d);
        if (!(mask >> j & 1)) {
          mask |= 1ull << j;
          ++c;
        }
      }
    }
    for (int j = 0; j < d; ++j)
      if (mask >> j & 1) {
        ix.push_back(j);
        v.push_back((float)((int64_t)(rnd() % 2001) - 1000) / 1000.f);
      }
    ip[r + 1] = (int)ix.size();
  }
  const int64_t nnz = (int64_t)ix.size();
  std::vector<double> probe((size_t)d * k);
  for (auto &p : probe) p = (double)((int64_t)(rnd() % 2001) - 1000) / 5000.0;
  int *dip, *dix;
  float *dv;
  double *dp, *ds1, *ds2;
  CK(cudaMalloc(&dip, (n + 1) * 4));
  CK(cudaMalloc(&dix, nnz * 4));
  CK(cudaMalloc(&dv, nnz * 4));
  CK(cudaMalloc(&dp, probe.size() * 8));
  CK(cudaMalloc(&ds1, n * 8));
  CK(cudaMalloc(&ds2, n * 8));
  CK(cudaMemcpy(dip, ip.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dix, ix.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, v.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dp, probe.data(), probe.size() * 8, cudaMemcpyHostToDevice));
  const int dk = 64;  // v1: d rounded up to whole 32-element swizzle atoms
  const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;
  // v1
  const size_t s1 = lev_tc_smem(dk, k);
  auto k1 = lev_tc_kernel<int, int, double, true>;  // k = 32: merged probe operand
  CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1));
  const int64_t b1 = std::min<int64_t>(ntiles, 148 * 2);
  for (int i = 0; i < 3; ++i) k1<<<b1, kTcThreads, s1>>>(n, d, dk, dip, dix, dv, dp, k, ds1);
  CK(cudaEventRecord(e0));
  for (int i = 0; i < 10; ++i) k1<<<b1, kTcThreads, s1>>>(n, d, dk, dip, dix, dv, dp, k, ds1);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double alg = (double)nnz * 8 + (n + 1) * 4.0 + n * 8.0;
  printf("v1: %.4f ms  %.0f GB/s\n", ms / 10, alg / (ms / 10 * 1e-3) / 1e9);
  // v2
  const T2Layout L = lev_tc2_layout(d, k, 4);
  printf("v2 layout: nst=%d cap=%d smem=%zu\n", L.nst, L.cap, L.smem);
  auto k2 = lev_tc2_kernel<int, int, double>;
  CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
  const int64_t b2 = std::min<int64_t>(ntiles, 148);
  for (int i = 0; i < 3; ++i) k2<<<b2, kT2Threads, L.smem>>>(n, d, dip, dix, dv, dp, k, ds2, L);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  unsigned long long zero[16] = {0};
  CK(cudaMemcpyToSymbol(g_t2_prof, zero, sizeof(zero)));
  CK(cudaEventRecord(e0));
  for (int i = 0; i < 10; ++i) k2<<<b2, kT2Threads, L.smem>>>(n, d, dip, dix, dv, dp, k, ds2, L);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("v2: %.4f ms  %.0f GB/s (nnz %lld)\n", ms / 10, alg / (ms / 10 * 1e-3) / 1e9, (long long)nnz);
  unsigned long long prof[16];
  CK(cudaMemcpyFromSymbol(prof, g_t2_prof, sizeof(prof)));
  const char *cn[8] = {"wait_full", "densify", "release", "mma_wait", "epi/clear", "bar2", "-", "loop"};
  const char *pn[3] = {"prod_misc", "prod_wait_empty", "prod_issue"};
  const double tiles = (double)ntiles * 10;
  for (int i = 0; i < 8; ++i) printf("  consumer %-16s %8.1f cycles/tile\n", cn[i], prof[i] / tiles);
  for (int i = 0; i < 3; ++i) printf("  producer %-16s %8.1f cycles/tile\n", pn[i], prof[8 + i] / tiles);
  std::vector<double> h1(n), h2(n);
  CK(cudaMemcpy(h1.data(), ds1, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), ds2, n * 8, cudaMemcpyDeviceToHost));
  double worst = 0;
  for (int64_t i = 0; i < n; ++i)
    if (h1[i] > 0) worst = std::max(worst, std::abs(h1[i] - h2[i]) / h1[i]);
  printf("v1 vs v2 max relative difference: %.3g\n", worst);
  return 0;
}
