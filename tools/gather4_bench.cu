// gather4_bench.cu -- can TMA's tile::gather4 (sm_100: four rows at arbitrary
// row coordinates per instruction) stream K3's access pattern -- random 512 B
// rows of a 16.8M x 128 fp32 matrix, config 3 -- faster than the register
// gather?  A 1D bulk copy per row is TMA-issue bound (~46 SM cycles per copy,
// 3.8 TB/s on 512 B rows, profiles/README.md); gather4 moves 2 KB per issue.
//
// Each warp owns a contiguous run of "row slots" (like a bucket's plan); lane 0
// issues one gather4 per 4 rows into the warp's S-stage shared-memory ring
// (mbarrier per stage, complete_tx), all lanes consume (LDS.128 + fp64 adds,
// the K3 accumulate) and lane 0 refills the stage.  Rows come from a random
// uint32 index array read ahead (the plan words).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather4_bench tools/gather4_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{ .reg .pred P; W_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W_%=; }" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *map, uint64_t *bar, int col, int r0, int r1,
                                        int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

template <int S, bool kHash>
__global__ void __launch_bounds__(256) g4_kernel(const __grid_constant__ CUtensorMap map, const uint32_t *__restrict__ idx,
                                                 int64_t nslots, int per_warp, double *out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned char *ring = smem + (size_t)w * S * 2048;
  __shared__ __align__(8) uint64_t bars[8][S];
  const int64_t gw = (int64_t)blockIdx.x * nw + w;
  const int64_t s0 = gw * per_warp;
  const int64_t s1 = s0 + per_warp < nslots ? s0 + per_warp : nslots;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[w][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int nq = s0 < s1 ? (int)((s1 - s0 + 3) / 4) : 0;
  auto issue = [&](int q) {
    const int64_t b = s0 + 4 * (int64_t)q;
    int r[4];
    for (int j = 0; j < 4; ++j) {
      if (kHash) {  // random rows without an index load (TMA capability alone)
        uint64_t x = (uint64_t)(b + j) * 0x9E3779B97F4A7C15ULL;
        x ^= x >> 29;
        r[j] = (int)(x % (uint64_t)nslots);
      } else {
        r[j] = (int)__ldg(idx + (b + j < s1 ? b + j : s1 - 1));
      }
    }
    mbar_expect_tx(&bars[w][q % S], 2048);
    gather4(ring + (q % S) * 2048, &map, &bars[w][q % S], 0, r[0], r[1], r[2], r[3]);
  };
  if (lane == 0)
    for (int q = 0; q < S && q < nq; ++q) issue(q);
  double acc[4] = {0, 0, 0, 0};
  for (int q = 0; q < nq; ++q) {
    mbar_wait(&bars[w][q % S], (uint32_t)((q / S) & 1));
    const float4 *rows = reinterpret_cast<const float4 *>(ring + (q % S) * 2048);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 v = rows[j * 32 + lane];
      acc[0] += v.x;
      acc[1] += v.y;
      acc[2] += v.z;
      acc[3] += v.w;
    }
    __syncwarp();
    if (lane == 0 && q + S < nq) issue(q + S);
  }
  if (acc[0] + acc[1] + acc[2] + acc[3] == 1234.5) out[0] = acc[0];
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t n = 16777216, d = 128;
  float *a;
  uint32_t *idx;
  double *out;
  if (cudaMalloc(&a, n * d * 4) != cudaSuccess) return 1;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, n * d * 4);
  std::vector<uint32_t> h(n);
  uint64_t st = 7;
  for (int64_t i = 0; i < n; ++i) {
    st = st * 6364136223846793005ULL + 1442695040888963407ULL;
    h[i] = (uint32_t)((st >> 33) % n);
  }
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  const cuuint64_t gdim[2] = {(cuuint64_t)d, (cuuint64_t)n};
  const cuuint64_t gstride[1] = {(cuuint64_t)d * 4};
  const cuuint32_t box[2] = {(cuuint32_t)d, 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, gdim, gstride, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  const double bytes = (double)n * d * 4;
  auto run = [&](auto kern, int S, int warps, int ctas_per_sm, const char *name) {
    const int per_warp = 256;  // like a bucket (n / m = 256 rows)
    const int64_t nwarps = (n + per_warp - 1) / per_warp;
    const int blocks = (int)((nwarps + warps - 1) / warps);
    const size_t smem = (size_t)warps * S * 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (void)ctas_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, warps * 32, smem>>>(map, idx, n, per_warp, out);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) kern<<<blocks, warps * 32, smem>>>(map, idx, n, per_warp, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%s S=%d warps/CTA=%d smem/CTA=%zu KB: %.3f ms  %.0f GB/s  (%s)\n", name, S, warps, smem >> 10, ms,
           bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run(g4_kernel<2, true>, 2, 8, 0, "gather4 hash-rows");
  run(g4_kernel<4, true>, 4, 8, 0, "gather4 hash-rows");
  run(g4_kernel<4, true>, 4, 4, 0, "gather4 hash-rows");
  run(g4_kernel<8, true>, 8, 4, 0, "gather4 hash-rows");
  run(g4_kernel<8, true>, 8, 2, 0, "gather4 hash-rows");
  run(g4_kernel<4, false>, 4, 8, 0, "gather4 idx-rows");
  run(g4_kernel<8, false>, 8, 4, 0, "gather4 idx-rows");
  return 0;
}
