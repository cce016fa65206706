// membench.cu -- read-bandwidth ceiling probes for the K3 design (tools only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libmembench.so tools/membench.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ float4 ld_nc(const float4 *p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// grid-stride streaming read of n float4, U loads in flight per thread
template <int U>
__global__ void __launch_bounds__(256) read_kernel(const float4 *__restrict__ p, int64_t n, float *out) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n; i += stride) {
    float4 v = ld_nc(p + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 123.456f) out[0] = acc;
}

// bulk-copy (TMA 1D) streaming read: one elected lane per warp issues
// cp.async.bulk of CHUNK bytes into a per-warp ring of STAGES buffers
template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(128) bulk_kernel(const char *__restrict__ p, int64_t nbytes, float *out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  unsigned char *ring = smem + (size_t)w * STAGES * CHUNK;
  __shared__ __align__(8) uint64_t bars[4 * 16];
  uint64_t *bar = bars + w * 16;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t nchunks = nbytes / CHUNK;
  const int64_t gw = (int64_t)blockIdx.x * nw + w, ngw = (int64_t)gridDim.x * nw;
  float acc = 0.f;
  // prologue
  int64_t c_issue = gw;
  for (int s = 0; s < STAGES; ++s, c_issue += ngw) {
    if (lane == 0 && c_issue < nchunks) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + s);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(ring + s * CHUNK)),
                   "l"(p + c_issue * CHUNK), "r"(CHUNK), "r"(b)
                   : "memory");
    }
  }
  int s = 0;
  uint32_t phase = 0;
  for (int64_t c = gw; c < nchunks; c += ngw) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + s);
    asm volatile(
        "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(b),
        "r"(phase)
        : "memory");
    const float4 *q = (const float4 *)(ring + s * CHUNK);
    for (int k = lane; k < CHUNK / 16; k += 32) {
      float4 v = q[k];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    if (lane == 0 && c_issue < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(ring + s * CHUNK)),
                   "l"(p + c_issue * CHUNK), "r"(CHUNK), "r"(b)
                   : "memory");
    }
    c_issue += ngw;
    if (++s == STAGES) {
      s = 0;
      phase ^= 1;
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

// per-warp streams: warp w reads its own contiguous chunk of `chunk` bytes in
// 512-byte rows, U rows in flight (the access pattern of K3 on an identity plan)
template <int U>
__global__ void __launch_bounds__(256) stream_kernel(const float4 *__restrict__ p, int64_t n_float4,
                                                     int64_t chunk_f4, float *out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t base = warp * chunk_f4;
  float acc = 0.f;
  if (base < n_float4) {
    for (int64_t r = 0; r < chunk_f4; r += 32 * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_nc(p + base + r + u * 32 + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

extern "C" int mb_stream(const void *p, int64_t n_float4, int64_t chunk_f4, int unroll, float *out,
                         void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t warps = n_float4 / chunk_f4;
  const int64_t blocks = (warps * 32 + 255) / 256;
  switch (unroll) {
    case 4: stream_kernel<4><<<blocks, 256, 0, st>>>((const float4 *)p, n_float4, chunk_f4, out); break;
    case 8: stream_kernel<8><<<blocks, 256, 0, st>>>((const float4 *)p, n_float4, chunk_f4, out); break;
    default: return 1;
  }
  return (int)cudaGetLastError();
}

extern "C" int mb_read(const void *p, int64_t n_float4, int unroll, int blocks, float *out, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (unroll) {
    case 4: read_kernel<4><<<blocks, 256, 0, st>>>((const float4 *)p, n_float4, out); break;
    case 8: read_kernel<8><<<blocks, 256, 0, st>>>((const float4 *)p, n_float4, out); break;
    case 16: read_kernel<16><<<blocks, 256, 0, st>>>((const float4 *)p, n_float4, out); break;
    default: return 1;
  }
  return (int)cudaGetLastError();
}

extern "C" int mb_bulk(const void *p, int64_t nbytes, int blocks, float *out, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  constexpr int STAGES = 8, CHUNK = 4096;
  const size_t smem = 4 * STAGES * CHUNK;
  cudaFuncSetAttribute(bulk_kernel<STAGES, CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bulk_kernel<STAGES, CHUNK><<<blocks, 128, smem, st>>>((const char *)p, nbytes, out);
  return (int)cudaGetLastError();
}
