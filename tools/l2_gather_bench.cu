// l2_gather_bench.cu -- can an L2 streaming prefetch turn config 4's
// bucket-ordered CSR gather into L2 hits?  Access pattern of csr_tile without
// its arithmetic (tools/gather_bench.cu csr_gather_kernel): rows in a random
// order inside contiguous row windows, windows in order; per row the indptr
// pair, then the index and value segments.  Variants:
//   * warm: a 262,144-row copy of the pattern (36 MB) that stays in L2
//     (no flush): the L2-hit gather rate;
//   * full size, L2 flushed, with and without a bulk prefetch
//     (cp.async.bulk.prefetch.L2) of window w + AHEAD issued by every warp
//     (its 1/nwarps slice) when it enters window w.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_gather_bench tools/l2_gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <utility>
#include <vector>

__device__ __forceinline__ void prefetch_l2(const void *p, uint64_t bytes) {
  // 16-byte-aligned interior only
  uint64_t a = ((uint64_t)p + 15) & ~15ull;
  uint64_t e = ((uint64_t)p + bytes) & ~15ull;
  while (e > a) {
    uint32_t sz = (uint32_t)((e - a) > (1u << 20) ? (1u << 20) : (e - a));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
    a += sz;
  }
}

template <int G, typename TV>
__global__ void __launch_bounds__(128) csr_gather_kernel(const uint32_t *__restrict__ perm, int64_t n,
                                                         const int *__restrict__ ip, const int *__restrict__ ix,
                                                         const TV *__restrict__ v, float *out, int64_t W,
                                                         int ahead) {
  constexpr int S = 32 / G;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  int64_t b = warp * 32;
  int rs = 0, len = 0;
  int64_t wlast = -1;
  if (b + lane < n) {
    const uint32_t r = perm[b + lane];
    rs = ip[r];
    len = ip[r + 1] - rs;
  }
  for (; b < n; b += nwarps * 32) {
    if (ahead > 0 && lane == 0) {
      const int64_t wc = b / W;
      if (wc != wlast) {
        for (int64_t wp = (wlast < 0 ? wc : wlast + 1); wp <= wc; ++wp) {
          const int64_t tw = wp + ahead;
          const int64_t r0 = tw * W, r1 = min(n, (tw + 1) * W);
          if (r0 < n) {
            const int64_t q0 = r0 + (r1 - r0) * warp / nwarps, q1 = r0 + (r1 - r0) * (warp + 1) / nwarps;
            const int e0 = ip[q0], e1 = ip[q1];
            prefetch_l2(ix + e0, (uint64_t)(e1 - e0) * 4);
            prefetch_l2(v + e0, (uint64_t)(e1 - e0) * sizeof(TV));
            prefetch_l2(ip + q0, (uint64_t)(q1 - q0 + 1) * 4);
          }
        }
        wlast = wc;
      }
    }
    int rs_n = 0, len_n = 0;
    const int64_t bn = b + nwarps * 32;
    if (bn + lane < n) {
      const uint32_t r = perm[bn + lane];
      rs_n = ip[r];
      len_n = ip[r + 1] - rs_n;
    }
    int c[G];
    TV x[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int row = S * i + lane / G;
      const int s = __shfl_sync(0xffffffffu, rs, row), l = __shfl_sync(0xffffffffu, len, row);
      c[i] = 0;
      x[i] = (TV)0;
      if ((lane % G) < l) {
        c[i] = __ldg(ix + s + (lane % G));
        x[i] = __ldg(v + s + (lane % G));
      }
    }
    const uint32_t longm = __ballot_sync(0xffffffffu, len > G);
    for (uint32_t m = longm; m; m &= m - 1) {
      const int row = __ffs(m) - 1;
      const int s = __shfl_sync(0xffffffffu, rs, row), l = __shfl_sync(0xffffffffu, len, row);
      for (int q = G + lane; q < l; q += 32) acc += (float)__ldg(ix + s + q) + (float)__ldg(v + s + q);
    }
#pragma unroll
    for (int i = 0; i < G; ++i) acc += (float)c[i] + (float)x[i];
    rs = rs_n;
    len = len_n;
  }
  if (acc == 12345.678f) out[0] = acc;
}

// plain streaming read of the same arrays (the HBM floor for this data)
__global__ void stream_kernel(const int4 *__restrict__ p, int64_t n16, float *out) {
  int acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    int4 x = __ldg(p + i);
    acc += x.x ^ x.y ^ x.z ^ x.w;
  }
  if (acc == 123456789) out[0] = (float)acc;
}

static uint64_t st = 1;
static uint64_t nxt() {
  st = st * 6364136223846793005ULL + 1442695040888963407ULL;
  return st >> 33;
}

template <int G, typename TV>
void run(const char *name, int64_t n, int per, int dense_len, bool flush_each) {
  std::vector<int> ip(n + 1);
  ip[0] = 0;
  for (int64_t r = 0; r < n; ++r) ip[r + 1] = ip[r] + ((dense_len > 0 && nxt() % 100 == 0) ? dense_len : per);
  const int64_t nnz = ip[n];
  int *dip, *dix;
  TV *dv;
  float *out;
  uint32_t *dperm;
  char *flush;
  cudaMalloc(&dip, (n + 1) * 4);
  cudaMalloc(&dix, nnz * 4);
  cudaMalloc(&dv, nnz * sizeof(TV));
  cudaMalloc(&dperm, n * 4);
  cudaMalloc(&out, 4);
  cudaMalloc(&flush, 512 << 20);
  cudaMemset(dix, 0, nnz * 4);
  cudaMemset(dv, 0, nnz * sizeof(TV));
  cudaMemcpy(dip, ip.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  const double alg = nnz * (4.0 + sizeof(TV)) + (n + 1) * 4.0;
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int i = 0; i < 4; ++i) {
      cudaMemsetAsync(flush, i, 512 << 20);
      cudaEventRecord(a);
      stream_kernel<<<148 * 16, 256>>>((const int4 *)dv, nnz * (int64_t)sizeof(TV) / 16, out);
      stream_kernel<<<148 * 16, 256>>>((const int4 *)dix, nnz / 4, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i) tot += ms;
    }
    printf("%s: n %lld nnz %lld, streaming read of idx+val: %.4f ms\n", name, (long long)n, (long long)nnz, tot / 3);
  }
  for (int64_t W : {(int64_t)0, (int64_t)32768, (int64_t)131072, (int64_t)262144, (int64_t)524288}) {
    std::vector<uint32_t> id(n);
    for (int64_t i = 0; i < n; ++i) id[i] = (uint32_t)i;
    const int64_t win = W == 0 ? n : W;
    for (int64_t lo = 0; lo < n; lo += win) {
      const int64_t hi = std::min(n, lo + win);
      for (int64_t i = hi - 1; i > lo; --i) std::swap(id[i], id[lo + (int64_t)(nxt() % (uint64_t)(i - lo + 1))]);
    }
    cudaMemcpy(dperm, id.data(), n * 4, cudaMemcpyHostToDevice);
    for (int ahead : {0, 1, 2, 3}) {
      if (W == 0 && ahead) continue;
      for (int blocks : {148 * 6, 148 * 12}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int64_t Wk = W == 0 ? n : W;
        csr_gather_kernel<G, TV><<<blocks, 128>>>(dperm, n, dip, dix, dv, out, Wk, ahead);
        float total = 0.f;
        for (int i = 0; i < 5; ++i) {
          if (flush_each) cudaMemsetAsync(flush, i, 512 << 20);
          cudaEventRecord(a);
          csr_gather_kernel<G, TV><<<blocks, 128>>>(dperm, n, dip, dix, dv, out, Wk, ahead);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          total += ms;
        }
        const float ms = total / 5;
        printf("%s: window %7lld rows ahead %d, %4d CTAs, %s: %.4f ms, %.0f GB/s algorithmic, x%.1f per full c4 (%s)\n",
               name, (long long)W, ahead, blocks, flush_each ? "L2 flushed" : "warm", ms, alg / (ms * 1e-3) / 1e9,
               4194304.0 / n, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  cudaFree(dip);
  cudaFree(dix);
  cudaFree(dv);
  cudaFree(dperm);
  cudaFree(out);
  cudaFree(flush);
}

int main() {
  run<16, float>("c4-small (L2 resident)", 262144, 16, 64, false);
  run<16, float>("c4-full", 4194304, 16, 64, true);
  run<8, double>("c2-full", 1000000, 5, 0, true);
  return 0;
}
