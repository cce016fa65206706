// gather_bench.cu -- ceiling of random segment gathers from HBM (the access
// pattern of CSR S.A: every row's index / value segment sits at an arbitrary
// 4-byte-aligned offset).  For segment sizes of 16..512 bytes, random starts
// over an 8 GB buffer, 8 warps x U independent loads in flight per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_bench tools/gather_bench.cu
// Prints useful GB/s (bytes of the segments / time) per segment size and the
// 64-byte-aligned variant.
#include <cstdint>
#include <cstdio>
#include <utility>
#include <vector>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__global__ void offsets_kernel(int64_t *off, int64_t nseg, int64_t nfloats, int seg_floats, int align_floats) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = (int64_t)(mix((uint64_t)s) % (uint64_t)(nfloats - seg_floats));
    off[s] = o - o % align_floats;
  }
}

template <int kSegFloats, int kU>
__global__ void __launch_bounds__(256) gather_kernel(const float *__restrict__ p, const int64_t *__restrict__ offs,
                                                     int64_t nseg, float *out) {
  constexpr int kPerWarp = 32 / kSegFloats > 0 ? 32 / kSegFloats : 1;  // segments per warp instruction
  constexpr int kLanesPerSeg = kSegFloats < 32 ? kSegFloats : 32;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int sub = lane / kLanesPerSeg, sl = lane % kLanesPerSeg;
  float acc = 0.f;
  for (int64_t base = warp * kPerWarp * kU; base < nseg; base += nwarps * kPerWarp * kU) {
    float v[kU][(kSegFloats + 31) / 32];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t s = base + (int64_t)u * kPerWarp + sub;
      const int64_t off = s < nseg ? __ldg(offs + s) : 0;
#pragma unroll
      for (int j = 0; j < (kSegFloats + 31) / 32; ++j) v[u][j] = s < nseg ? __ldg(p + off + sl + 32 * j) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int j = 0; j < (kSegFloats + 31) / 32; ++j) acc += v[u][j];
  }
  if (acc == 12345.678f) out[0] = acc;
}

// CSR S.A's access pattern without its arithmetic: rows visited in a random
// order (a permutation, like the bucket-ordered plan), per row the indptr
// pair, then the row's index and value segments (G lanes per row, 32/G rows
// per instruction, the batch's 32 rows' loads all issued before use, the next
// batch's indptr pairs in flight) -- the ceiling for configs 2 / 4.
template <int G, typename TV>
__global__ void __launch_bounds__(128) csr_gather_kernel(const uint32_t *__restrict__ perm, int64_t n,
                                                         const int *__restrict__ ip, const int *__restrict__ ix,
                                                         const TV *__restrict__ v, float *out) {
  constexpr int S = 32 / G;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  int64_t b = warp * 32;
  int rs = 0, len = 0;
  if (b + lane < n) {
    const uint32_t r = perm[b + lane];
    rs = ip[r];
    len = ip[r + 1] - rs;
  }
  for (; b < n; b += nwarps * 32) {
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

// name, rows, nonzeros per row (1% of rows dense_len when dense_len > 0), value type
template <int G, typename TV>
void run_csr(const char *name, int64_t n, int per, int dense_len) {
  std::vector<int> ip(n + 1);
  ip[0] = 0;
  uint64_t st = 1;
  for (int64_t r = 0; r < n; ++r) {
    st = st * 6364136223846793005ULL + 1442695040888963407ULL;
    ip[r + 1] = ip[r] + ((dense_len > 0 && (st >> 33) % 100 == 0) ? dense_len : per);
  }
  const int64_t nnz = ip[n];
  std::vector<uint32_t> perm(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
  for (int64_t i = n - 1; i > 0; --i) {
    st = st * 6364136223846793005ULL + 1442695040888963407ULL;
    const int64_t j = (int64_t)((st >> 33) % (uint64_t)(i + 1));
    std::swap(perm[i], perm[j]);
  }
  int *dip, *dix;
  TV *dv;
  float *out;
  uint32_t *dperm;
  cudaMalloc(&dip, (n + 1) * 4);
  cudaMalloc(&dix, nnz * 4);
  cudaMalloc(&dv, nnz * sizeof(TV));
  cudaMalloc(&dperm, n * 4);
  cudaMalloc(&out, 4);
  cudaMemset(dix, 0, nnz * 4);
  cudaMemset(dv, 0, nnz * sizeof(TV));
  cudaMemcpy(dip, ip.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  // L2 flush buffer for inputs that fit in L2
  char *flush;
  cudaMalloc(&flush, 512 << 20);
  // windows: 1 = random permutation of all rows (the bucket-ordered plan);
  // P > 1 = rows grouped into P contiguous row windows visited in order,
  // random inside a window (a phased sweep); 0 = sequential rows
  for (int windows : {1, 4, 8, 16, 32, 64, 0}) {
    const int ordered = windows == 0;
    if (windows == 1) {
      cudaMemcpy(dperm, perm.data(), n * 4, cudaMemcpyHostToDevice);
    } else {
      std::vector<uint32_t> id(n);
      for (int64_t i = 0; i < n; ++i) id[i] = (uint32_t)i;
      if (windows > 1) {
        for (int wi = 0; wi < windows; ++wi) {
          const int64_t lo = n * wi / windows, hi = n * (wi + 1) / windows;
          for (int64_t i = hi - 1; i > lo; --i) {
            st = st * 6364136223846793005ULL + 1442695040888963407ULL;
            const int64_t j = lo + (int64_t)((st >> 33) % (uint64_t)(i - lo + 1));
            std::swap(id[i], id[j]);
          }
        }
      }
      cudaMemcpy(dperm, id.data(), n * 4, cudaMemcpyHostToDevice);
    }
    for (int blocks : {148 * 6, 148 * 12, 148 * 16}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      csr_gather_kernel<G, TV><<<blocks, 128>>>(dperm, n, dip, dix, dv, out);
      float total = 0.f;
      for (int i = 0; i < 5; ++i) {
        cudaMemsetAsync(flush, i, 512 << 20);
        cudaEventRecord(a);
        csr_gather_kernel<G, TV><<<blocks, 128>>>(dperm, n, dip, dix, dv, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        total += ms;
      }
      const float ms = total / 5;
      const double alg = nnz * (4.0 + sizeof(TV)) + (n + 1) * 4.0;
      printf("csr gather (%s shape, %s rows, windows %d, %d CTAs, L2 flushed): %.4f ms, %.0f GB/s algorithmic (%s)\n", name,
             ordered ? "sequential" : "random", windows, blocks, ms, alg / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaFree(dip);
  cudaFree(dix);
  cudaFree(dv);
  cudaFree(dperm);
  cudaFree(out);
  cudaFree(flush);
}

template <int kSeg, int kU>
void run(const float *p, int64_t nfloats, float *out, int align) {
  const int64_t nseg = (int64_t)1 << 26;
  static int64_t *offs = nullptr;
  if (!offs) cudaMalloc(&offs, nseg * 8);
  offsets_kernel<<<148 * 8, 256>>>(offs, nseg, nfloats, kSeg, align);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 8;
  gather_kernel<kSeg, kU><<<blocks, 256>>>(p, offs, nseg, out);
  cudaEventRecord(a);
  for (int i = 0; i < 3; ++i) gather_kernel<kSeg, kU><<<blocks, 256>>>(p, offs, nseg, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 3;
  printf("seg %4d B  align %3d B  U=%d: %7.1f GB/s useful  (%.3f ms, %s)\n", kSeg * 4, align * 4, kU,
         nseg * kSeg * 4.0 / (ms * 1e-3) / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char **argv) {
  run_csr<16, float>("config-4", 4194304, 16, 64);
  run_csr<8, double>("config-2", 1000000, 5, 0);
  if (argc > 1) return 0;  // CSR patterns only
  const int64_t nfloats = (int64_t)2 << 30;  // 8 GB
  float *p, *out;
  cudaMalloc(&p, nfloats * 4);
  cudaMalloc(&out, 4);
  cudaMemset(p, 0, nfloats * 4);
  run<4, 8>(p, nfloats, out, 1);
  run<8, 8>(p, nfloats, out, 1);
  run<16, 8>(p, nfloats, out, 1);
  run<16, 16>(p, nfloats, out, 1);
  run<16, 8>(p, nfloats, out, 16);
  run<32, 8>(p, nfloats, out, 1);
  run<32, 8>(p, nfloats, out, 32);
  run<64, 8>(p, nfloats, out, 1);
  run<128, 4>(p, nfloats, out, 1);
  return 0;
}
