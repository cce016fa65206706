// srht.cu -- subsampled randomized Hadamard transform of a tall fp64 matrix
// (reference SrhtOperator.apply, sketch.py:241-297: zero-pad to n_pad = 2^L
// rows, flip row signs, unnormalised Walsh-Hadamard transform along the rows
// (_fwht, sketch.py:241-252), keep t sampled rows scaled by sqrt(n_pad/t) /
// sqrt(n_pad)).  Used on the sparse-embedding sketch S.A by
// approx_leverage_scores (leverage.py:81-82) when t1 exceeds the SRHT rows.
//
// Bit-exact with the reference: _fwht's stage h replaces rows (i, i + h) of
// every 2h-block by (x_i + x_{i+h}, x_i - x_{i+h}) in fp64; the passes below
// perform exactly those butterflies, stage after stage, only several stages
// per trip through HBM.  A pass takes groups of 2^k rows spaced h0 apart
// (stages h0 .. h0 2^(k-1)) into shared memory, 16 columns at a time, runs k
// stages there and writes the group back; ceil(L / 9) passes cover all L
// stages.  Sign flip and padding are fused into the load, sampling and
// scaling into a final gather.
#include "common.cuh"

namespace skt {
namespace {

constexpr int kSrhtThreads = 256;
constexpr int kSrhtCols = 16;   // column slice per block
constexpr int kSrhtMaxK = 9;    // stages per pass: 512 rows x 16 cols x 8 B = 64 KB

__global__ void srht_load_kernel(const double *__restrict__ a, int64_t n, int64_t d, int64_t lda,
                                 const int8_t *__restrict__ sign, int64_t n_pad, double *__restrict__ ws) {
  const int64_t total = n_pad * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d, c = e - i * d;
    ws[e] = i < n ? a[i * lda + c] * (double)sign[i] : 0.0;
  }
}

__global__ void __launch_bounds__(kSrhtThreads) fwht_pass_kernel(double *__restrict__ ws, int64_t n_pad, int64_t d,
                                                                 int64_t h0, int k) {
  extern __shared__ double tile[];  // [2^k][kSrhtCols]
  const int64_t rows = (int64_t)1 << k;
  const int64_t gi = blockIdx.x;  // group: base = (gi / h0) * h0 * 2^k + gi % h0
  const int64_t c0 = (int64_t)blockIdx.y * kSrhtCols;
  const int cw = (int)(d - c0 < kSrhtCols ? d - c0 : kSrhtCols);
  const int64_t base = (gi / h0) * h0 * rows + gi % h0;
  for (int64_t e = threadIdx.x; e < rows * kSrhtCols; e += blockDim.x) {
    const int64_t j = e / kSrhtCols;
    const int c = (int)(e % kSrhtCols);
    if (c < cw) tile[e] = ws[(base + j * h0) * d + c0 + c];
  }
  __syncthreads();
  for (int s = 0; s < k; ++s) {
    const int64_t hs = (int64_t)1 << s;
    for (int64_t e = threadIdx.x; e < (rows >> 1) * kSrhtCols; e += blockDim.x) {
      const int64_t p = e / kSrhtCols;
      const int c = (int)(e % kSrhtCols);
      const int64_t j = (p / hs) * (hs << 1) + (p % hs);
      const double x = tile[j * kSrhtCols + c], y = tile[(j + hs) * kSrhtCols + c];
      tile[j * kSrhtCols + c] = x + y;
      tile[(j + hs) * kSrhtCols + c] = x - y;
    }
    __syncthreads();
  }
  for (int64_t e = threadIdx.x; e < rows * kSrhtCols; e += blockDim.x) {
    const int64_t j = e / kSrhtCols;
    const int c = (int)(e % kSrhtCols);
    if (c < cw) ws[(base + j * h0) * d + c0 + c] = tile[e];
  }
}

__global__ void srht_gather_kernel(const double *__restrict__ ws, int64_t d, const uint32_t *__restrict__ rows,
                                   int64_t t, double scale, double *__restrict__ out, int64_t ldo) {
  const int64_t total = t * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d, c = e - r * d;
    out[r * ldo + c] = scale * ws[(int64_t)rows[r] * d + c];
  }
}

inline int64_t pad_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_srht_workspace(int64_t n, int64_t d, size_t *bytes) {
  if (n < 1 || d < 0 || !bytes) return fail(SKT_EINVAL, "skt_srht_workspace", "bad arguments");
  *bytes = (size_t)pad_pow2(n) * (size_t)d * sizeof(double);
  return SKT_OK;
}

extern "C" skt_status skt_srht_apply(const double *a, int64_t n, int64_t d, int64_t lda, const int8_t *sign,
                                     const uint32_t *rows, int64_t t, double scale, double *out, int64_t ldo,
                                     void *ws, size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_srht_apply";
  if (n < 1 || d < 0 || t < 0 || lda < d || ldo < d || (n > 0 && d > 0 && (!a || !sign)) ||
      (t > 0 && d > 0 && (!rows || !out)))
    return fail(SKT_EINVAL, fn, "bad arguments");
  const int64_t n_pad = pad_pow2(n);
  if (d == 0 || t == 0) return SKT_OK;
  if (!ws || ws_bytes < (size_t)n_pad * (size_t)d * sizeof(double)) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  cudaStream_t st = as_stream(stream_);
  double *w = (double *)ws;
  const int64_t lb = std::max<int64_t>(1, std::min<int64_t>((n_pad * d + 255) / 256, (int64_t)kNumSMs * 16));
  SKT_LAUNCH(srht_load_kernel, (unsigned)lb, 256, 0, st, a, n, d, lda, sign, n_pad, w);
  int L = 0;
  while (((int64_t)1 << L) < n_pad) ++L;
  const int64_t cslices = (d + kSrhtCols - 1) / kSrhtCols;
  SKT_CUDA_TRY(cudaFuncSetAttribute(fwht_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(((size_t)1 << kSrhtMaxK) * kSrhtCols * sizeof(double))), fn);
  for (int done = 0; done < L;) {
    const int k = std::min(kSrhtMaxK, L - done);
    const int64_t h0 = (int64_t)1 << done;
    const int64_t groups = n_pad >> k;
    if (groups > 0x7fffffffLL || cslices > 65535) return fail(SKT_ENOTSUP, fn, "matrix too large");
    const size_t smem = ((size_t)1 << k) * kSrhtCols * sizeof(double);
    SKT_LAUNCH(fwht_pass_kernel, dim3((unsigned)groups, (unsigned)cslices), kSrhtThreads, smem, st, w, n_pad, d, h0,
               k);
    done += k;
  }
  const int64_t gb = std::max<int64_t>(1, std::min<int64_t>((t * d + 255) / 256, (int64_t)kNumSMs * 16));
  SKT_LAUNCH(srht_gather_kernel, (unsigned)gb, 256, 0, st, w, d, rows, t, scale, out, ldo);
  return check_launch(fn);
}
