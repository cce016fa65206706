// apply_csr_window.cu -- C ABI of the row-window CSR kernel (csr_window.cuh):
// the window plan (rows of every W-row window stably sorted by bucket) and
// skt_apply_csr_window, SA = S.A for canonical fp32 / int32-index CSR streamed
// once in row order (reference sketch.py:155-164, bit-identical).
#include <cstdlib>

#include "common.cuh"
#include "csr_cta.cuh"
#include "csr_window.cuh"

namespace skt {
namespace {

int win_sms() {
  static const int sms = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return v;
  }();
  return sms;
}

int win_env(const char *name, int dflt) {
  const char *e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// shared-memory bytes of one CTA for (t, d) on a grid of G CTAs; 0 = unsupported
size_t win_smem_bytes(uint64_t t, int64_t d, int G, int *bpw_out, int *dp_out) {
  if (G <= 0 || d < 1 || d > 256) return 0;
  const int dp = (int)((d + 3) & ~3LL);  // rows of the fp32 tile stay 16-byte multiples
  const int64_t bpw = ((int64_t)t + (int64_t)G * kWinAcc - 1) / ((int64_t)G * kWinAcc);
  if (bpw > 31) return 0;
  const size_t bytes = (size_t)kWinScat * kWinSpw * kWinStageBytes +
                       (size_t)kWinAcc * ((size_t)bpw * dp * 8 + (size_t)kWinTileRows * dp * 4);
  if (bytes > 226 * 1024) return 0;
  *bpw_out = (int)bpw;
  *dp_out = dp;
  return bytes;
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_csr_window_config(int64_t n, uint64_t t, int64_t d, int32_t *rows_per_window,
                                            int32_t *n_windows) {
  static const char *fn = "skt_csr_window_config";
  if (!rows_per_window || !n_windows || n < 0 || t < 1) return fail(SKT_EINVAL, fn, "bad arguments");
  *rows_per_window = 0;
  *n_windows = 0;
  const int G = win_sms();
  int bpw, dp;
  if (n < 1 || n >= (1LL << 31) || win_smem_bytes(t, d, G, &bpw, &dp) == 0) return SKT_OK;  // not supported
  int cpb = win_env("SKT_WIN_CPB", 32);
  if (cpb < kWinScat * kWinSpw || cpb % kWinScat != 0 || cpb > 32 * kWinScat) cpb = 32;
  const int64_t W = (int64_t)G * cpb * 32;
  *rows_per_window = (int32_t)W;
  *n_windows = (int32_t)((n + W - 1) / W);
  return SKT_OK;
}

extern "C" skt_status skt_plan_window_build(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                                            int32_t W, uint32_t *pos, int32_t *wpi, void *stream_) {
  static const char *fn = "skt_plan_window_build";
  if (!indptr || !rows || !pos || !wpi || t < 1 || t > (1ull << 31) || n < 1 || n >= (1LL << 31) || W < 32)
    return fail(SKT_EINVAL, fn, "bad arguments");
  cudaStream_t s = as_stream(stream_);
  const int64_t nwin = (n + W - 1) / W;
  SKT_CUDA_TRY(cudaMemsetAsync(wpi, 0, (size_t)nwin * (t + 1) * sizeof(int32_t), s), fn);
  const unsigned blocks = (unsigned)((t + 7) / 8);  // warp per bucket, 8 warps per CTA
  SKT_LAUNCH((win_plan_kernel<0>), blocks, 256, 0, s, indptr, rows, t, W, wpi, pos);
  SKT_LAUNCH(win_scan_kernel, (unsigned)nwin, 1024, 0, s, wpi, t);
  SKT_LAUNCH((win_plan_kernel<1>), blocks, 256, 0, s, indptr, rows, t, W, wpi, pos);
  return check_launch(fn);
}

extern "C" skt_status skt_apply_csr_window_workspace(int64_t n, int32_t W, size_t *bytes) {
  static const char *fn = "skt_apply_csr_window_workspace";
  if (!bytes || n < 1 || W < 32) return fail(SKT_EINVAL, fn, "bad arguments");
  const int64_t nwin = (n + W - 1) / W;
  int nbuf = win_env("SKT_WIN_NBUF", 3);
  if (nbuf < 2 || nbuf > 8) nbuf = 3;
  const size_t flags = ((size_t)2 * nwin * 4 + 255) & ~(size_t)255;
  *bytes = flags + (size_t)nbuf * (size_t)W * 128;
  return SKT_OK;
}

namespace {
template <typename IP, typename TOut>
skt_status win_launch(const WinParams &p, int chunks, int G, size_t smem, cudaStream_t s) {
  static const char *fn = "skt_apply_csr_window";
  auto k = chunks <= 1 ? csr_window_kernel<IP, TOut, 1>
                       : chunks <= 2 ? csr_window_kernel<IP, TOut, 2> : csr_window_kernel<IP, TOut, 4>;
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
  // The scatter and accumulate warps of different CTAs wait on each other, so all
  // G CTAs must be resident at once: a cooperative launch fails (instead of
  // hanging) when the device cannot hold them.
  WinParams pc = p;
  void *args[] = {(void *)&pc};
  cudaError_t e = cudaLaunchCooperativeKernel((const void *)k, dim3((unsigned)G), dim3(kWinThreads), args, smem, s);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(SKT_ENOTSUP, fn, std::string("the row-window kernel needs all its CTAs resident: ") + cudaGetErrorString(e));
  }
  return check_launch(fn);
}
}  // namespace

extern "C" skt_status skt_apply_csr_window(const uint32_t *pos, const int32_t *wpi, int32_t W, uint64_t t, int64_t n,
                                           const void *a_indptr, skt_itype indptr_type, const int32_t *a_indices,
                                           const float *a_vals, int64_t nnz, int64_t d, void *sa,
                                           skt_dtype sa_dtype, int64_t ldsa, void *ws, size_t ws_bytes,
                                           void *stream_) {
  static const char *fn = "skt_apply_csr_window";
  if (!pos || !wpi || !a_indptr || !sa || t < 1 || n < 1 || n >= (1LL << 31) || nnz < 0 || d < 1 || ldsa < d ||
      (indptr_type != SKT_I32 && indptr_type != SKT_I64) || (sa_dtype != SKT_F32 && sa_dtype != SKT_F64) ||
      (nnz > 0 && (!a_indices || !a_vals)))
    return fail(SKT_EINVAL, fn, "bad arguments");
  const int G = win_sms();
  int bpw = 0, dp = 0;
  const size_t smem = win_smem_bytes(t, d, G, &bpw, &dp);
  if (smem == 0) return fail(SKT_ENOTSUP, fn, "shape not supported by the row-window kernel");
  if (W < 32 || W % (G * 32 * kWinScat) != 0) return fail(SKT_EINVAL, fn, "W does not match this device");
  if (((uintptr_t)a_indices | (uintptr_t)a_vals | (uintptr_t)a_indptr | (uintptr_t)pos) & 15)
    return fail(SKT_ENOTSUP, fn, "CSR arrays must be 16-byte aligned");
  size_t need = 0;
  skt_apply_csr_window_workspace(n, W, &need);
  if (!ws || ws_bytes < need) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  cudaStream_t s = as_stream(stream_);
  const int64_t nwin = (n + W - 1) / W;
  const size_t flags = ((size_t)2 * nwin * 4 + 255) & ~(size_t)255;
  SKT_CUDA_TRY(cudaMemsetAsync(ws, 0, flags, s), fn);
  WinParams p;
  p.aip = a_indptr;
  p.aix = a_indices;
  p.av = a_vals;
  p.n = n;
  p.nnz = nnz;
  p.d = (int)d;
  p.dp = dp;
  p.t = t;
  p.pos = pos;
  p.wpi = wpi;
  p.scat_done = (uint32_t *)ws;
  p.acc_done = p.scat_done + nwin;
  p.slots = (unsigned char *)ws + flags;
  p.W = W;
  p.nwin = (int32_t)nwin;
  p.nbuf = (int32_t)((need - flags) / ((size_t)W * 128));
  p.cpb = W / (G * 32);
  p.bpw = bpw;
  p.sa = sa;
  p.ldsa = ldsa;
  const int chunks = (dp + 63) / 64;
  if (indptr_type == SKT_I32)
    return sa_dtype == SKT_F64 ? win_launch<int32_t, double>(p, chunks, G, smem, s)
                               : win_launch<int32_t, float>(p, chunks, G, smem, s);
  return sa_dtype == SKT_F64 ? win_launch<int64_t, double>(p, chunks, G, smem, s)
                             : win_launch<int64_t, float>(p, chunks, G, smem, s);
}


// ---- window gather kernel (csr_cta.cuh) -----------------------------------
namespace {
size_t cta_smem_bytes(uint64_t t, int64_t d, int G, int *bpc_out) {
  if (G <= 0 || d < 1 || d >= (1 << 20)) return 0;
  const int64_t bpc = ((int64_t)t + G - 1) / G;
  if (bpc > 16 * kCtaAcc) return 0;  // <= 8 buckets per accumulating half warp
  const size_t bytes = (size_t)kCtaBufs * kCtaRing * (128 + 4) + (size_t)bpc * d * 8;
  if (bytes > 226 * 1024) return 0;
  *bpc_out = (int)bpc;
  return bytes;
}
}  // namespace

extern "C" skt_status skt_csr_cta_config(int64_t n, uint64_t t, int64_t d, int32_t *rows_per_window,
                                         int32_t *n_windows) {
  static const char *fn = "skt_csr_cta_config";
  if (!rows_per_window || !n_windows || n < 0 || t < 1) return fail(SKT_EINVAL, fn, "bad arguments");
  *rows_per_window = 0;
  *n_windows = 0;
  const int G = win_sms();
  int bpc;
  if (n < 1 || n >= (1LL << 31) || t > (1ull << 31) || cta_smem_bytes(t, d, G, &bpc) == 0) return SKT_OK;
  int rpc = win_env("SKT_CTA_ROWS", 512);  // mean rows per CTA and window
  if (rpc < 32 || rpc > 1 << 16) rpc = 512;
  const int64_t W = (int64_t)G * rpc;
  *rows_per_window = (int32_t)W;
  *n_windows = (int32_t)((n + W - 1) / W);
  return SKT_OK;
}

extern "C" skt_status skt_plan_window_rows(const uint32_t *pos, int64_t n, int32_t W, uint32_t *wrows,
                                           void *stream_) {
  static const char *fn = "skt_plan_window_rows";
  if (!pos || !wrows || n < 1 || n >= (1LL << 31) || W < 32) return fail(SKT_EINVAL, fn, "bad arguments");
  SKT_LAUNCH(win_rows_kernel, (unsigned)((n + 255) / 256), 256, 0, as_stream(stream_), pos, n, W, wrows);
  return check_launch(fn);
}

extern "C" skt_status skt_apply_csr_cta(const uint32_t *wrows, const int32_t *wpi, int32_t W, uint64_t t, int64_t n,
                                        const void *a_indptr, skt_itype indptr_type, const int32_t *a_indices,
                                        const float *a_vals, int64_t nnz, int64_t d, void *sa, skt_dtype sa_dtype,
                                        int64_t ldsa, void *stream_) {
  static const char *fn = "skt_apply_csr_cta";
  if (!wrows || !wpi || !a_indptr || !sa || t < 1 || n < 1 || n >= (1LL << 31) || nnz < 0 || d < 1 || ldsa < d ||
      W < 32 || (indptr_type != SKT_I32 && indptr_type != SKT_I64) ||
      (sa_dtype != SKT_F32 && sa_dtype != SKT_F64) || (nnz > 0 && (!a_indices || !a_vals)))
    return fail(SKT_EINVAL, fn, "bad arguments");
  const int G = win_sms();
  int bpc = 0;
  const size_t smem = cta_smem_bytes(t, d, G, &bpc);
  if (smem == 0) return fail(SKT_ENOTSUP, fn, "shape not supported by the window gather kernel");
  CtaParams p;
  p.aip = a_indptr;
  p.aix = a_indices;
  p.av = a_vals;
  p.n = n;
  p.d = (int)d;
  p.dp = (int)d;
  p.t = t;
  p.wrows = wrows;
  p.wpi = wpi;
  p.W = W;
  p.nwin = (int32_t)((n + W - 1) / W);
  p.bpc = bpc;
  p.sa = sa;
  p.ldsa = ldsa;
  cudaStream_t s = as_stream(stream_);
  typedef void (*KFn)(const CtaParams);
  const KFn k = indptr_type == SKT_I32
                    ? (sa_dtype == SKT_F64 ? (KFn)csr_cta_kernel<int32_t, double> : (KFn)csr_cta_kernel<int32_t, float>)
                    : (sa_dtype == SKT_F64 ? (KFn)csr_cta_kernel<int64_t, double> : (KFn)csr_cta_kernel<int64_t, float>);
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
  SKT_LAUNCH(k, (unsigned)G, kCtaThreads, smem, s, p);
  return check_launch(fn);
}
