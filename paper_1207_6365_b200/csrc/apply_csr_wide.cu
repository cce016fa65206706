// apply_csr_wide.cu -- K4 for CSR A too wide for on-chip accumulators of
// whole SA rows: the fine-block path (csr_fine.cuh, default), the 16384-column
// partition path (csr_partition.cuh, SKT_CSR_WIDE=partition) and the
// column-block kernel (csr_colblock.cuh, SKT_CSR_WIDE=colblock) behind
// skt_apply_csr_wide (sketch.py:155-164, BASELINE config 5).
#include <cstdlib>

#include "common.cuh"
#include "csr_colblock.cuh"
#include "csr_fine.cuh"
#include "csr_partition.cuh"

namespace skt {
namespace {

// ---- wide CSR: launch ----------------------------------------------------
inline int num_sms() {
  static const int n = [] {
    int dev = 0, v = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// SKT_CSR_WIDE=colblock selects the single-kernel column-block path (16 MB of
// workspace for config 5 instead of ~nnz x 6 B), SKT_CSR_WIDE=partition the
// 16384-column partition path (A/B)
inline int wide_kernel() {
  static const int k = [] {
    const char *e = getenv("SKT_CSR_WIDE");
    return (e && e[0] == 'c') ? 1 : (e && e[0] == 'p') ? 2 : 3;  // 3 = fine blocks (default)
  }();
  return k;
}
// the path taken for width d: fine blocks, else the partition, else colblock
inline int wide_path(int64_t d) {
  const int k = wide_kernel();
  if (k == 3 && fine_nblk(d) <= kFbMaxBlocks) return 3;
  if (k >= 2 && (d + kCbCols - 1) / kCbCols <= kPtMaxBlocks) return 2;
  return 1;
}
inline int colblock_nblk(int64_t d) { return (int)std::max<int64_t>(1, (d + kCbCols - 1) / kCbCols); }

struct PartLayout {
  size_t np, pstart, pnz, pbase, reg, key, val, total;
  int64_t maxpieces;
};
inline PartLayout part_layout(int64_t n, uint64_t t, int nblk, int64_t nnz, size_t vsize) {
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  PartLayout L;
  L.maxpieces = n / kPtPiece + (int64_t)t + 1;  // sum over buckets of ceil(rows / piece)
  L.np = 0;
  L.pstart = L.np + up((size_t)t * 8);
  L.pnz = L.pstart + up(((size_t)t + 1) * 8);
  L.pbase = L.pnz + up((size_t)L.maxpieces * 8);
  L.reg = L.pbase + up(((size_t)L.maxpieces + 1) * 8);
  L.key = L.reg + up((size_t)L.maxpieces * (nblk + 1) * 8);
  L.val = L.key + up((size_t)std::max<int64_t>(1, nnz) * 2);
  L.total = L.val + up((size_t)std::max<int64_t>(1, nnz) * vsize);
  return L;
}

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch_partition(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                            const void *aix, const void *av, int64_t nnz, int64_t d, void *sa, int64_t ldsa,
                            void *ws, cudaStream_t stream) {
  static const char *fn = "skt_apply_csr_wide";
  const int nblk = colblock_nblk(d);
  const PartLayout L = part_layout(n, t, nblk, nnz, sizeof(TV));
  char *w = (char *)ws;
  int64_t *np = (int64_t *)(w + L.np), *pstart = (int64_t *)(w + L.pstart), *pnz = (int64_t *)(w + L.pnz);
  int64_t *pbase = (int64_t *)(w + L.pbase), *reg = (int64_t *)(w + L.reg);
  uint16_t *wkey = (uint16_t *)(w + L.key);
  TV *wval = (TV *)(w + L.val);
  SKT_LAUNCH(csr_part_npieces_kernel, (unsigned)((t + 255) / 256), 256, 0, stream, pindptr, t, np);
  SKT_LAUNCH(csr_part_scan_kernel, 1, 1024, 0, stream, np, (int64_t)t, pstart);
  SKT_LAUNCH((csr_part_piece_nnz_kernel<IP>), (unsigned)((L.maxpieces * 32 + 255) / 256), 256, 0, stream, pindptr,
             prow, t, pstart, (const IP *)aip, pnz);
  // pieces past the real count were not written: the scan reads pstart[t] of them
  SKT_LAUNCH(csr_part_scan_kernel, 1, 1024, 0, stream, pnz, L.maxpieces, pbase);
  auto ks = csr_part_scatter_kernel<IP, IX, TV>;
  const int smem_s = (int)part_scatter_smem(nblk);
  SKT_CUDA_TRY(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s), fn);
  SKT_LAUNCH(ks, (unsigned)L.maxpieces, kPtThreads, smem_s, stream, pindptr, prow, t, pstart, pbase, nblk,
             (const IP *)aip, (const IX *)aix, (const TV *)av, reg, wkey, wval);
  auto ka = csr_part_accum_kernel<TV, TOut>;
  const int smem_a = (int)sizeof(PtSmem);
  SKT_CUDA_TRY(cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a), fn);
  SKT_LAUNCH(ka, (unsigned)(t * nblk), kPaThreads, smem_a, stream, nblk, d, pstart, reg, wkey, wval, (TOut *)sa, ldsa);
  return check_launch(fn);
}

struct FineLayout {
  size_t np, pstart, pnz, pbase, reg, key, val, total;
  int64_t maxpieces, slots;
};
inline FineLayout fine_layout(int64_t n, uint64_t t, int nblk, int64_t nnz, size_t vsize) {
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  FineLayout L;
  L.maxpieces = n / kFpRows + (int64_t)t + 1;  // sum over buckets of ceil(rows / piece)
  L.slots = std::max<int64_t>(1, nnz) + 8 * L.maxpieces;  // every piece padded to a multiple of 8
  L.np = 0;
  L.pstart = L.np + up((size_t)t * 8);
  L.pnz = L.pstart + up(((size_t)t + 1) * 8);
  L.pbase = L.pnz + up((size_t)L.maxpieces * 8);
  L.reg = L.pbase + up(((size_t)L.maxpieces + 1) * 8);
  L.key = L.reg + up((size_t)L.maxpieces * (nblk + 1) * 8);
  L.val = L.key + up((size_t)L.slots * 2);
  L.total = L.val + up((size_t)L.slots * vsize);
  return L;
}

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch_fine(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                       const void *aix, const void *av, int64_t nnz, int64_t d, void *sa, int64_t ldsa, void *ws,
                       cudaStream_t stream) {
  static const char *fn = "skt_apply_csr_wide";
  const int nblk = fine_nblk(d);
  const FineLayout L = fine_layout(n, t, nblk, nnz, sizeof(TV));
  char *w = (char *)ws;
  int64_t *np = (int64_t *)(w + L.np), *pstart = (int64_t *)(w + L.pstart), *pnz = (int64_t *)(w + L.pnz);
  int64_t *pbase = (int64_t *)(w + L.pbase), *reg = (int64_t *)(w + L.reg);
  uint16_t *wkey = (uint16_t *)(w + L.key);
  TV *wval = (TV *)(w + L.val);
  SKT_LAUNCH(csr_fine_npieces_kernel, (unsigned)((t + 255) / 256), 256, 0, stream, pindptr, t, np);
  SKT_LAUNCH(csr_part_scan_kernel, 1, 1024, 0, stream, np, (int64_t)t, pstart);
  SKT_LAUNCH((csr_fine_piece_nnz_kernel<IP>), (unsigned)((L.maxpieces * 32 + 255) / 256), 256, 0, stream, pindptr,
             prow, t, pstart, (const IP *)aip, pnz);
  // pieces past the real count were not written: the scan reads pstart[t] of them
  SKT_LAUNCH(csr_part_scan_kernel, 1, 1024, 0, stream, pnz, L.maxpieces, pbase);
  auto ks = csr_fine_scatter_kernel<IP, IX, TV>;
  const int smem_s = (int)fine_scatter_smem(nblk, sizeof(TV));
  SKT_CUDA_TRY(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s), fn);
  SKT_LAUNCH(ks, (unsigned)L.maxpieces, kFsThreads, smem_s, stream, pindptr, prow, t, pstart, pbase, nblk,
             (const IP *)aip, (const IX *)aix, (const TV *)av, reg, wkey, wval);
  auto ka = csr_fine_accum_kernel<TV, TOut>;
  const int smem_a = kFaWarps * kFaWarpBytes;
  SKT_CUDA_TRY(cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a), fn);
  const int64_t units = (int64_t)t * nblk;
  SKT_LAUNCH(ka, (unsigned)((units + kFaWarps - 1) / kFaWarps), kFaWarps * 32, smem_a, stream, nblk, d, t, pstart, reg,
             wkey, wval, (TOut *)sa, ldsa);
  return check_launch(fn);
}

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch_colblock(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                           const void *aix, const void *av, int64_t d, void *sa, int64_t ldsa, int32_t *bnd,
                           cudaStream_t stream) {
  static const char *fn = "skt_apply_csr_wide";
  const int nblk = colblock_nblk(d);
  if (nblk > 1 && n > 0) {
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)num_sms() * 16);
    SKT_LAUNCH((csr_colblock_bounds_kernel<IP, IX>), (unsigned)blocks, 256, 0, stream, n, nblk, (const IP *)aip,
               (const IX *)aix, bnd);
    SKT_CUDA_TRY(cudaGetLastError(), fn);
  }
  auto k = csr_colblock_kernel<IP, IX, TV, TOut>;
  const int smem = (int)sizeof(CbSmem);
  SKT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), fn);
  SKT_LAUNCH(k, (unsigned)(t * nblk), kCbThreads, smem, stream, pindptr, prow, nblk, d, (const IP *)aip,
             (const IX *)aix, (const TV *)av, bnd, (TOut *)sa, ldsa);
  return check_launch(fn);
}

template <typename IP, typename IX, typename TV, typename TOut>
skt_status launch_wide(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                       const void *aix, const void *av, int64_t nnz, int64_t d, void *sa, int64_t ldsa, void *ws,
                       cudaStream_t stream) {
  const int path = wide_path(d);
  if (path == 3)
    return launch_fine<IP, IX, TV, TOut>(pindptr, prow, t, n, aip, aix, av, nnz, d, sa, ldsa, ws, stream);
  if (path == 2)
    return launch_partition<IP, IX, TV, TOut>(pindptr, prow, t, n, aip, aix, av, nnz, d, sa, ldsa, ws, stream);
  return launch_colblock<IP, IX, TV, TOut>(pindptr, prow, t, n, aip, aix, av, d, sa, ldsa, (int32_t *)ws, stream);
}

template <typename IP, typename IX>
skt_status wide_by_vals(const int64_t *pindptr, const uint32_t *prow, uint64_t t, int64_t n, const void *aip,
                            const void *aix, const void *av, skt_dtype vt, int64_t nnz, int64_t d, void *sa,
                            skt_dtype ot, int64_t ldsa, int32_t *cursor, cudaStream_t s) {  // cursor: the workspace
  if (vt == SKT_F32)
    return ot == SKT_F64 ? launch_wide<IP, IX, float, double>(pindptr, prow, t, n, aip, aix, av, nnz, d, sa, ldsa, cursor, s)
                         : launch_wide<IP, IX, float, float>(pindptr, prow, t, n, aip, aix, av, nnz, d, sa, ldsa, cursor, s);
  return ot == SKT_F64 ? launch_wide<IP, IX, double, double>(pindptr, prow, t, n, aip, aix, av, nnz, d, sa, ldsa, cursor, s)
                       : launch_wide<IP, IX, double, float>(pindptr, prow, t, n, aip, aix, av, nnz, d, sa, ldsa, cursor, s);
}

}  // namespace
}  // namespace skt

using namespace skt;

extern "C" skt_status skt_apply_csr_wide_workspace(int64_t n, uint64_t t, int64_t d, int64_t nnz, skt_dtype val_dtype,
                                                   size_t *bytes) {
  if (!bytes || n < 0 || t < 1 || d < 0 || nnz < 0 || (val_dtype != SKT_F32 && val_dtype != SKT_F64))
    return fail(SKT_EINVAL, "skt_apply_csr_wide_workspace", "bad arguments");
  const size_t block = (size_t)std::max<int64_t>(1, n) * (size_t)std::max(1, colblock_nblk(d) - 1) * sizeof(int32_t);
  const size_t vsize = val_dtype == SKT_F32 ? 4 : 8;
  const int path = wide_path(d);
  const size_t part = path == 3   ? fine_layout(n, t, fine_nblk(d), nnz, vsize).total
                      : path == 2 ? part_layout(n, t, colblock_nblk(d), nnz, vsize).total
                                  : (size_t)0;
  *bytes = std::max(block, part);
  return SKT_OK;
}

extern "C" skt_status skt_apply_csr_wide(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                                         const void *a_indptr, skt_itype indptr_type, const void *a_indices,
                                         skt_itype index_type, const void *a_vals, skt_dtype val_dtype,
                                         int64_t nnz, int64_t d, void *sa, skt_dtype sa_dtype, int64_t ldsa,
                                         void *ws, size_t ws_bytes, void *stream_) {
  static const char *fn = "skt_apply_csr_wide";
  if (!indptr || t < 1 || t > (1ull << 32) || n < 0 || d < 0 || ldsa < d || !a_indptr || nnz < 0 ||
      (indptr_type != SKT_I32 && indptr_type != SKT_I64) || (index_type != SKT_I32 && index_type != SKT_I64) ||
      (val_dtype != SKT_F32 && val_dtype != SKT_F64) || (sa_dtype != SKT_F32 && sa_dtype != SKT_F64) ||
      d >= (1LL << 31))
    return fail(SKT_EINVAL, fn, "bad arguments");
  if (d == 0) return SKT_OK;
  if (!sa || (n > 0 && !rows)) return fail(SKT_EINVAL, fn, "NULL buffer");
  size_t need = 0;
  skt_apply_csr_wide_workspace(n, t, d, nnz, val_dtype, &need);
  if (!ws || ws_bytes < need) return fail(SKT_EWORKSPACE, fn, "workspace too small");
  cudaStream_t s = as_stream(stream_);
  int32_t *cur = (int32_t *)ws;
  if (indptr_type == SKT_I32)
    return index_type == SKT_I32
               ? wide_by_vals<int32_t, int32_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, cur, s)
               : wide_by_vals<int32_t, int64_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, cur, s);
  return index_type == SKT_I32
             ? wide_by_vals<int64_t, int32_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, cur, s)
             : wide_by_vals<int64_t, int64_t>(indptr, rows, t, n, a_indptr, a_indices, a_vals, val_dtype, nnz, d, sa, sa_dtype, ldsa, cur, s);
}
