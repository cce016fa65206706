// lev_dmma.cu -- launcher of the fp64 tensor-core leverage contraction
// (lev_dmma.cuh) behind skt_lev_rownorms_csr for fp64 values (leverage.py:90-91).
#include <cstdlib>

#include "common.cuh"
#include "lev_dmma.cuh"

namespace skt {
namespace {

inline bool dmma_enabled() {  // SKT_LEV_DMMA=0: the CUDA-core fp64 kernels (A/B)
  static const bool on = [] {
    const char *e = getenv("SKT_LEV_DMMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename IP, typename IX, typename TS, int KS, int NB>
skt_status launch(int64_t n, int64_t d, const void *aip, const void *aix, const void *av, const double *p,
                  int64_t k, void *scores, cudaStream_t st) {
  static const char *fn = "skt_lev_rownorms_csr";
  auto kern = lev_dmma_kernel<IP, IX, double, TS, KS, NB>;
  const size_t smem = dmma_smem<KS>();
  SKT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), fn);
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (n + kDmRows - 1) / kDmRows;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sms));
  SKT_LAUNCH(kern, (unsigned)blocks, kDmThreads, smem, st, n, (int)d, (const IP *)aip, (const IX *)aix,
             (const double *)av, p, (int)k, (TS *)scores);
  return check_launch(fn);
}

template <typename IP, typename IX>
skt_status by_shape(int64_t n, int64_t d, const void *aip, const void *aix, const void *av, const double *p,
                    int64_t k, void *scores, skt_dtype sdt, cudaStream_t st) {
#define SKT_DM(KS, NB)                                                                                  \
  (sdt == SKT_F64 ? launch<IP, IX, double, KS, NB>(n, d, aip, aix, av, p, k, scores, st)                 \
                  : launch<IP, IX, float, KS, NB>(n, d, aip, aix, av, p, k, scores, st))
  if (d <= 32) return k == 16 ? SKT_DM(8, 2) : SKT_DM(8, 4);
  return k == 16 ? SKT_DM(16, 2) : SKT_DM(16, 4);
#undef SKT_DM
}

}  // namespace

// fp64 CSR values, d <= 64, k in {16, 32}; SKT_ENOTSUP otherwise (the caller
// then runs the CUDA-core kernels)
skt_status lev_dmma_csr(int64_t n, int64_t d, const void *aip, skt_itype ipt, const void *aix, skt_itype ixt,
                        const void *av, skt_dtype vt, const double *p, int64_t k, void *scores, skt_dtype sdt,
                        cudaStream_t st) {
  if (!dmma_enabled() || vt != SKT_F64 || d < 1 || d > 64 || (k != 16 && k != 32) || n < 1) return SKT_ENOTSUP;
  if (ipt == SKT_I32)
    return ixt == SKT_I32 ? by_shape<int32_t, int32_t>(n, d, aip, aix, av, p, k, scores, sdt, st)
                          : by_shape<int32_t, int64_t>(n, d, aip, aix, av, p, k, scores, sdt, st);
  return ixt == SKT_I32 ? by_shape<int64_t, int32_t>(n, d, aip, aix, av, p, k, scores, sdt, st)
                        : by_shape<int64_t, int64_t>(n, d, aip, aix, av, p, k, scores, sdt, st);
}

}  // namespace skt
