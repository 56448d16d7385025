// Explicit instantiation + runtime dispatch of the stage kernels for one
// precision.  Included by kernels_f64.cu / kernels_f32.cu with TFFFT_REAL set.
#include <algorithm>
#include <atomic>

#include "kernels.cuh"
#include "fourstep.cuh"
#include "stage1_fused.cuh"
#include "fourstep_tma.cuh"
#include "col_tma.cuh"
#include "col_wpc.cuh"
#include "col_wpc2.cuh"

namespace tffft {

// Per-device launch state.  cudaFuncSetAttribute(MaxDynamicSharedMemorySize)
// and the occupancy / SM-count queries apply to the current device only, so a
// process that plans on several devices (comm_init_all, make_communicators on
// device 1 after device 0) caches them per device.
constexpr int kMaxDevices = 64;
static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : d % kMaxDevices;
}

// one per kernel instantiation (a static of its launcher)
struct KernelCache {
  std::atomic<unsigned long long> prepped{0};  // bit d: smem attribute set on device d
  std::atomic<int> occ[kMaxDevices] = {};      // resident CTAs per SM on device d (0: not queried)
};

template <typename K>
static cudaError_t prep_smem(K kernel, KernelCache& kc, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  const unsigned long long bit = 1ull << current_device();
  if (kc.prepped.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) kc.prepped.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// resident CTAs per SM of `kernel` on the current device (after prep_smem)
template <typename K>
static int occupancy(K kernel, KernelCache& kc, int threads, size_t smem) {
  std::atomic<int>& c = kc.occ[current_device()];
  int n = c.load(std::memory_order_relaxed);
  if (n > 0) return n;
  n = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  n = n < 1 ? 1 : n;
  c.store(n, std::memory_order_relaxed);
  return n;
}

static int num_sms() {
  static std::atomic<int> cache[kMaxDevices] = {};
  const int dev = current_device();
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

template <typename T, int L, bool INV, bool TWO, int RD, bool WIDE>
static cudaError_t col_one(const ColParams& p, cudaStream_t s) {
  using CF = ColCfg<T, L, WIDE>;
  const size_t sm = col_smem_bytes<T, L, WIDE>();
  auto k = col_fft_kernel<T, L, INV, TWO, RD, WIDE>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, sm);
  if (prep != cudaSuccess) return prep;
  const int per_sm = occupancy(k, kc, CF::THREADS, sm);
  const long long tiles = (p.ncols + CF::CL * CF::B - 1) / (CF::CL * CF::B);
  if (tiles <= 0) return cudaSuccess;
  long long blocks = CF::PERSISTENT ? std::min<long long>(tiles * CF::CL, (long long)per_sm * num_sms())
                                    : tiles * CF::CL;
  blocks = std::max<long long>(CF::CL, blocks / CF::CL * CF::CL);
  (void)cudaGetLastError();  // clear any stale error of this thread
  if constexpr (CF::CL == 1) {
    k<<<(unsigned)blocks, CF::THREADS, sm, s>>>(p);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(CF::THREADS);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CF::CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, p);
  }
  return cudaGetLastError();
}

template <typename T, int L>
static cudaError_t r2c_one(const RowParams& p, cudaStream_t s) {
  using RC = RowCfg<L, r2c_radix_bits(L, sizeof(T))>;
  const size_t sm = row_smem_bytes<T, L, r2c_radix_bits(L, sizeof(T))>();
  auto k = r2c_rows_kernel<T, L>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, sm);
  if (prep != cudaSuccess) return prep;
  const long long blocks = (p.nrows + RC::B - 1) / RC::B;
  if (blocks <= 0) return cudaSuccess;
  (void)cudaGetLastError();  // clear any stale error of this thread
  k<<<(unsigned)blocks, RC::THREADS, sm, s>>>(p);
  return cudaGetLastError();
}

template <typename T, int L>
static cudaError_t c2r_one(const RowParams& p, cudaStream_t s) {
  using RC = RowCfg<L, c2r_radix_bits(L, sizeof(T))>;
  const size_t sm = row_smem_bytes<T, L, c2r_radix_bits(L, sizeof(T))>();
  auto k = c2r_rows_kernel<T, L>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, sm);
  if (prep != cudaSuccess) return prep;
  const long long blocks = (p.nrows + RC::B - 1) / RC::B;
  if (blocks <= 0) return cudaSuccess;
  (void)cudaGetLastError();  // clear any stale error of this thread
  k<<<(unsigned)blocks, RC::THREADS, sm, s>>>(p);
  return cudaGetLastError();
}

// instantiated variants: stage 1b fwd (+redirect), stage 1b' inv, stage 3 fwd
// (single / two-level), stage 3' inv (single / two-level + redirect)
template <typename T, int L>
static cudaError_t col_dispatch(bool inv, bool two, int rd, bool wide, const ColParams& p, cudaStream_t s) {
  // stage 1b (narrow): forward in place / + peer bands to staging (p > 1)
  //          1b':      inverse in place / + peer bands read from landing (p > 1)
  // stage 3  (wide):   forward in place (p = 1) / two-level + landing reads (p > 1)
  //          3':       inverse in place (p = 1) / two-level + staging writes (p > 1)
  if (!wide) {
    if (two) return cudaErrorInvalidValue;
    if (!inv && rd == 0) return col_one<T, L, false, false, 0, false>(p, s);
    if (!inv && rd == 1) return col_one<T, L, false, false, 1, false>(p, s);
    if (inv && rd == 0) return col_one<T, L, true, false, 0, false>(p, s);
    if (inv && rd == 2) return col_one<T, L, true, false, 2, false>(p, s);
    return cudaErrorInvalidValue;
  }
  if (!inv && !two && rd == 0) return col_one<T, L, false, false, 0, true>(p, s);
  if (!inv && two && rd == 2) return col_one<T, L, false, true, 2, true>(p, s);
  if (inv && !two && rd == 0) return col_one<T, L, true, false, 0, true>(p, s);
  if (inv && two && rd == 1) return col_one<T, L, true, true, 1, true>(p, s);
  return cudaErrorInvalidValue;
}
#define TFFFT_COL_CASE(LL) \
  case LL: return col_dispatch<TFFFT_REAL, LL>(inv, two, rd, wide, p, s);
#define TFFFT_ROW_CASE(LL, FN) \
  case LL: return FN<TFFFT_REAL, LL>(p, s);

template <>
cudaError_t launch_col_fft<TFFFT_REAL>(int L, bool inv, bool two, int rd, bool wide, const ColParams& p,
                                       cudaStream_t s) {
  switch (L) {
    TFFFT_COL_CASE(1) TFFFT_COL_CASE(2) TFFFT_COL_CASE(3) TFFFT_COL_CASE(4)
    TFFFT_COL_CASE(5) TFFFT_COL_CASE(6) TFFFT_COL_CASE(7) TFFFT_COL_CASE(8)
    TFFFT_COL_CASE(9) TFFFT_COL_CASE(10) TFFFT_COL_CASE(11) TFFFT_COL_CASE(12)
    default: return cudaErrorInvalidValue;
  }
}

template <>
cudaError_t launch_r2c_rows<TFFFT_REAL>(int L, const RowParams& p, cudaStream_t s) {
  switch (L) {
    TFFFT_ROW_CASE(0, r2c_one) TFFFT_ROW_CASE(1, r2c_one) TFFFT_ROW_CASE(2, r2c_one)
    TFFFT_ROW_CASE(3, r2c_one) TFFFT_ROW_CASE(4, r2c_one) TFFFT_ROW_CASE(5, r2c_one)
    TFFFT_ROW_CASE(6, r2c_one) TFFFT_ROW_CASE(7, r2c_one) TFFFT_ROW_CASE(8, r2c_one)
    TFFFT_ROW_CASE(9, r2c_one) TFFFT_ROW_CASE(10, r2c_one) TFFFT_ROW_CASE(11, r2c_one)
    default: return cudaErrorInvalidValue;
  }
}

template <>
cudaError_t launch_c2r_rows<TFFFT_REAL>(int L, const RowParams& p, cudaStream_t s) {
  switch (L) {
    TFFFT_ROW_CASE(0, c2r_one) TFFFT_ROW_CASE(1, c2r_one) TFFFT_ROW_CASE(2, c2r_one)
    TFFFT_ROW_CASE(3, c2r_one) TFFFT_ROW_CASE(4, c2r_one) TFFFT_ROW_CASE(5, c2r_one)
    TFFFT_ROW_CASE(6, c2r_one) TFFFT_ROW_CASE(7, c2r_one) TFFFT_ROW_CASE(8, c2r_one)
    TFFFT_ROW_CASE(9, c2r_one) TFFFT_ROW_CASE(10, c2r_one) TFFFT_ROW_CASE(11, c2r_one)
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int LA, int LB, bool INV, bool TWO, bool REDIR>
static cudaError_t fs_one(const FourStepParams& p, cudaStream_t s) {
  const size_t sm = fourstep_smem_bytes<T, LA, LB>();
  auto k = fourstep_kernel<T, LA, LB, INV, TWO, REDIR>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, sm);
  if (prep != cudaSuccess) return prep;
  const int per_sm = occupancy(k, kc, kFsThreads, sm);
  (void)cudaGetLastError();
  k<<<(unsigned)(per_sm * num_sms()), kFsThreads, sm, s>>>(p);
  return cudaGetLastError();
}

template <typename T, int LA, int LB>
static cudaError_t fs_dispatch(bool inv, int variant, const FourStepParams& p, cudaStream_t s) {
  if (!inv) {
    if (variant == 0) return fs_one<T, LA, LB, false, false, false>(p, s);
    if (variant == 2) return fs_one<T, LA, LB, false, true, false>(p, s);
  } else {
    if (variant == 0) return fs_one<T, LA, LB, true, false, false>(p, s);
    if (variant == 3) return fs_one<T, LA, LB, true, true, true>(p, s);
  }
  return cudaErrorInvalidValue;
}

template <typename T, int LR, int LC, bool FWD, bool REDIR>
static cudaError_t s1_one(const Stage1Params& p, cudaStream_t s) {
  const size_t sm = S1Cfg<T, LR, LC>::SMEM;
  auto k = stage1_fused_kernel<T, LR, LC, FWD, REDIR>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, sm);
  if (prep != cudaSuccess) return prep;
  const int per_sm = occupancy(k, kc, kS1Threads, sm);
  (void)cudaGetLastError();
  k<<<(unsigned)(per_sm * num_sms()), kS1Threads, sm, s>>>(p);
  return cudaGetLastError();
}

template <typename T, int LR>
static cudaError_t s1_dispatch(bool fwd, bool redir, const Stage1Params& p, cudaStream_t s) {
  if (!fwd) return s1_one<T, LR, LR + 1, false, false>(p, s);
  return redir ? s1_one<T, LR, LR + 1, true, true>(p, s) : s1_one<T, LR, LR + 1, true, false>(p, s);
}

template <>
cudaError_t launch_stage1_fused<TFFFT_REAL>(int LR, int LC, bool fwd, bool redir, const Stage1Params& p,
                                            cudaStream_t s) {
  if (LC != LR + 1) return cudaErrorInvalidValue;
  switch (LR) {
    case 8: return s1_dispatch<TFFFT_REAL, 8>(fwd, redir, p, s);
    case 9: return s1_dispatch<TFFFT_REAL, 9>(fwd, redir, p, s);
    case 10: return s1_dispatch<TFFFT_REAL, 10>(fwd, redir, p, s);
    case 11: return s1_dispatch<TFFFT_REAL, 11>(fwd, redir, p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int LA, int LB, bool INV>
static cudaError_t ft_one(const CUtensorMap* maps, const FsTmaParams& p, cudaStream_t s) {
  const size_t sm = FtCfg<T, LA, LB>::SMEM;
  auto k = fourstep_tma_kernel<T, LA, LB, INV>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, sm);
  if (prep != cudaSuccess) return prep;
  const int per_sm = occupancy(k, kc, kFtThreads, sm);
  (void)cudaGetLastError();
  k<<<(unsigned)(per_sm * num_sms()), kFtThreads, sm, s>>>(maps[0], maps[1], maps[2], maps[3], p);
  return cudaGetLastError();
}

template <>
cudaError_t launch_fourstep_tma<TFFFT_REAL>(int L, bool inv, const CUtensorMap* maps, const FsTmaParams& p,
                                            cudaStream_t s) {
  switch (L) {
    case 10: return inv ? ft_one<TFFFT_REAL, 5, 5, true>(maps, p, s) : ft_one<TFFFT_REAL, 5, 5, false>(maps, p, s);
    case 12: return inv ? ft_one<TFFFT_REAL, 6, 6, true>(maps, p, s) : ft_one<TFFFT_REAL, 6, 6, false>(maps, p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int L, bool INV, int NB, bool TWO, bool FPF>
static cudaError_t tc_one(const CUtensorMap& map, const CUtensorMap& map_odd, const TmaColParams& p, cudaStream_t s) {
  using TC = TmaColCfg<T, L, NB, FPF>;
  if constexpr (!TC::OK) {
    return cudaErrorNotSupported;  // col_tma_width() reports 0 for this shape: never launched
  } else {
  auto k = col_tma_kernel<T, L, INV, NB, TWO, FPF>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, TC::SMEM);
  if (prep != cudaSuccess) return prep;
  if (p.ntiles <= 0) return cudaSuccess;
  // persistent: every resident CTA slot of the GPU (one per SM wide, two narrow)
  const long long blocks =
      std::min<long long>(p.ntiles, (long long)occupancy(k, kc, TC::THREADS, TC::SMEM) * num_sms());
  (void)cudaGetLastError();
  k<<<(unsigned)blocks, TC::THREADS, TC::SMEM, s>>>(map, map_odd, p);
  return cudaGetLastError();
  }
}

// full-prefetch variant (col_tma.cuh FPF), the default; TFFFT_TMA_FPF=0
// selects the half-and-half prefetch.  Measured at 1024^3
// (profiles/r02/fpf_ab.txt): isolated (ncu) 3.00 vs 2.97 ms per launch, but in
// the live pair at the power cap stage 3 + 3' take 6.61-6.76 ms instead of
// 7.00-7.05 (float32: 3.31 vs 3.43 ms).
static bool tma_fpf() {
  static const bool v = [] {
    const char* e = getenv("TFFFT_TMA_FPF");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}
// narrow shape (half-width tiles, two CTAs per SM) for the stage-1b passes:
// TFFFT_TMA_NARROW=1.  Measured on one box (profiles/r02/narrow_ab.txt):
// 2.96 vs 2.86 ms per isolated 1024^3 stage-1b launch and no gain in the live
// pair, so the wide shape is the default everywhere.
static bool tma_narrow() {
  static const bool v = [] {
    const char* e = getenv("TFFFT_TMA_NARROW");
    return e ? atoi(e) != 0 : false;
  }();
  return v;
}

template <typename T, int L, bool TWO, int NB>
static cudaError_t tc_dispatch3(bool inv, const CUtensorMap& map, const CUtensorMap& map_odd, const TmaColParams& p,
                                cudaStream_t s) {
  if (tma_fpf() && TmaColCfg<T, L, NB, true>::OK)
    return inv ? tc_one<T, L, true, NB, TWO, true>(map, map_odd, p, s)
               : tc_one<T, L, false, NB, TWO, true>(map, map_odd, p, s);
  return inv ? tc_one<T, L, true, NB, TWO, false>(map, map_odd, p, s)
             : tc_one<T, L, false, NB, TWO, false>(map, map_odd, p, s);
}

template <typename T, int L, bool TWO>
static cudaError_t tc_dispatch2(bool inv, bool wide, const CUtensorMap& map, const CUtensorMap& map_odd,
                                const TmaColParams& p, cudaStream_t s) {
  if (wide || !tma_narrow()) return tc_dispatch3<T, L, TWO, tma_cols_per_cta<T, L>(true)>(inv, map, map_odd, p, s);
  return tc_dispatch3<T, L, TWO, tma_cols_per_cta<T, L>(false)>(inv, map, map_odd, p, s);
}

template <typename T, int L>
static cudaError_t tc_dispatch(bool inv, bool wide, bool two, const CUtensorMap& map, const CUtensorMap& map_odd,
                               const TmaColParams& p, cudaStream_t s) {
  return two ? tc_dispatch2<T, L, true>(inv, wide, map, map_odd, p, s)
             : tc_dispatch2<T, L, false>(inv, wide, map, map_odd, p, s);
}

template <>
cudaError_t launch_col_tma<TFFFT_REAL>(int L, bool inv, bool wide, bool two, const CUtensorMap& map,
                                       const CUtensorMap& map_odd, const TmaColParams& p, cudaStream_t s) {
  switch (L) {
    case 9: return tc_dispatch<TFFFT_REAL, 9>(inv, wide, two, map, map_odd, p, s);
    case 10: return tc_dispatch<TFFFT_REAL, 10>(inv, wide, two, map, map_odd, p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <>
int col_tma_width<TFFFT_REAL>(int L, bool wide) {
  const bool w = wide || !tma_narrow();
  constexpr int W9 = tma_cols_per_cta<TFFFT_REAL, 9>(true), N9 = tma_cols_per_cta<TFFFT_REAL, 9>(false);
  constexpr int W10 = tma_cols_per_cta<TFFFT_REAL, 10>(true), N10 = tma_cols_per_cta<TFFFT_REAL, 10>(false);
  switch (L) {
    case 9: return w ? (TmaColCfg<TFFFT_REAL, 9, W9>::OK ? W9 : 0) : (TmaColCfg<TFFFT_REAL, 9, N9>::OK ? N9 : 0);
    case 10: return w ? (TmaColCfg<TFFFT_REAL, 10, W10>::OK ? W10 : 0) : (TmaColCfg<TFFFT_REAL, 10, N10>::OK ? N10 : 0);
    default: return 0;
  }
}

template <typename T, int L, bool INV>
static cudaError_t wpc_one(const WpcMaps& maps, const WpcParams& p, cudaStream_t s) {
  using WC = WpcCfg<T, L>;
  auto k = col_wpc_kernel<T, L, INV>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, WC::SMEM);
  if (prep != cudaSuccess) return prep;
  if (p.ntiles <= 0) return cudaSuccess;
  // persistent: one CTA per SM
  const long long blocks = std::min<long long>(p.ntiles, (long long)num_sms());
  (void)cudaGetLastError();
  k<<<(unsigned)blocks, WC::THREADS, WC::SMEM, s>>>(maps, p);
  return cudaGetLastError();
}

template <typename T, bool INV>
static cudaError_t wpc2_one(const WpcMaps& maps, const WpcParams& p, cudaStream_t s) {
  using WC = WpcCfg<T, 10>;
  using W2 = Wpc2Cfg<T>;
  auto k = col_wpc2_kernel<T, INV>;
  static KernelCache kc;
  const cudaError_t prep = prep_smem(k, kc, W2::SMEM);
  if (prep != cudaSuccess) return prep;
  if (p.ntiles <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>(p.ntiles, (long long)num_sms());  // one CTA per SM (all of its TMEM)
  (void)cudaGetLastError();
  k<<<(unsigned)blocks, WC::THREADS, W2::SMEM, s>>>(maps, p);
  return cudaGetLastError();
}

template <>
cudaError_t launch_col_wpc<TFFFT_REAL>(int L, bool inv, const WpcMaps& maps, const WpcParams& p, cudaStream_t s) {
  if (L == 11) return inv ? wpc2_one<TFFFT_REAL, true>(maps, p, s) : wpc2_one<TFFFT_REAL, false>(maps, p, s);
  if (L == 9) return inv ? wpc_one<TFFFT_REAL, 9, true>(maps, p, s) : wpc_one<TFFFT_REAL, 9, false>(maps, p, s);
  if (L != 10) return cudaErrorInvalidValue;
  return inv ? wpc_one<TFFFT_REAL, 10, true>(maps, p, s) : wpc_one<TFFFT_REAL, 10, false>(maps, p, s);
}

template <>
int col_wpc_width<TFFFT_REAL>(int L) {
  if (L == 11) return Wpc2Cfg<TFFFT_REAL>::OK ? WpcCfg<TFFFT_REAL, 10>::B : 0;
  if (L == 9) return WpcCfg<TFFFT_REAL, 9>::OK ? WpcCfg<TFFFT_REAL, 9>::B : 0;
  return L == 10 && WpcCfg<TFFFT_REAL, 10>::OK ? WpcCfg<TFFFT_REAL, 10>::B : 0;
}

template <>
cudaError_t launch_fourstep<TFFFT_REAL>(int L, bool inv, int variant, const FourStepParams& p, cudaStream_t s) {
  switch (L) {
    case 9: return fs_dispatch<TFFFT_REAL, 5, 4>(inv, variant, p, s);
    case 10: return fs_dispatch<TFFFT_REAL, 5, 5>(inv, variant, p, s);
    case 11: return fs_dispatch<TFFFT_REAL, 6, 5>(inv, variant, p, s);
    case 12: return fs_dispatch<TFFFT_REAL, 6, 6>(inv, variant, p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tffft
