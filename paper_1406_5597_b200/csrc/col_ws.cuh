// Column c2c (stages 1b / 1b' / 3 / 3' at p = 1) moved entirely by the
// tensor-memory-access unit (sm_100a).
//
// Why: the cp.async column kernel (kernels.cuh) spends as long on its memory
// instructions as on its arithmetic.  Measured on a 1024^3 f64 launch
// (TFFFT_PROBE_COL): compute + shared-memory exchange alone 1.58 ms, + the
// per-thread cp.async loads 2.22-2.30 ms, + the per-thread stores 3.26-3.69 ms,
// and just as long with the slab L2-resident (TFFFT_PROBE_ALIAS): the stores
// (STG.128, one L2 request per row segment) and loads occupy the load/store
// unit while the FP64 pipe idles.  Per-thread stores of 64-byte row segments
// were measured 2x slower still.
//
// Here one thread per CTA moves every byte with cp.async.bulk.tensor: a tile
// of W columns (64-byte rows) lands in a 64 KB shared stage, the radix-32
// passes exchange through the same stage (rows XOR-swizzled so every access is
// bank-conflict free), the results are written back into the stage in natural
// order and stored by the TMA unit.  Two CTAs share an SM, so one CTA's
// arithmetic overlaps the other's store/load turnaround:
//
//   thread 0: wait until the previous store has read the stage (per 256-row
//             box, so loads of the next tile start box by box) -> N/256 box
//             loads on mbarrier `full`
//   all     : wait full -> operands -> pass 0 -> exchange -> pass 1 ->
//             results -> fence.proxy.async -> thread 0 issues the box stores
//
// Column tiles: the map is [grp][row][col] (cols contiguous, rows `rstride`
// apart, groups `gstride` apart); tile t covers columns [c0, c0 + W) of group
// t / tpg.  Out-of-range columns of a group's last tile are zero-filled by the
// load and clipped by the store.  The arithmetic is the Stockham engine of
// fft_engine.cuh (same radix schedule and twiddles), so the results are
// bit-identical to col_fft_kernel's.
#pragma once
#include <cuda.h>

#include "fourstep_tma.cuh"

namespace tffft {

template <typename T, int L>
struct WsCfg {
  using SH = Shape<L>;
  static constexpr int N = SH::N, E = SH::E, TPT = SH::TPT;
  static_assert(SH::P == 2, "two-pass radix schedules only");
  static constexpr int W = 64 / (int)sizeof(cx<T>);  // columns per tile: 64-byte rows
  static constexpr int THREADS = W * TPT;
  static constexpr int BOX = N < 256 ? N : 256;      // rows per TMA box (hardware limit 256)
  static constexpr int NBOX = N / BOX;
  static constexpr size_t STAGE = sizeof(cx<T>) * (size_t)N * W;
  static constexpr int TW = SH::TW > 0 ? SH::TW : 1;
  static constexpr size_t SMEM = STAGE + sizeof(cx<T>) * TW + 64;
  static constexpr int LR0 = pass_bits(L, 0);        // log2 of the first radix
};

struct WsParams {
  void* data;            // column base (element 0 of group 0, column 0)
  const void* tw;        // pass tables (fft_engine.cuh layout)
  long long ntiles;
  int tpg;               // tiles per group
  int cols;              // columns per group
  long long rstride;     // elements between the rows of a column
  long long gstride;     // elements between groups
  int evict_first;       // L2 eviction priority of the loads
};

// wait until at most n bulk groups of this thread are still reading shared memory
__device__ __forceinline__ void bulk_wait_read_n(int n) {
  if (n >= 3) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
  else if (n == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
  else if (n == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <typename T, int L, bool INV>
__global__ void __launch_bounds__(WsCfg<T, L>::THREADS, 2)
col_ws_kernel(const __grid_constant__ CUtensorMap map, const WsParams prm) {
  using CF = WsCfg<T, L>;
  using SH = Shape<L>;
  using ST = Stockham<T, L, INV, 1, 30, false, 0, true>;  // compute<p> only (the exchange is done here)
  constexpr int N = CF::N, E = CF::E, TPT = CF::TPT, W = CF::W;
  constexpr int R0 = SH::R0, R1 = SH::RL, LR0 = CF::LR0;

  extern __shared__ __align__(1024) unsigned char smem_ws[];
  cx<T>* st = reinterpret_cast<cx<T>*>(smem_ws);
  cx<T>* s_tw = reinterpret_cast<cx<T>*>(smem_ws + CF::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_ws + CF::STAGE + sizeof(cx<T>) * CF::TW);

  const int t = threadIdx.x;
  const int b = t % W, tt = t / W;
  if (t == 0) {
    mbar_init(full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const cx<T>* g = reinterpret_cast<const cx<T>*>(prm.tw);
    for (int k = t; k < SH::TW; k += CF::THREADS) s_tw[k] = g[k];
  }
  __syncthreads();

  const long long first = blockIdx.x, step = gridDim.x;
  const long long mine = prm.ntiles > first ? (prm.ntiles - 1 - first) / step + 1 : 0;
  const uint64_t pol_ld = prm.evict_first ? policy_evict_first() : policy_evict_normal();
  const uint64_t pol_st = policy_evict_first();
  auto coords = [&](long long i, int& grp, int& c0) {
    const long long tile = first + i * step;
    grp = (int)(tile / prm.tpg);
    c0 = (int)(tile % prm.tpg) * W;
  };
  // exchange row of element a: flip bit 0 with bit LR0 (rows 2^LR0 apart share banks)
  auto xrow = [](int a) { return a ^ ((a >> LR0) & 1); };

  if (t == 0 && mine > 0) {
    mbar_arrive_tx(full, (unsigned)CF::STAGE);
    int grp, c0;
    coords(0, grp, c0);
#pragma unroll
    for (int q = 0; q < CF::NBOX; ++q)
      tma_load3(st + (size_t)q * CF::BOX * W, &map, 2 * c0, q * CF::BOX, grp, full, pol_ld);
  }
  for (long long i = 0; i < mine; ++i) {
    mbar_wait(full, (unsigned)(i & 1));
    cx<T> v[E];
#pragma unroll
    for (int kk = 0; kk < E; ++kk) v[SH::in_slot(kk)] = st[(tt + TPT * kk) * W + b];
    __syncthreads();  // every operand read before the exchange overwrites the stage
    ST::template compute<0>(v, tt, s_tw);
    // pass-0 outputs: butterfly j = tt + TPT u, value m -> element j R0 + m (Stockham, Ns = 1)
#pragma unroll
    for (int u = 0; u < E / R0; ++u)
#pragma unroll
      for (int m = 0; m < R0; ++m) st[xrow((tt + TPT * u) * R0 + m) * W + b] = v[u * R0 + m];
    __syncthreads();
    // pass-1 inputs: butterfly j = tt + TPT u, value m <- element j + m N / R1
#pragma unroll
    for (int u = 0; u < E / R1; ++u)
#pragma unroll
      for (int m = 0; m < R1; ++m) v[u * R1 + m] = st[xrow(tt + TPT * u + m * (N / R1)) * W + b];
    __syncthreads();
    ST::template compute<1>(v, tt, s_tw);
#pragma unroll
    for (int u = 0; u < E / R1; ++u)
#pragma unroll
      for (int m = 0; m < R1; ++m) st[SH::out_elem(tt, u, m) * W + b] = v[u * R1 + m];
    fence_async_shared();  // generic-proxy writes -> visible to the TMA store
    __syncthreads();
    if (t == 0) {
      int grp, c0;
      coords(i, grp, c0);
#pragma unroll
      for (int q = 0; q < CF::NBOX; ++q) {
        tma_store3(&map, 2 * c0, q * CF::BOX, grp, st + (size_t)q * CF::BOX * W, pol_st);
        bulk_commit();
      }
      if (i + 1 < mine) {
        // reload box by box as soon as the store has read it out of the stage
        mbar_arrive_tx(full, (unsigned)CF::STAGE);
        coords(i + 1, grp, c0);
#pragma unroll
        for (int q = 0; q < CF::NBOX; ++q) {
          bulk_wait_read_n(CF::NBOX - 1 - q);
          tma_load3(st + (size_t)q * CF::BOX * W, &map, 2 * c0, q * CF::BOX, grp, full, pol_ld);
        }
      }
    }
  }
  if (t == 0) bulk_wait0();  // stores complete before the CTA (and its shared memory) retires
}

// lengths with a TMA column kernel (two radix passes)
__host__ __device__ constexpr bool col_ws_supported(int L) { return L == 9 || L == 10; }

template <typename T>
cudaError_t launch_col_ws(int L, bool inv, const CUtensorMap& map, const WsParams& p, cudaStream_t s);

}  // namespace tffft
