// Column c2c (stages 1b / 1b' / 3 / 3' at p = 1) fed by the tensor-memory-
// access unit (sm_100a).
//
// Same tiles, thread mapping, arithmetic and stores as col_fft_kernel
// (kernels.cuh): B adjacent columns (128-byte row visits), one persistent CTA
// per SM, the N-point columns as Stockham radix passes with a shared-memory
// exchange.  What changes is how the next tile gets in.  col_fft_kernel issues
// one 16-byte (float64) or 8-byte (float32) cp.async per element and thread,
// plus its address arithmetic; here thread 0 moves each tile with N / 256 box
// copies (cp.async.bulk.tensor, 256 rows x B columns each):
//
//   boxes [0, NBOX/2)    -> the prefetch region, issued as soon as every
//                           thread has read the current tile's operands;
//   boxes [NBOX/2, NBOX) -> the exchange buffer, issued once the current
//                           tile's last exchange has drained it (Stockham hook).
//
// Each half completes on its own mbarrier.  Tile t covers columns
// [c0, c0 + B) of group t / tpg of a [grp][row][col] tensor map; columns past
// the end of a group are zero-filled by the load and never stored.  Results
// are bit-identical to col_fft_kernel's (same engine, same twiddles).
//
// Two-level addressing (p > 1, template TWO and the 4D load mode): the rows
// of a STRIDED_INPLACE column are n0/p planes x p blocks, and the landing
// buffer holds block s of every column at landing[s][i][c].  Loads then go
// through a 4D map (cols, rows_in, rows_out, groups) -- row r is (r mod rows_in,
// r / rows_in) -- in boxes that never cross a block; stores go through a table
// of up to kTmaTab block pointers: element r of column c of group g lands at
// tab[r >> sin_shift] + g * sgstride + c + (r mod 2^sin_shift) * sin_stride.
// That is the forward stage-3 read of the landing bands and in-place write,
// the inverse stage-3' write-redirect of every block (self block to
// landing[rank], peers to staging or straight into the peer's landing
// buffer), the forward stage-1b write-redirect and the inverse stage-1b' read
// of the landing bands -- the reference's strided exchange datatype
// (exchange.py:114-121) applied by the FFT's own TMA boxes and stores.
//
// Measured on 1024^3 (profiles/r01s10/tma_f64_ticket.txt, r01s11/tma_512.txt):
// with the ticket tile order this kernel beat col_fft_kernel on every 512- and
// 1024-point column pass of either precision (2.96 ms per float64 1024^3
// launch against 3.25-3.69 ms).  Storing half of each tile through the TMA
// unit as well (staged behind the next tile's boxes in the exchange buffer)
// did not change the time.
//
// Since round 2 session 4 the warp-per-column kernels (col_wpc.cuh,
// col_wpc2.cuh) run most of those passes (tffft.cu columns_wpc).  This kernel
// keeps the float64 1024-point stage-3 / 3' passes (a tie in isolation, faster
// live, profiles/r02s4/wpc_ab.txt), the float32 stage-1b rows that miss
// 16-byte alignment on odd rows (the two-map parity scheme below; a swizzled
// box cannot start off alignment), and anything TFFFT_WPC=0 sends back.
#pragma once
#include <cuda.h>

#include "fourstep_tma.cuh"
#include "kernels.cuh"

namespace tffft {

// column-kernel store flavour: 0 plain, 1 L2 cache-hint policy, 2 st.global.cs
#ifndef TFFFT_COL_STORE
#define TFFFT_COL_STORE 0
#endif
__device__ __forceinline__ void st_cs(cx<double>* a, cx<double> z) { __stcs(reinterpret_cast<double2*>(a), make_double2(z.x, z.y)); }
__device__ __forceinline__ void st_cs(cx<float>* a, cx<float> z) { __stcs(reinterpret_cast<float2*>(a), make_float2(z.x, z.y)); }

// FPF (full prefetch): the whole next tile streams into a dedicated region as
// soon as the current tile's operands are read, and the Stockham exchange runs
// in a separate, half-size buffer of real words (re round, then im round).
// Without FPF the next tile's second half must wait for the exchange buffer
// to drain (about half a tile later).
// Columns per CTA: WIDE passes (stage 3 / 3', rows megabytes apart) take
// 128-byte row segments -- 8 float64 or 16 float32 columns at 1024 points (at
// least 256 threads), one CTA per SM; NARROW passes (stage 1b / 1b', rows n2c
// elements apart) may take half as many columns, two CTAs per SM
// (TFFFT_TMA_NARROW=1; profiles/r02/narrow_ab.txt: slower in isolation and no
// gain live, so off; at the 8.4 MB stage-3 stride 64-byte boxes over-fetch
// 1.5x and are much slower, profiles/r02/b4_ab.txt).
template <typename T, int L>
__host__ __device__ constexpr int tma_cols_per_cta(bool wide) {
  // wide: 128-byte rows and at least 256 threads; narrow: half of that
  const int rowc = 8 * (int)(16 / sizeof(cx<T>)), tpt = Shape<L>::TPT;
  const int w = 256 / tpt > rowc ? 256 / tpt : rowc;
  return wide ? w : w / 2;
}

template <typename T, int L, int NB, bool FPF = false>
struct TmaColCfg {
  using SH = Shape<L>;
  static constexpr int N = SH::N, B = NB, TPT = SH::TPT, THREADS = TPT * NB;
  // resident CTAs per SM the registers are capped for: two for the narrow shape
  static constexpr int MINB = NB < tma_cols_per_cta<T, L>(true) ? 2 : 1;
  static constexpr int PS = SH::EB > 0 ? SH::EB : 30;
  static constexpr int RAW = N + (N >> (PS > 20 ? 30 : PS));  // one pad word per E words
  static constexpr int BOX = N < 256 ? N : 256;   // rows per TMA box (hardware limit 256)
  static constexpr int NBOX = N / BOX;
  static constexpr int NPF = NBOX > 1 ? NBOX / 2 : 1;  // boxes of the first half
  static constexpr size_t BOXB = sizeof(cx<T>) * (size_t)BOX * B;
  // the odd-row boxes of the parity mode (float32 rows only) are two complex
  // wider (pitch B + 2)
  static constexpr size_t XB = sizeof(cx<T>) * (size_t)BOX * (sizeof(T) == 4 ? B + 2 : B) * (NBOX - NPF);
  // exchange buffer of W-byte words (whole complex values, or real words in
  // the FPF split exchange), column stride S: B columns x QW / B threads per
  // wavefront cover every bank once
  static constexpr int W = FPF ? (int)sizeof(T) : (int)sizeof(cx<T>);
  static constexpr int QW = 128 / W;
  static constexpr int S = ((RAW + QW - 1) / QW) * QW + (QW / B > 0 ? QW / B : 1);
  static constexpr size_t XS = (size_t)W * B * S;
  static constexpr size_t PF = FPF ? BOXB * NPF + XB : BOXB * NPF;  // FPF: both halves (odd rows wider)
  static constexpr size_t X = FPF ? XS : (XS > XB ? XS : XB);
  static constexpr bool SPLIT = FPF;
  static constexpr int TW = SH::TW > 0 ? SH::TW : 1;
  static constexpr size_t SMEM = PF + X + sizeof(cx<T>) * TW + 64;
  static constexpr bool OK = SH::P > 1 && SMEM * MINB <= 227 * 1024 && THREADS <= 1024 &&
                             B * sizeof(cx<T>) <= 256 && (NBOX == 1 || 2 * NPF == NBOX) && SH::TPT % 2 == 0;
};

constexpr int kTmaTab = 16;  // block pointers of the two-level stores (p <= 16)

struct TmaColParams {
  void* data;            // column base (element 0 of group 0, column 0)
  const void* tw;        // pass tables (fft_engine.cuh layout)
  long long ntiles;
  int tpg;               // tiles per group
  int cols;              // columns per group
  long long rstride;     // elements between the rows of a column
  long long gstride;     // elements between groups
  int evict_first;       // L2 priority of the loads: 1 evict_first, 0 evict_normal (rows not 128-byte aligned)
  unsigned long long* ticket;  // dynamic tile order (zeroed before the launch), or null: round robin
  int parity;            // rows 8 bytes off 16-byte alignment on odd rows: even rows through `map`, odd
                         // rows through `map_odd`, whose boxes start on the aligned address before the
                         // row segment and are one complex wider on each side (pitch B + 2, data at +1)
  int load4;             // 4D map (2*cols, rows_in, rows_out, groups): row r at (r mod rows_in, r >> lin_shift)
  int lin_shift;         // log2(rows_in)
  int brows;             // rows per box in the 4D mode (<= rows_in, <= 256)
  int sin_shift;         // TWO stores: log2(rows per table block)
  long long sin_stride;  // TWO stores: elements between the rows of a block
  long long sgstride;    // TWO stores: elements between groups
  void* tab[kTmaTab];    // TWO stores: block base pointers
  int tma_store;         // FPF, in place through `map` (parity 0): the first half of each output tile leaves
                         // through TMA boxes staged in the drained exchange buffer, the rest through STG
};

template <typename T, int L, bool INV, int NB, bool TWO, bool FPF>
__global__ void __launch_bounds__(TmaColCfg<T, L, NB, FPF>::THREADS, TmaColCfg<T, L, NB, FPF>::MINB)
col_tma_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap map_odd,
               const TmaColParams prm) {
  using TC = TmaColCfg<T, L, NB, FPF>;
  using SH = Shape<L>;
  using ST = Stockham<T, L, INV, TC::S, TC::PS, TC::SPLIT, 0, true>;
  constexpr int E = SH::E, TPT = SH::TPT, B = TC::B, BOX = TC::BOX, N = SH::N;
  static_assert(TC::OK, "unsupported column-kernel shape for the TMA path");
  static_assert(BOX % TPT == 0, "a thread's operand rows tt + TPT kk stay inside box (TPT kk) / BOX");

  extern __shared__ __align__(1024) unsigned char smem_tc[];
  cx<T>* pf = reinterpret_cast<cx<T>*>(smem_tc);                       // boxes [0, NPF)
  unsigned char* xs = smem_tc + TC::PF;                                // exchange buffer
  // boxes [NPF, NBOX): behind the first half (FPF) or in the exchange buffer
  cx<T>* xb = FPF ? pf + (size_t)TC::BOX * B * TC::NPF : reinterpret_cast<cx<T>*>(xs);
  cx<T>* s_tw = reinterpret_cast<cx<T>*>(xs + TC::X);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(s_tw) + sizeof(cx<T>) * TC::TW);

  const int t = threadIdx.x;
  const int b = t % B, tt = t / B;
  if (t == 0) {
    mbar_init(bar + 0, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const cx<T>* g = reinterpret_cast<const cx<T>*>(prm.tw);
    for (int k = t; k < SH::TW; k += TC::THREADS) s_tw[k] = g[k];
  }
  __syncthreads();

  const long long step = gridDim.x;
  const uint64_t pol = prm.evict_first ? policy_evict_first() : policy_evict_normal();
  auto coords = [&](long long tile, int& grp, int& c0) {
    grp = (int)(tile / prm.tpg);
    c0 = (int)(tile % prm.tpg) * B;
  };
  // tile order: a ticket counter keeps the tiles in flight within a window of
  // ~gridDim consecutive tiles (DRAM page locality of neighbours, as in
  // col_fft_kernel); round robin without one
  const bool dyn = prm.ticket != nullptr;
  __shared__ long long s_tk[2];
  long long cur = blockIdx.x;
  if (dyn) {
    if (t == 0) {
      cur = (long long)atomicAdd(prm.ticket, 1ull);
      s_tk[0] = (long long)atomicAdd(prm.ticket, 1ull);
      s_tk[1] = cur;
    }
    __syncthreads();
    cur = s_tk[1];
  }
  // half h of tile i: boxes [0, NPF) into the prefetch region, the rest into the exchange buffer
  // Parity mode: half 0 = the even rows (map, row index r/2), half 1 = the odd
  // rows (map_odd); a thread's operand rows tt + TPT kk all share tt's parity.
  auto load_half = [&](long long tile, int h) {
    int grp, c0;
    coords(tile, grp, c0);
    const int q0 = h ? TC::NPF : 0, q1 = h ? TC::NBOX : TC::NPF;
    if (q1 <= q0) return;
    fence_async_shared();  // the CTA's generic accesses to the region are ordered before the TMA writes
    const bool par = sizeof(T) == 4 && prm.parity;  // float64 rows are always 16-byte aligned
    const int pitch = (par && h) ? B + 2 : B;
    mbar_arrive_tx(bar + h, (unsigned)(sizeof(cx<T>) * (size_t)BOX * pitch * (q1 - q0)));
    cx<T>* dst = h ? xb : pf;
    if (prm.load4) {  // two-level rows: boxes of brows rows, never across a block
      const int r0 = q0 * BOX, r1 = q1 * BOX, rmask = (1 << prm.lin_shift) - 1;
      for (int r = r0; r < r1; r += prm.brows)
        tma_load4(dst + (size_t)(r - r0) * B, &map, 2 * c0, r & rmask, r >> prm.lin_shift, grp, bar + h, pol);
      return;
    }
    for (int q = q0; q < q1; ++q) {
      if (par)
        tma_load3(dst + (size_t)(q - q0) * BOX * pitch, h ? &map_odd : &map, 2 * c0, (q - q0) * BOX, grp, bar + h,
                  pol);
      else
        tma_load3(dst + (size_t)(q - q0) * BOX * B, &map, 2 * c0, q * BOX, grp, bar + h, pol);
    }
  };
  auto operand = [&](int kk) -> cx<T> {  // row tt + TPT kk; kk is a compile-time constant after unrolling
    const int r = tt + TPT * kk;
    if (sizeof(T) == 4 && prm.parity) return (tt & 1) ? xb[(r >> 1) * (B + 2) + 1 + b] : pf[(r >> 1) * B + b];
    return (TPT * kk) / BOX < TC::NPF ? pf[r * B + b] : xb[(r - TC::NPF * BOX) * B + b];
  };

  if (t == 0 && cur < prm.ntiles) {
    load_half(cur, 0);
    load_half(cur, 1);
  }
  for (long long i = 0; cur < prm.ntiles; ++i) {
    const long long nxt = dyn ? s_tk[i & 1] : cur + step;
    const unsigned par = (unsigned)(i & 1);
    mbar_wait(bar + 0, par);
    if (TC::NBOX > TC::NPF) mbar_wait(bar + 1, par);
    cx<T> v[E];
#pragma unroll
    for (int kk = 0; kk < E; ++kk) v[SH::in_slot(kk)] = operand(kk);
    // the previous tile's TMA store has read its staging (the exchange buffer)
    if (FPF && !TWO && t == 0 && prm.tma_store) bulk_wait_read0();
    __syncthreads();  // every operand read: both halves may be overwritten
    unsigned long long tk = 0;
    if (t == 0) {
      // the next tile's boxes first, then the ticket after next: its atomic
      // returns while pass 0 computes (storing it right away would hold the
      // loads behind the atomic's round trip)
      if (nxt < prm.ntiles) {
        load_half(nxt, 0);
        if (FPF) load_half(nxt, 1);
      }
      if (dyn) tk = atomicAdd(prm.ticket, 1ull);
    }
    ST::first(v, tt, s_tw);
    if (t == 0 && dyn) s_tk[(i + 1) & 1] = (long long)tk;  // read next iteration, after the exchange barriers
    auto hook = [&] {  // the last exchange has drained the buffer
      if (!FPF && t == 0 && nxt < prm.ntiles) load_half(nxt, 1);
    };
    ST::finish(xs, v, tt, b, s_tw, hook);
    int grp, c0;
    coords(cur, grp, c0);
    if constexpr (FPF && !TWO) {
      if (prm.tma_store) {
        // rows [0, N/2): stage them as the [row][B] box layout in the drained
        // exchange buffer and store them with N/2/BOX TMA boxes; the other half
        // leaves from registers below
        cx<T>* ob = reinterpret_cast<cx<T>*>(xs);
#pragma unroll
        for (int u = 0; u < E / SH::RL; ++u)
#pragma unroll
          for (int m = 0; m < SH::RL; ++m)
            if ((TPT * u + m * (N / SH::RL)) < N / 2) ob[SH::out_elem(tt, u, m) * B + b] = v[u * SH::RL + m];
        fence_async_shared();
        __syncthreads();
        if (t == 0) {
          for (int q = 0; q < TC::NPF; ++q) tma_store3(&map, 2 * c0, q * BOX, grp, ob + (size_t)q * BOX * B, pol);
          bulk_commit();
        }
        if (c0 + b < prm.cols) {
          cx<T>* col = reinterpret_cast<cx<T>*>(prm.data) + (long long)grp * prm.gstride + (c0 + b);
          const unsigned rs = (unsigned)prm.rstride;
#pragma unroll
          for (int u = 0; u < E / SH::RL; ++u)
#pragma unroll
            for (int m = 0; m < SH::RL; ++m)
              if ((TPT * u + m * (N / SH::RL)) >= N / 2) col[(unsigned)SH::out_elem(tt, u, m) * rs] = v[u * SH::RL + m];
        }
        cur = nxt;
        continue;
      }
    }
    if (TWO && c0 + b < prm.cols) {
      const long long cofs = (long long)grp * prm.sgstride + (c0 + b);
      const unsigned msk = (1u << prm.sin_shift) - 1u, ss = (unsigned)prm.sin_stride;
#pragma unroll
      for (int u = 0; u < E / SH::RL; ++u)
#pragma unroll
        for (int m = 0; m < SH::RL; ++m) {
          const unsigned r = (unsigned)SH::out_elem(tt, u, m);
          cx<T>* a = reinterpret_cast<cx<T>*>(prm.tab[r >> prm.sin_shift]) + cofs + (r & msk) * ss;
          *a = v[u * SH::RL + m];
        }
    } else if (c0 + b < prm.cols) {
      cx<T>* col = reinterpret_cast<cx<T>*>(prm.data) + (long long)grp * prm.gstride + (c0 + b);
      const unsigned rs = (unsigned)prm.rstride;
#pragma unroll
      for (int u = 0; u < E / SH::RL; ++u)
#pragma unroll
        for (int m = 0; m < SH::RL; ++m) {
          cx<T>* a = col + (unsigned)SH::out_elem(tt, u, m) * rs;
#if TFFFT_COL_STORE == 1
          st_hint(a, v[u * SH::RL + m], pol);  // the loads' L2 policy on the stores too
#elif TFFFT_COL_STORE == 2
          st_cs(a, v[u * SH::RL + m]);  // streaming (evict-first) stores
#else
          *a = v[u * SH::RL + m];
#endif
        }
    }
    cur = nxt;
  }
  if (FPF && !TWO && t == 0 && prm.tma_store) bulk_wait0();  // the staging must outlive the last TMA store
}

// lengths with a TMA-fed column kernel
__host__ __device__ constexpr bool col_tma_supported(int L) { return L == 9 || L == 10; }

template <typename T>
cudaError_t launch_col_tma(int L, bool inv, bool wide, bool two, const CUtensorMap& map, const CUtensorMap& map_odd,
                           const TmaColParams& p, cudaStream_t s);
// the full-prefetch variant is the default (TFFFT_TMA_FPF=0 disables it, launch_col_tma)
// columns per tile (the box width) of the TMA column kernel
template <typename T>
int col_tma_width(int L, bool wide);

}  // namespace tffft
