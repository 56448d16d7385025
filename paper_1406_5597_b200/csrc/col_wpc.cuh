// Warp-per-column, warp-specialised column c2c for sm_100a (1024-point columns:
// stages 1b / 1b' / 3 / 3' at p = 1, and the two-level stage-1b / 1b' passes at
// p > 1 -- band-redirected stores, landing-band loads).
//
// col_tma_kernel (col_tma.cuh) spreads every column over all warps of the CTA
// (thread = 4 rows x 8 columns slices), so the operand read, both FFT passes,
// the shared-memory exchange and the stores run in lock step behind CTA
// barriers: while the eight warps store, the FP64 pipe idles, and the other
// way round (profiles/r02/stage3_full.txt: exchange barriers 15% and the store
// phase 19% of the stall samples).  Here a column belongs to ONE warp:
//
//   warps 0..B-1 (consumers): warp w owns column w of the tile; lane tt holds
//       rows tt + 32 kk.  Operands come out of the TMA landing ring, the single
//       Stockham exchange runs in a warp-private buffer behind __syncwarp, the
//       results go into a shared output stage.  No CTA barrier in the loop:
//       the warps drift apart, so one warp's FP64 pass overlaps another's
//       shared-memory traffic.
//   warp B (producer, one thread of a four-warp group): owns all global traffic.  It takes tiles
//       from the ticket counter, refills each 256-row box of the landing ring
//       as soon as every consumer has read it (cp.async.bulk.tensor loads), and
//       sends every finished output quarter with a cp.async.bulk.tensor store.
//
// The boxes use the 128-byte TMA swizzle: row r of a box keeps its 16-byte
// chunk c at chunk position c ^ (r mod 8).  Lane tt reads rows congruent to
// tt mod 8, so the eight lanes of a shared-memory wavefront hit eight different
// chunks: a column (128-byte row pitch) reads and writes without bank
// conflicts, which is what lets one warp own a column at all.
//
// Shared memory (float64, 1024 points): landing ring 4 x 32 KB, exchange
// 8 x 8.25 KB of 8-byte words (re round, then im round); the output stage
// (two 32 KB quarters) aliases the exchange buffer, which is idle from the last
// exchange of a tile to the first of the next.  Hand-offs are mbarriers:
//   full[q]  / empty[q]   landing box q: TMA bytes landed / all warps read it
//   xdrained              every warp finished its exchange (stage may be written)
//   ofull[s] / oempty[s]  output quarter slot s written / read out by the TMA store
// p > 1: only the producer changes.  Loads may go through a 4D map over the
// landing bands (cols, rows within a block, block, group) in sub-boxes that
// never cross a block; stores may go through one map per destination block
// (the forward band redirects: self band to landing[rank], peer bands to
// staging or straight into the peer's landing buffer) -- the reference's
// strided exchange datatype (exchange.py:114-121) applied by the TMA boxes.
// Same engine, twiddles and arithmetic as col_tma_kernel: results are bitwise
// identical (tests/test_gpu_parity.py::test_wpc_column_kernel_bitwise).
//
// Replaces the strided column loops of the reference (kernels.py:176-200 via
// dfft.py:170-171, 196-197; the n1 pass of kernels.py:262-303).
#pragma once
#include <cuda.h>

#include "col_tma.cuh"

namespace tffft {

__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read2() { asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); }

template <typename T, int L>
struct WpcCfg {
  using SH = Shape<L>;
  static constexpr int N = SH::N, E = SH::E;
  static constexpr int B = 128 / (int)sizeof(cx<T>);  // columns per tile: 128-byte rows
  // B consumer warps + one producer warpgroup (four warps, one active thread).  A sub-partition holds 16 K
  // registers and ends up with two (four) consumer warps and one producer warp: the CTA starts with the
  // uniform count of its launch bound and the roles trade registers with setmaxnreg (whole warpgroups).
  static constexpr int THREADS = 32 * (B + 4);
  // setmaxnreg.inc only hands out what the producers' setmaxnreg.dec released:
  // float64 128 x (168 - 40) = 256 x (232 - 168); float32 128 x (96 - 24) >= 512 x (112 - 96)
  static constexpr int CREG = sizeof(T) == 8 ? 232 : 112;  // consumers, after setmaxnreg.inc
  static constexpr int PREG = sizeof(T) == 8 ? 40 : 24;    // producer warpgroup, after setmaxnreg.dec
  static constexpr int BOX = 256, NBOX = N / BOX;     // rows per TMA box (hardware limit 256)
  static constexpr size_t BOXB = (size_t)BOX * 128;
  static constexpr size_t RING = BOXB * NBOX;
  static constexpr int PS = SH::EB;                   // one pad word per E words
  static constexpr int S = N + (N >> PS);             // words per warp-private exchange region
  static constexpr size_t XS = sizeof(T) * (size_t)B * S;
  static constexpr int TW = SH::TW > 0 ? SH::TW : 1;
  static constexpr int NBAR = 2 * NBOX + 5;
  static constexpr size_t SMEM = RING + XS + sizeof(cx<T>) * TW + 8 * NBAR + 16;
  static constexpr bool OK = SH::TPT == 32 && SH::P == 2 && NBOX >= 2 && 2 * BOXB <= XS && SMEM <= 227 * 1024 &&
                             E % NBOX == 0 && SH::RL == E && SH::R0 == E;
};

constexpr int kWpcMaps = 16;  // store maps (destination blocks, p <= 16)

struct WpcParams {
  const void* tw;              // pass tables (fft_engine.cuh layout)
  const void* tw2;             // 2 x 1024 kernel (col_wpc2.cuh): exp(-2 pi i k / 2048), k < 1024
  long long ntiles;
  int tpg;                     // tiles per group
  int evict_first;             // L2 priority of the loads and stores
  unsigned long long* ticket;  // dynamic tile order (zeroed before the launch), or null: round robin
  int load4;                   // 4D load map (2*cols, rows_in, blocks, groups): row r at (r mod rows_in, r >> lin_shift)
  int lin_shift;               // log2(rows_in)
  int lbrows;                  // rows per load sub-box (divides 256, multiple of 8, <= rows_in)
  int nst;                     // store maps: 1 = uniform (row r of the column at row r of st[0])
  int sst_shift;               // nst > 1: log2(rows per destination block); row r -> st[r >> sst_shift]
  int sbrows;                  // rows per store sub-box (divides 256, multiple of 8, <= rows per block)
};

// tensor maps of one launch: every box is B columns x (sub-box rows), 128-byte swizzle
struct alignas(64) WpcMaps {
  CUtensorMap ld;
  CUtensorMap st[kWpcMaps];
};

template <typename T, int L, bool INV>
__global__ void __launch_bounds__(WpcCfg<T, L>::THREADS, 1)
col_wpc_kernel(const __grid_constant__ WpcMaps maps, const WpcParams prm) {
  using WC = WpcCfg<T, L>;
  using SH = Shape<L>;
  using ST = Stockham<T, L, INV, WC::S, WC::PS, true, 32, true>;
  constexpr int E = SH::E, B = WC::B, BOX = WC::BOX, NBOX = WC::NBOX, KPB = E / NBOX;  // operands per box
  static_assert(WC::OK, "unsupported shape for the warp-per-column kernel");

  extern __shared__ __align__(1024) unsigned char smem_wc[];
  unsigned char* ring = smem_wc;                 // NBOX swizzled boxes [row][128 B]
  unsigned char* xs = smem_wc + WC::RING;        // exchange buffer; output stage slots 0/1 alias it
  cx<T>* s_tw = reinterpret_cast<cx<T>*>(xs + WC::XS);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(s_tw) + sizeof(cx<T>) * WC::TW);
  uint64_t* full = bar;                // [NBOX]
  uint64_t* empty = bar + NBOX;        // [NBOX]
  uint64_t* xdrained = bar + 2 * NBOX;
  uint64_t* ofull = bar + 2 * NBOX + 1;   // [2]
  uint64_t* oempty = bar + 2 * NBOX + 3;  // [2]
  volatile int* s_flag = reinterpret_cast<volatile int*>(bar + WC::NBAR);  // [2]: tile of this parity exists

  const int t = threadIdx.x, w = t >> 5, tt = t & 31;
  if (t == 0) {
    for (int q = 0; q < NBOX; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, B);
    }
    mbar_init(xdrained, B);
    for (int s = 0; s < 2; ++s) {
      mbar_init(ofull + s, B);
      mbar_init(oempty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const cx<T>* g = reinterpret_cast<const cx<T>*>(prm.tw);
    for (int k = t; k < SH::TW; k += WC::THREADS) s_tw[k] = g[k];
  }
  __syncthreads();

  if (w >= B) {
    // ---------------- producer: every global access of the CTA ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(WC::PREG));
    if (t != 32 * B) return;
    const uint64_t pol = prm.evict_first ? policy_evict_first() : policy_evict_normal();
    const bool dyn = prm.ticket != nullptr;
    const long long step = gridDim.x;
    long long cur = dyn ? (long long)atomicAdd(prm.ticket, 1ull) : (long long)blockIdx.x;
    long long nxt = dyn ? (long long)atomicAdd(prm.ticket, 1ull) : cur + step;
    auto load_box = [&](long long tile, int q) {
      const int grp = (int)(tile / prm.tpg), c0 = (int)(tile % prm.tpg) * B;
      fence_async_shared();
      mbar_arrive_tx(full + q, (unsigned)WC::BOXB);
      unsigned char* dst = ring + (size_t)q * WC::BOXB;
      if (prm.load4) {  // two-level rows: sub-boxes never cross a block
        const int rmask = (1 << prm.lin_shift) - 1;
        for (int r = q * BOX; r < (q + 1) * BOX; r += prm.lbrows)
          tma_load4(dst + (size_t)(r - q * BOX) * 128, &maps.ld, 2 * c0, r & rmask, r >> prm.lin_shift, grp, full + q,
                    pol);
      } else {
        tma_load3(dst, &maps.ld, 2 * c0, q * BOX, grp, full + q, pol);
      }
    };
    // the output stage starts empty
    mbar_arrive(oempty + 0);
    mbar_arrive(oempty + 1);
    s_flag[0] = cur < prm.ntiles;
    if (cur >= prm.ntiles) {
      mbar_arrive(full + 0);
      return;
    }
    for (int q = 0; q < NBOX; ++q) load_box(cur, q);
    for (unsigned it = 0;; ++it) {
      const unsigned par = it & 1u;
      // the ticket after next: its round trip hides behind this tile
      unsigned long long tk = 0;
      if (dyn) tk = atomicAdd(prm.ticket, 1ull);
      const bool more = nxt < prm.ntiles;
      s_flag[par ^ 1u] = more;
      for (int q = 0; q < NBOX; ++q) {
        mbar_wait(empty + q, par);  // every warp holds its operands of box q
        if (more) load_box(nxt, q);
        else if (q == 0) mbar_arrive(full + 0);  // wake the consumers: no further tile
      }
      const int grp = (int)(cur / prm.tpg), c0 = (int)(cur % prm.tpg) * B;
#pragma unroll
      for (int qq = 0; qq < NBOX; ++qq) {
        const int s = qq & 1;
        mbar_wait(ofull + s, (unsigned)(((it * (NBOX / 2)) + (qq >> 1)) & 1u));
        const unsigned char* src = xs + (size_t)s * WC::BOXB;
        if (prm.nst > 1) {  // block redirect: row r goes to row (r mod block rows) of st[r / block rows]
          const int smask = (1 << prm.sst_shift) - 1;
          for (int r = qq * BOX; r < (qq + 1) * BOX; r += prm.sbrows)
            tma_store3(&maps.st[r >> prm.sst_shift], 2 * c0, r & smask, grp, src + (size_t)(r - qq * BOX) * 128, pol);
        } else {
          tma_store3(&maps.st[0], 2 * c0, qq * BOX, grp, src, pol);
        }
        bulk_commit();
        if (s == 1) {
          bulk_wait_read1();  // slot 0 has been read out
          mbar_arrive(oempty + 0);
          bulk_wait_read0();
          mbar_arrive(oempty + 1);
        }
      }
      if (!more) break;
      cur = nxt;
      nxt = dyn ? (long long)tk : nxt + step;
    }
    bulk_wait0();  // the stage must outlive the last TMA store
    return;
  }

  // ---------------- consumers: warp w owns column w of every tile ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(WC::CREG));
  // chunk of column w in a row congruent to tt mod 8 (128-byte swizzle)
  const int cchunk = (int)((w * sizeof(cx<T>)) >> 4) ^ (tt & 7);
  const int lane_ofs = tt * 128 + (cchunk << 4) + (int)((w * sizeof(cx<T>)) & 15);
  unsigned oe = 0;  // phases of oempty[s] consumed (the same count for both slots)
  for (unsigned it = 0;; ++it) {
    const unsigned par = it & 1u;
    cx<T> v[E];
#pragma unroll
    for (int q = 0; q < NBOX; ++q) {
      mbar_wait(full + q, par);
      if (q == 0 && !s_flag[par]) return;
      const unsigned char* bx = ring + (size_t)q * WC::BOXB + lane_ofs;
#pragma unroll
      for (int k = 0; k < KPB; ++k)  // row tt + 32 (q KPB + k) = box q, row tt + 32 k
        v[SH::in_slot(q * KPB + k)] = *reinterpret_cast<const cx<T>*>(bx + (size_t)k * 32 * 128);
      __syncwarp();
      if (tt == 0) mbar_arrive(empty + q);
    }
    ST::first(v, tt, s_tw);
    // the exchange buffer doubles as the output stage: both slots read out
    mbar_wait(oempty + 0, oe & 1u);
    mbar_wait(oempty + 1, oe & 1u);
    ++oe;
    auto hook = [&] {  // this warp's last exchange has drained its region
      __syncwarp();
      if (tt == 0) mbar_arrive(xdrained);
    };
    ST::finish(xs, v, tt, w, s_tw, hook);
    mbar_wait(xdrained, par);  // every warp is out of the exchange buffer
#pragma unroll
    for (int qq = 0; qq < NBOX; ++qq) {
      const int s = qq & 1;
      if (qq >= 2) {
        mbar_wait(oempty + s, oe & 1u);
        if (s == 1) ++oe;
      }
      unsigned char* ob = xs + (size_t)s * WC::BOXB + lane_ofs;
#pragma unroll
      for (int k = 0; k < KPB; ++k)  // output row tt + 32 m, m = qq KPB + k (RL = E: v[m])
        *reinterpret_cast<cx<T>*>(ob + (size_t)k * 32 * 128) = v[qq * KPB + k];
      fence_async_shared();  // the TMA store reads the stage through the async proxy
      __syncwarp();
      if (tt == 0) mbar_arrive(ofull + s);
    }
  }
}

// 1024-point columns; 2048-point columns as 2 x 1024 (col_wpc2.cuh)
__host__ __device__ constexpr bool col_wpc_supported(int L) { return L == 10 || L == 11; }

template <typename T>
cudaError_t launch_col_wpc(int L, bool inv, const WpcMaps& maps, const WpcParams& p, cudaStream_t s);
// columns per tile (the box width; 0: no kernel for this length)
template <typename T>
int col_wpc_width(int L);

}  // namespace tffft
