// Warp-per-column, warp-specialised column c2c for sm_100a (1024-point columns,
// and 512-point columns two per warp: stages 1b / 1b' / 3 / 3' at p = 1, and
// the two-level passes at p > 1 -- band-redirected stores, landing-band loads).
//
// col_tma_kernel (col_tma.cuh) spreads every column over all warps of the CTA
// (thread = 4 rows x 8 columns slices), so the operand read, both FFT passes,
// the shared-memory exchange and the stores run in lock step behind CTA
// barriers: while the eight warps store, the FP64 pipe idles, and the other
// way round (profiles/r02/stage3_full.txt: exchange barriers 15% and the store
// phase 19% of the stall samples).  Here a column belongs to ONE warp:
//
//   consumer warps: warp w owns column w of the tile; lane tt holds rows
//       tt + 32 kk (512 points: two columns per warp, a half-warp each, a
//       tile row being two 128-byte sub-boxes side by side).  Operands come
//       out of the TMA landing ring, the single Stockham exchange runs in a
//       warp-private buffer behind __syncwarp, the results go into a shared
//       output stage.  No CTA barrier in the loop: the warps drift apart, so
//       one warp's FP64 pass overlaps another's shared-memory traffic.
//   producer (one thread of a four-warp group behind the consumers): owns
//       all global traffic.  It takes tiles from the ticket counter, refills
//       each 256-row box of the landing ring as soon as every consumer has
//       read it (cp.async.bulk.tensor loads), and sends every finished output
//       quarter with a cp.async.bulk.tensor store.
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
  static constexpr int N = SH::N, E = SH::E, TPT = SH::TPT;
  // columns per warp (1024 points: one; 512 points: two, a half-warp each) and 128-byte sub-boxes side by side
  // in a row of the tile (512 points: two -- 256-byte row visits, as col_tma_kernel's 16 float64 columns)
  static constexpr int CPW = 32 / TPT, NSIDE = CPW;
  static constexpr int BS = 128 / (int)sizeof(cx<T>);  // columns of one sub-box
  static constexpr int B = NSIDE * BS;                 // columns per tile
  static constexpr int WARPS = B / CPW;                // consumer warps: 8 (float64), 16 (float32)
  // WARPS consumer warps + one producer warpgroup (four warps, one active thread).  A sub-partition holds 16 K
  // registers and ends up with two (four) consumer warps and one producer warp: the CTA starts with the
  // uniform count of its launch bound and the roles trade registers with setmaxnreg (whole warpgroups).
  static constexpr int THREADS = 32 * (WARPS + 4);
  // setmaxnreg.inc only hands out what the producers' setmaxnreg.dec released:
  // float64 128 x (168 - 40) = 256 x (232 - 168); float32 128 x (96 - 24) >= 512 x (112 - 96)
  static constexpr int CREG = sizeof(T) == 8 ? 232 : 112;  // consumers, after setmaxnreg.inc
  static constexpr int PREG = sizeof(T) == 8 ? 40 : 24;    // producer warpgroup, after setmaxnreg.dec
  static constexpr int BOX = 256, NQ = N / BOX;        // rows per TMA box (hardware limit 256), row blocks per tile
  static constexpr int NBOX = NQ * NSIDE;              // ring boxes: box (q, side) at q NSIDE + side
  static constexpr size_t BOXB = (size_t)BOX * 128;
  static constexpr size_t RING = BOXB * NBOX;
  static constexpr int KPB = E / NQ;                   // operands a lane takes from one row block
  static constexpr int NROUND = 4, OROWS = N / NROUND; // output rounds; slot = NSIDE sub-boxes of OROWS rows
  static constexpr size_t SLOTB = (size_t)NSIDE * OROWS * 128;
  static constexpr int PS = SH::EB;                    // one pad word per E words
  static constexpr int S = N + (N >> PS);              // words per column of the exchange buffer
  static constexpr size_t XS = sizeof(T) * (size_t)B * S;
  static constexpr int TW = SH::TW > 0 ? SH::TW : 1;
  static constexpr int NBAR = 2 * NBOX + 5;
  static constexpr size_t SMEM = RING + XS + sizeof(cx<T>) * TW + 8 * NBAR + 16;
  static constexpr bool OK = (TPT == 32 || TPT == 16) && SH::P == 2 && NBOX == 4 && 2 * SLOTB <= XS &&
                             SMEM <= 227 * 1024 && E % NQ == 0 && SH::R0 == E && E % NROUND == 0 &&
                             (TPT * KPB) % 8 == 0 && OROWS % 32 == 0;
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
  constexpr int E = SH::E, B = WC::B, BOX = WC::BOX, NBOX = WC::NBOX, NQ = WC::NQ, NSIDE = WC::NSIDE, KPB = WC::KPB;
  constexpr int TPT = WC::TPT, WARPS = WC::WARPS, NROUND = WC::NROUND, OROWS = WC::OROWS, RL = SH::RL;
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
      mbar_init(empty + q, WARPS / NSIDE);  // the warps whose columns lie in this side of the tile
    }
    mbar_init(xdrained, WARPS);
    for (int s = 0; s < 2; ++s) {
      mbar_init(ofull + s, WARPS);
      mbar_init(oempty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const cx<T>* g = reinterpret_cast<const cx<T>*>(prm.tw);
    for (int k = t; k < SH::TW; k += WC::THREADS) s_tw[k] = g[k];
  }
  __syncthreads();

  if (w >= WARPS) {
    // ---------------- producer: every global access of the CTA ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(WC::PREG));
    if (t != 32 * WARPS) return;
    const uint64_t pol = prm.evict_first ? policy_evict_first() : policy_evict_normal();
    const bool dyn = prm.ticket != nullptr;
    const long long step = gridDim.x;
    long long cur = dyn ? (long long)atomicAdd(prm.ticket, 1ull) : (long long)blockIdx.x;
    long long nxt = dyn ? (long long)atomicAdd(prm.ticket, 1ull) : cur + step;
    auto load_box = [&](long long tile, int bx) {  // box (q, side): rows [256 q, 256 q + 256), sub-box `side`
      const int q = bx / NSIDE, side = bx % NSIDE;
      const int grp = (int)(tile / prm.tpg), x0 = 2 * ((int)(tile % prm.tpg) * B + side * WC::BS);
      fence_async_shared();
      mbar_arrive_tx(full + bx, (unsigned)WC::BOXB);
      unsigned char* dst = ring + (size_t)bx * WC::BOXB;
      if (prm.load4) {  // two-level rows: sub-boxes never cross a block
        const int rmask = (1 << prm.lin_shift) - 1;
        for (int r = q * BOX; r < (q + 1) * BOX; r += prm.lbrows)
          tma_load4(dst + (size_t)(r - q * BOX) * 128, &maps.ld, x0, r & rmask, r >> prm.lin_shift, grp, full + bx, pol);
      } else {
        tma_load3(dst, &maps.ld, x0, q * BOX, grp, full + bx, pol);
      }
    };
    // the output stage starts empty
    mbar_arrive(oempty + 0);
    mbar_arrive(oempty + 1);
    s_flag[0] = cur < prm.ntiles;
    if (cur >= prm.ntiles) {
      for (int side = 0; side < NSIDE; ++side) mbar_arrive(full + side);
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
        mbar_wait(empty + q, par);  // every warp of the side holds its operands of box q
        if (more) load_box(nxt, q);
        else if (q < NSIDE) mbar_arrive(full + q);  // wake the consumers (row block 0 of each side): no further tile
      }
      const int grp = (int)(cur / prm.tpg), c0 = (int)(cur % prm.tpg) * B;
#pragma unroll
      for (int qq = 0; qq < NROUND; ++qq) {
        const int s = qq & 1;
        mbar_wait(ofull + s, (unsigned)(((it * (NROUND / 2)) + (qq >> 1)) & 1u));
#pragma unroll
        for (int side = 0; side < NSIDE; ++side) {
          const unsigned char* src = xs + (size_t)s * WC::SLOTB + (size_t)side * OROWS * 128;
          const int x0 = 2 * (c0 + side * WC::BS);
          if (prm.nst > 1) {  // block redirect: row r goes to row (r mod block rows) of st[r / block rows]
            const int smask = (1 << prm.sst_shift) - 1;
            for (int r = qq * OROWS; r < (qq + 1) * OROWS; r += prm.sbrows)
              tma_store3(&maps.st[r >> prm.sst_shift], x0, r & smask, grp, src + (size_t)(r - qq * OROWS) * 128, pol);
          } else {
            tma_store3(&maps.st[0], x0, qq * OROWS, grp, src, pol);
          }
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

  // ---------------- consumers: warp w owns columns w CPW .. of every tile ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(WC::CREG));
  const int tl = tt % TPT;                    // lane within its transform
  const int c = w * WC::CPW + tt / TPT;       // this lane's column of the tile
  const int cb = c * (int)sizeof(cx<T>);      // byte offset of the column in a tile row
  const int side = cb >> 7;
  // chunk of the column in a row congruent to tl mod 8 (128-byte swizzle)
  const int lane_ofs = tl * 128 + ((((cb & 127) >> 4) ^ (tl & 7)) << 4) + (cb & 15);
  unsigned oe = 0;  // phases of oempty[s] consumed (the same count for both slots)
  for (unsigned it = 0;; ++it) {
    const unsigned par = it & 1u;
    cx<T> v[E];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int bx = q * NSIDE + side;
      mbar_wait(full + bx, par);
      if (q == 0 && !s_flag[par]) return;
      const unsigned char* bxp = ring + (size_t)bx * WC::BOXB + lane_ofs;
#pragma unroll
      for (int k = 0; k < KPB; ++k)  // row tl + TPT (q KPB + k) = row block q, row tl + TPT k
        v[SH::in_slot(q * KPB + k)] = *reinterpret_cast<const cx<T>*>(bxp + (size_t)k * TPT * 128);
      __syncwarp();
      if (tt == 0) mbar_arrive(empty + bx);
    }
    ST::first(v, tl, s_tw);
    // the exchange buffer doubles as the output stage: both slots read out
    mbar_wait(oempty + 0, oe & 1u);
    mbar_wait(oempty + 1, oe & 1u);
    ++oe;
    auto hook = [&] {  // this warp's last exchange has drained its region
      __syncwarp();
      if (tt == 0) mbar_arrive(xdrained);
    };
    ST::finish(xs, v, tl, c, s_tw, hook);
    mbar_wait(xdrained, par);  // every warp is out of the exchange buffer
#pragma unroll
    for (int qq = 0; qq < NROUND; ++qq) {
      const int s = qq & 1;
      if (qq >= 2) {
        mbar_wait(oempty + s, oe & 1u);
        if (s == 1) ++oe;
      }
      unsigned char* ob = xs + (size_t)s * WC::SLOTB + (size_t)side * OROWS * 128 + lane_ofs;
      // output row tl + TPT u + (N / RL) m in v[u RL + m]: the rows of round qq are m in [qq RL / 4, (qq + 1) RL / 4)
#pragma unroll
      for (int u = 0; u < E / RL; ++u)
#pragma unroll
        for (int m = 0; m < RL / NROUND; ++m)
          *reinterpret_cast<cx<T>*>(ob + (size_t)(TPT * u + (SH::N / RL) * m) * 128) = v[u * RL + qq * (RL / NROUND) + m];
      fence_async_shared();  // the TMA store reads the stage through the async proxy
      __syncwarp();
      if (tt == 0) mbar_arrive(ofull + s);
    }
  }
}

// 512- and 1024-point columns; 2048-point columns as 2 x 1024 (col_wpc2.cuh)
__host__ __device__ constexpr bool col_wpc_supported(int L) { return L == 9 || L == 10 || L == 11; }

template <typename T>
cudaError_t launch_col_wpc(int L, bool inv, const WpcMaps& maps, const WpcParams& p, cudaStream_t s);
// columns per tile (the box width; 0: no kernel for this length)
template <typename T>
int col_wpc_width(int L);

}  // namespace tffft
