// 2048-point columns on the warp-per-column kernel: 2 x 1024 with the first
// half parked in tensor memory (sm_100a).
//
// A tile of 8 float64 columns x 2048 rows is 256 KB: it fits neither the
// register file (one warp per column holds 32 values per lane) nor shared
// memory next to the landing ring.  col_fft_kernel therefore runs 2048-point
// columns 4 at a time (64-byte row visits) and reaches 3.4-3.6 TB/s
// (profiles/r02s4/l11_before.txt).  Here the column splits by row parity
// (decimation in time):
//
//   E = FFT_1024(even rows), O = FFT_1024(odd rows),
//   X[k] = E[k] + w^k O[k],  X[k + 1024] = E[k] - w^k O[k],  w = exp(-+2 pi i / 2048)
//
// Both halves run through the col_wpc_kernel pipeline unchanged (swizzled TMA
// landing ring, one warp per column, warp-private exchange).  After the even
// half every lane holds E[k] for k = tt + 32 m -- exactly the k it will hold of
// O after the odd half -- so the 128 KB of E need no exchange, only a place to
// wait: each lane parks its 32 values in its own tensor-memory lane
// (tcgen05.st, 128 columns of 32 bits; TMEM is 256 KB per SM and otherwise
// idle in an FFT) and reads them back eight at a time while it combines
// (tcgen05.ld).  TMEM here is a register-spill parking lot next to the SM, not
// an MMA accumulator.  The 2048 output rows leave through the shared output
// stage in sixteen 128-row rounds over four 16 KB slots; the producer releases
// a slot two rounds after its store was issued, so no warp waits for a store
// that has only just been committed (with two 32 KB slots the consumers spent
// 19% of their stall samples in that rendezvous, profiles/r02s4/wpc2_2048.txt).
// Only the first eight rounds (X[k]) follow the combine directly: X[k + 1024]
// is parked in a second tensor-memory region and drained after the NEXT half's
// transform.  Both half-iterations then have the same length (one 1024-point
// transform plus eight output rounds), so the landing ring is refilled at an
// even pace instead of idling through sixteen rounds: 3.24 -> 2.93 ms per
// 17.2 GB stage-1b launch, 3.25 -> 3.14 ms for stage 3.  All 512 tensor-memory
// columns are in use (two regions of 128 KB).
//
// Loads go through a map with the row parity as its own dimension: (cols,
// parity, half rows, groups), or at p > 1 (cols, parity, half rows within a
// block, block, groups) over the landing bands.  Stores are col_wpc_kernel's
// (uniform, or one map per destination block).
//
// Replaces the strided column loops of the reference (kernels.py:176-200 via
// dfft.py:170-171, 196-197; the n1 pass of kernels.py:262-303) for n = 2048
// (BASELINE config 4: 2048^3 at p = 4, 8).
#pragma once
#include "col_wpc.cuh"

namespace tffft {

__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                          uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// tensor memory: allocation by one warp, 32x32b accesses (lane i of a warp <-> TMEM lane 32 (warp % 4) + i)
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* w) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
               ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* w) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* w) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
               ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* w) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
               : "r"(taddr)
               : "memory");
}

// 8 complex values <-> their 32-bit words
__device__ __forceinline__ void cx_to_words(const cx<double>* z, uint32_t* w) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[4 * k + 0] = (uint32_t)__double2loint(z[k].x);
    w[4 * k + 1] = (uint32_t)__double2hiint(z[k].x);
    w[4 * k + 2] = (uint32_t)__double2loint(z[k].y);
    w[4 * k + 3] = (uint32_t)__double2hiint(z[k].y);
  }
}
__device__ __forceinline__ void words_to_cx(const uint32_t* w, cx<double>* z) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    z[k].x = __hiloint2double((int)w[4 * k + 1], (int)w[4 * k + 0]);
    z[k].y = __hiloint2double((int)w[4 * k + 3], (int)w[4 * k + 2]);
  }
}
__device__ __forceinline__ void cx_to_words(const cx<float>* z, uint32_t* w) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[2 * k + 0] = __float_as_uint(z[k].x);
    w[2 * k + 1] = __float_as_uint(z[k].y);
  }
}
__device__ __forceinline__ void words_to_cx(const uint32_t* w, cx<float>* z) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    z[k].x = __uint_as_float(w[2 * k + 0]);
    z[k].y = __uint_as_float(w[2 * k + 1]);
  }
}
template <typename T>
__device__ __forceinline__ void tmem_park8(uint32_t taddr, const cx<T>* z) {
  uint32_t w[2 * sizeof(cx<T>)];
  cx_to_words(z, w);
  if constexpr (sizeof(T) == 8) tmem_st32(taddr, w); else tmem_st16(taddr, w);
}
template <typename T>
__device__ __forceinline__ void tmem_fetch8(uint32_t taddr, cx<T>* z) {
  uint32_t w[2 * sizeof(cx<T>)];
  if constexpr (sizeof(T) == 8) tmem_ld32(taddr, w); else tmem_ld16(taddr, w);
  tmem_wait_ld();
  words_to_cx(w, z);
}

template <typename T>
struct Wpc2Cfg {
  using WC = WpcCfg<T, 10>;
  static constexpr int NH = 1024;                                 // points per half
  static constexpr int W8 = 2 * (int)sizeof(cx<T>);               // 32-bit words of 8 complex values
  static constexpr int NW = 4 * W8;                               // words a lane parks (32 values)
  static constexpr int TREG = 256;                                // TMEM columns of one region: (consumer warps / 4) x NW
  static constexpr int TCOLS = 2 * TREG;                          // region A: E of this tile; region B: the second
                                                                  // output half of the previous tile
  static_assert((WC::B / 4) * NW == TREG, "tensor-memory columns");
  static constexpr size_t W2B = sizeof(cx<T>) * (size_t)NH;       // w^k, k < 1024
  static constexpr int NSLOT = 4, OROWS = 128;                    // output stage: slots of OROWS rows
  static constexpr size_t SLOTB = (size_t)OROWS * 128;
  static constexpr int NBAR = 2 * WC::NBOX + 1 + 2 * NSLOT;
  static constexpr size_t SMEM = WC::RING + WC::XS + sizeof(cx<T>) * WC::TW + W2B + 8 * NBAR + 32;
  static constexpr bool OK = WC::OK && SMEM <= 227 * 1024 && NSLOT * SLOTB <= WC::XS;
};

template <typename T, bool INV>
__global__ void __launch_bounds__(WpcCfg<T, 10>::THREADS, 1)
col_wpc2_kernel(const __grid_constant__ WpcMaps maps, const WpcParams prm) {
  using WC = WpcCfg<T, 10>;
  using W2 = Wpc2Cfg<T>;
  using SH = Shape<10>;
  using ST = Stockham<T, 10, INV, WC::S, WC::PS, true, 32, true>;
  constexpr int E = SH::E, B = WC::B, BOX = WC::BOX, NBOX = WC::NBOX, KPB = E / NBOX;
  constexpr int NSLOT = W2::NSLOT, OROWS = W2::OROWS, NR = 2 * W2::NH / OROWS, KPR = OROWS / 32;  // rounds, values per round
  static_assert(W2::OK && KPB == 8 && KPR == 4 && NR % (2 * NSLOT) == 0, "unsupported shape for the 2 x 1024 kernel");

  extern __shared__ __align__(1024) unsigned char smem_w2[];
  unsigned char* ring = smem_w2;
  unsigned char* xs = smem_w2 + WC::RING;
  cx<T>* s_tw = reinterpret_cast<cx<T>*>(xs + WC::XS);
  cx<T>* s_w2 = s_tw + WC::TW;  // exp(-2 pi i k / 2048), k < 1024
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(s_w2) + W2::W2B);
  uint64_t* full = bar;
  uint64_t* empty = bar + NBOX;
  uint64_t* xdrained = bar + 2 * NBOX;
  uint64_t* ofull = bar + 2 * NBOX + 1;           // [NSLOT]
  uint64_t* oempty = bar + 2 * NBOX + 1 + NSLOT;  // [NSLOT]
  volatile int* s_flag = reinterpret_cast<volatile int*>(bar + W2::NBAR);  // [2]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(const_cast<int*>(s_flag) + 2);

  const int t = threadIdx.x, w = t >> 5, tt = t & 31;
  if (t == 0) {
    for (int q = 0; q < NBOX; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, B);
    }
    mbar_init(xdrained, B);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(ofull + s, B);
      mbar_init(oempty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const cx<T>* g = reinterpret_cast<const cx<T>*>(prm.tw);
    for (int k = t; k < SH::TW; k += WC::THREADS) s_tw[k] = g[k];
    const cx<T>* g2 = reinterpret_cast<const cx<T>*>(prm.tw2);
    for (int k = t; k < W2::NH; k += WC::THREADS) s_w2[k] = g2[k];
  }
  if (w == 0) tmem_alloc(s_tmem, W2::TCOLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *s_tmem;

  if (w >= B) {
    // ---------------- producer ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(WC::PREG));
    if (t != 32 * B) return;
    const uint64_t pol = prm.evict_first ? policy_evict_first() : policy_evict_normal();
    const bool dyn = prm.ticket != nullptr;
    const long long step = gridDim.x;
    long long cur = dyn ? (long long)atomicAdd(prm.ticket, 1ull) : (long long)blockIdx.x;
    long long nxt = dyn ? (long long)atomicAdd(prm.ticket, 1ull) : cur + step;
    // box q of half h (row parity) of a tile: half rows [256 q, 256 q + 256)
    auto load_box = [&](long long tile, int h, int q) {
      const int grp = (int)(tile / prm.tpg), c0 = (int)(tile % prm.tpg) * B;
      fence_async_shared();
      mbar_arrive_tx(full + q, (unsigned)WC::BOXB);
      unsigned char* dst = ring + (size_t)q * WC::BOXB;
      if (prm.load4) {  // half rows within a block: sub-boxes never cross a block
        const int hshift = prm.lin_shift - 1, hmask = (1 << hshift) - 1;
        for (int r = q * BOX; r < (q + 1) * BOX; r += prm.lbrows)
          tma_load5(dst + (size_t)(r - q * BOX) * 128, &maps.ld, 2 * c0, h, r & hmask, r >> hshift, grp, full + q, pol);
      } else {
        tma_load4(dst, &maps.ld, 2 * c0, h, q * BOX, grp, full + q, pol);
      }
    };
    for (int s = 0; s < NSLOT; ++s) mbar_arrive(oempty + s);  // the output stage starts empty
    s_flag[0] = cur < prm.ntiles;
    if (cur >= prm.ntiles) {
      mbar_arrive(full + 0);
      return;
    }
    for (int q = 0; q < NBOX; ++q) load_box(cur, 0, q);
    unsigned long long tk = 0;
    unsigned pu[NSLOT] = {0, 0, 0, 0};  // uses of each output slot stored so far
    // eight 128-row rounds of one tile: rows [128 (8 half + r), ...) through slots r & 3, each slot released two
    // rounds after its store was issued
    auto store_half = [&](long long tile, int half) {
      const int grp = (int)(tile / prm.tpg), c0 = (int)(tile % prm.tpg) * B;
#pragma unroll 1
      for (int r8 = 0; r8 < NR / 2; ++r8) {
        const int rr = half * (NR / 2) + r8, s = r8 & (NSLOT - 1);
        mbar_wait(ofull + s, pu[s] & 1u);
        ++pu[s];
        const unsigned char* src = xs + (size_t)s * W2::SLOTB;
        if (prm.nst > 1) {
          const int smask = (1 << prm.sst_shift) - 1;
          for (int r = rr * OROWS; r < (rr + 1) * OROWS; r += prm.sbrows)
            tma_store3(&maps.st[r >> prm.sst_shift], 2 * c0, r & smask, grp, src + (size_t)(r - rr * OROWS) * 128, pol);
        } else {
          tma_store3(&maps.st[0], 2 * c0, rr * OROWS, grp, src, pol);
        }
        bulk_commit();
        if (r8 >= 2) {  // the store of two rounds ago has read its slot
          bulk_wait_read2();
          mbar_arrive(oempty + ((r8 - 2) & (NSLOT - 1)));
        }
      }
      bulk_wait_read1();
      mbar_arrive(oempty + ((NR / 2 - 2) & (NSLOT - 1)));
      bulk_wait_read0();
      mbar_arrive(oempty + ((NR / 2 - 1) & (NSLOT - 1)));
    };
    long long prev = -1;  // tile whose second output half is still parked in tensor memory
    for (unsigned it = 0;; ++it) {  // one iteration per half tile
      const unsigned par = it & 1u;
      const int h = (int)(it & 1u);
      if (dyn && h == 0) tk = atomicAdd(prm.ticket, 1ull);  // the ticket after next
      const bool more = h == 0 || nxt < prm.ntiles;
      s_flag[par ^ 1u] = more;
      for (int q = 0; q < NBOX; ++q) {
        mbar_wait(empty + q, par);
        if (more) load_box(h == 0 ? cur : nxt, h ^ 1, q);
        else if (q == 0) mbar_arrive(full + 0);
      }
      if (h == 0) {  // the consumers drain the previous tile's second half after this half's transform
        if (prev >= 0) store_half(prev, 1);
        continue;
      }
      store_half(cur, 0);
      prev = cur;
      if (!more) break;
      cur = nxt;
      nxt = dyn ? (long long)tk : nxt + step;
    }
    store_half(prev, 1);  // drained by the consumers on their way out
    bulk_wait0();
    return;
  }

  // ---------------- consumers ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(WC::CREG));
  const int cchunk = (int)((w * sizeof(cx<T>)) >> 4) ^ (tt & 7);
  const int lane_ofs = tt * 128 + (cchunk << 4) + (int)((w * sizeof(cx<T>)) & 15);
  // this lane's parking space: TMEM lane 32 (w % 4) + tt, NW columns from (w / 4) NW (region A), and the same
  // columns of region B
  const uint32_t taddr = tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * W2::NW);
  const uint32_t taddr_b = taddr + W2::TREG;
  unsigned oe[NSLOT] = {0, 0, 0, 0};  // phases of oempty[s] consumed
  unsigned U = 0;                     // uses of every slot begun so far (use j is released by phase j + 1)
  auto need = [&](int s, unsigned phase) {  // slot s has been read out for every use before `phase`
    while (oe[s] <= phase) {
      mbar_wait(oempty + s, oe[s] & 1u);
      ++oe[s];
    }
  };
  // the second output half of the previous tile, X[k + 1024], parked in region B: eight rounds to the stage
  auto drain = [&] {
    cx<T> d[8];
#pragma unroll
    for (int r8 = 0; r8 < NR / 2; ++r8) {
      const int s = r8 & (NSLOT - 1);
      need(s, U + r8 / NSLOT);
      if (r8 % 2 == 0) tmem_fetch8<T>(taddr_b + (r8 / 2) * W2::W8, d);
      unsigned char* ob = xs + (size_t)s * W2::SLOTB + lane_ofs;
#pragma unroll
      for (int k = 0; k < KPR; ++k) *reinterpret_cast<cx<T>*>(ob + (size_t)k * 32 * 128) = d[(r8 % 2) * KPR + k];
      fence_async_shared();
      __syncwarp();
      if (tt == 0) mbar_arrive(ofull + s);
    }
    U += NR / 2 / NSLOT;
  };
  bool pend = false;
  for (unsigned it = 0;; ++it) {
    const unsigned par = it & 1u;
    const int h = (int)(it & 1u);
    cx<T> v[E];
    bool stop = false;
#pragma unroll
    for (int q = 0; q < NBOX; ++q) {
      mbar_wait(full + q, par);
      if (q == 0 && !s_flag[par]) { stop = true; break; }
      const unsigned char* bx = ring + (size_t)q * WC::BOXB + lane_ofs;
#pragma unroll
      for (int k = 0; k < KPB; ++k)
        v[SH::in_slot(q * KPB + k)] = *reinterpret_cast<const cx<T>*>(bx + (size_t)k * 32 * 128);
      __syncwarp();
      if (tt == 0) mbar_arrive(empty + q);
    }
    if (stop) break;
    ST::first(v, tt, s_tw);
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) need(s, U);  // the exchange buffer doubles as the output stage
    auto hook = [&] {
      __syncwarp();
      if (tt == 0) mbar_arrive(xdrained);
    };
    ST::finish(xs, v, tt, w, s_tw, hook);
    if (h == 0) {  // E[tt + 32 m] waits in region A
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_park8<T>(taddr + c * W2::W8, v + 8 * c);
      tmem_wait_st();
      if (pend) {  // now the previous tile's second half, once every warp has left the exchange buffer
        mbar_wait(xdrained, par);
        drain();
        pend = false;
      }
      continue;
    }
    mbar_wait(xdrained, par);
    cx<T> e[8];
#pragma unroll
    for (int rr = 0; rr < NR / 2; ++rr) {  // rows tt + 32 m, m = KPR rr + k: X[k] = E + w^k O; E - w^k O goes to region B
      const int s = rr & (NSLOT - 1);
      need(s, U + rr / NSLOT);
      unsigned char* ob = xs + (size_t)s * W2::SLOTB + lane_ofs;
      if (rr % 2 == 0) tmem_fetch8<T>(taddr + (rr / 2) * W2::W8, e);
#pragma unroll
      for (int k = 0; k < KPR; ++k) {
        const int m = rr * KPR + k;
        const cx<T> ek = e[(rr % 2) * KPR + k];
        const cx<T> tw = ctw<INV>(v[m], s_w2[tt + 32 * m]);
        *reinterpret_cast<cx<T>*>(ob + (size_t)k * 32 * 128) = cadd(ek, tw);
        v[m] = csub(ek, tw);
      }
      fence_async_shared();
      __syncwarp();
      if (tt == 0) mbar_arrive(ofull + s);
    }
    U += NR / 2 / NSLOT;
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_park8<T>(taddr_b + c * W2::W8, v + 8 * c);
    tmem_wait_st();
    pend = true;
  }
  if (pend) drain();  // the last tile's second half (every warp left the exchange buffer long ago)
  // every consumer warp is done with tensor memory: warp 0 frees it
  tmem_fence_before();
  asm volatile("bar.sync 1, %0;" ::"n"(32 * WpcCfg<T, 10>::B) : "memory");
  if (w == 0) tmem_dealloc(tbase, W2::TCOLS);
}

}  // namespace tffft
