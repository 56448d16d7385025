// Stage kernels of the transpose-free slab 3D real FFT (sm_100a).
//
//  r2c_rows   stage 1a  : r2c along n2 of every row of the local planes
//                         (reference kernels.py:203-209, 262-286 first half)
//  col_fft    stage 1b  : c2c along n1 of every (plane, k) column, epilogue
//                         routes peer bands to the exchange staging buffer
//             stage 3   : c2c along n0 of every STRIDED_INPLACE column, read
//                         in place through the two-level stride
//                         (kernels.py:176-200, layout.py:201-219)
//             stage 3'/1b' likewise for the inverse
//  c2r_rows   stage 1a' : c2r along n2, 1/(n0 n1 n2) folded in, Hermitian
//                         consistency statistics (kernels.py:212-239)
#pragma once
#include "fft_engine.cuh"

namespace tffft {

// Column c of a batch: base = (c / cpb) * grp_stride + (c % cpb).
// Element e of a column: (e & (1<<ic_shift)-1) * inner_stride + (e >> ic_shift) * block_stride.
// Redirect (peer bands): band = e >> band_shift; if staging && band != self_band
//   -> staging + band*stg_band + (e & band_mask)*stg_within + (c / cpb)*stg_grp + (c % cpb)
struct ColParams {
  void* data;
  void* staging;          // RD == 2: peer bands read from here (landing)
  void* const* band_dst;  // RD == 1: destination block of band q (p pointers): the rank's
                          // staging block q, or -- peer stores -- rank q's landing block for us
  const void* tw;
  long long ncols;
  int cpb;
  long long grp_stride;
  int ic_shift;
  long long inner_stride, block_stride;
  int band_shift, self_band;
  long long stg_band, stg_within, stg_grp;
  long long stg_base;     // added to every staging / landing offset (plane chunk of stage 1b)
  // L2 prefetch of wide row segments for the tile `pf_ahead` tiles ahead
  // (0 = off): DRAM then sees pf_bytes-wide row visits instead of B*sizeof(cx)
  long long pf_ahead;
  int pf_bytes;
  unsigned long long* ticket;  // TFFFT_COL_TICKET: dynamic tile order (a zeroed counter per launch)
  int probe;  // profiling builds only (TFFFT_PROBES=1): bit 0 skips the epilogue stores, bit 1 the prefetch loads
};

// Rows: row r of real data at real + r*n2 (reals); complex row at spec + r*n2c.
struct RowParams {
  void* real;
  void* spec;
  const void* tw;       // pass tables for N = n2/2
  const void* tw_post;  // exp(-2 pi i k / n2), k < n2/2
  long long nrows;
  int n2c;
  int rows_per_plane;
  double scale;                   // c2r output scale
  double* row_stats;              // c2r: per row [max |X|^2, max |Im X_0|,|Im X_N|, |Im X_0|+|Im X_N|]
};

// Column CTA: B adjacent columns, TPT threads per column, E elements per
// thread.  Shared memory = the prefetch slots P (each thread's own slots for
// PF_E of its E next-tile operands) + the exchange buffer X.  X holds whole
// complex words (TFFFT_SPLIT=0: one 16-byte STS/LDS per element and two
// barriers per exchange; measured 2.6% / 5% faster per f64 / f32 pair than
// exchanging real and imaginary words in separate rounds, TFFFT_SPLIT=1).
// X layout: one pad word per E words inside a column, column stride S chosen
// so one wavefront (B columns x QW/B threads) covers every bank once.
// profiling builds (tools/build_variants.sh ... -DTFFFT_PROBES=1): runtime probe
// bits that skip the column kernel's loads or stores (profiles/r01s2/col_probes.txt)
#ifndef TFFFT_PROBES
#define TFFFT_PROBES 0
#endif
#ifndef TFFFT_COL_TICKET
#define TFFFT_COL_TICKET 1
#endif
#ifndef TFFFT_COLB
#define TFFFT_COLB 8
#endif
#ifndef TFFFT_SPLIT
#define TFFFT_SPLIT 0
#endif
// fewest threads of a column CTA (columns are added until reached)
#ifndef TFFFT_COL_MINTHREADS
#define TFFFT_COL_MINTHREADS 256
#endif
#ifndef TFFFT_PREFETCH
#define TFFFT_PREFETCH 1
#endif
// narrow (stage 1b, rows kilobytes apart) column-kernel shape: columns per CTA,
// cp.async prefetch, persistent grid
#ifndef TFFFT_NARROW_B
#define TFFFT_NARROW_B 8
#endif
#ifndef TFFFT_NARROW_PREFETCH
#define TFFFT_NARROW_PREFETCH 1
#endif
// Cluster pairing: a tile of CL*B columns is split over a thread-block cluster
// of CL CTAs (B columns each).  The CTAs of a cluster run side by side, so the
// two halves of each 128-byte line are fetched together, while every SM hosts
// more, independently-barriered CTAs.
#ifndef TFFFT_COLCLUSTER
#define TFFFT_COLCLUSTER 1
#endif
#ifndef TFFFT_COLCLUSTER_SYNC
#define TFFFT_COLCLUSTER_SYNC 0
#endif
#ifndef TFFFT_COLGROUPS
#define TFFFT_COLGROUPS 1
#endif
// columns per CTA: at least 256 threads, at most 1024 threads and 227 KB of
// shared memory (prefetch slots B*N complex + ~B*N words of exchange buffer)
// WIDE (stage 3, rows megabytes apart): 128-byte row visits, i.e. 8 float64 or
// 16 float32 columns; otherwise 8 columns
template <typename T, int L, bool WIDE>
__host__ __device__ constexpr int col_batch() {
  constexpr int TPT = Shape<L>::TPT, N = Shape<L>::N;
  constexpr int want = WIDE ? TFFFT_COLB * (int)(16 / sizeof(cx<T>)) : TFFFT_NARROW_B;
  int b = TFFFT_COL_MINTHREADS / TPT > want ? TFFFT_COL_MINTHREADS / TPT : want;
  // split exchange: prefetch slots (complex) + exchange buffer (real words);
  // whole-complex exchange: the next tile's operands fit slots + exchange buffer
  constexpr size_t per_elem = TFFFT_SPLIT ? sizeof(cx<T>) + sizeof(T) : sizeof(cx<T>);
  // the shared-memory bound applies per CTA: a WIDE tile may span a cluster of TFFFT_COLCLUSTER CTAs
  constexpr int cl = WIDE ? TFFFT_COLCLUSTER : 1;
  while (b > 1 && (TPT * (b / cl) > 1024 || (size_t)(b / cl) * N * per_elem + 8192 > 227 * 1024)) b /= 2;
  return b;
}
template <typename T, int L, bool WIDE = false> struct ColCfg {
  static constexpr int TPT = Shape<L>::TPT;
  static constexpr int CL = (col_batch<T, L, WIDE>() % TFFFT_COLCLUSTER == 0 &&
                             TPT * (col_batch<T, L, WIDE>() / TFFFT_COLCLUSTER) >= 128) ? TFFFT_COLCLUSTER : 1;
  static constexpr int B = col_batch<T, L, WIDE>() / CL;     // columns per CTA
  static constexpr int THREADS = TPT * B;
  // The CTA's B columns are split over GROUPS independent thread groups (own
  // exchange buffer, own named barrier): their smem-exchange and FP64 phases
  // drift apart and overlap instead of alternating CTA-wide.
  static constexpr int GROUPS = (B % TFFFT_COLGROUPS == 0 && THREADS / TFFFT_COLGROUPS >= 128) ? TFFFT_COLGROUPS : 1;
  static constexpr int GB = B / GROUPS;               // columns per group
  static constexpr int GT = THREADS / GROUPS;         // threads per group
  static constexpr int PS = Shape<L>::EB > 0 ? Shape<L>::EB : 30;
  static constexpr int RAW = Shape<L>::N + (Shape<L>::N >> (PS > 20 ? 30 : PS));
  // exchange in real-valued words (re round, then im round): halves the buffer
  static constexpr bool SPLIT = TFFFT_SPLIT;
  static constexpr int WORD = SPLIT ? (int)sizeof(T) : (int)sizeof(cx<T>);  // exchange word bytes
  static constexpr int QW = 128 / WORD;                          // words per 128 bytes
  // B columns x (QW/B) consecutive threads share one wavefront: offset column b
  // by b*QW/B words so the wavefront covers every bank exactly once
  static constexpr int S = ((RAW + QW - 1) / QW) * QW + (QW / GB > 0 ? QW / GB : 1);
  static constexpr bool XCHG = Shape<L>::P > 1;
  // stage 3 (WIDE): persistent CTAs prefetch the next tile; stage 1b: one tile
  // per CTA, several CTAs per SM overlap instead
  static constexpr bool PREFETCH = WIDE ? TFFFT_PREFETCH : TFFFT_NARROW_PREFETCH;
  static constexpr bool PERSISTENT = PREFETCH;
  static constexpr size_t X_BYTES = XCHG ? (size_t)WORD * B * S : 0;
  // Prefetch: PF_E of each thread's E next-tile operands go to private slots
  // while the tile computes; when slots for all E do not fit beside the
  // exchange buffer, the other LO_E are fetched into the exchange buffer as
  // soon as the tile's last exchange has drained it.
  static constexpr size_t SMEM_MAX = 227 * 1024;
  static constexpr int PF_FIT = (int)((SMEM_MAX - X_BYTES) / (sizeof(cx<T>) * THREADS));
  static constexpr int PF_E = !PREFETCH ? 0 : (PF_FIT < Shape<L>::E ? PF_FIT : Shape<L>::E);
  static constexpr int LO_E = PREFETCH ? Shape<L>::E - PF_E : 0;
  static_assert(LO_E == 0 || (GROUPS == 1 && (size_t)LO_E * THREADS * sizeof(cx<T>) <= X_BYTES),
                "leftover operands must fit the (single-group) exchange buffer");
  static constexpr size_t P_BYTES = sizeof(cx<T>) * THREADS * PF_E;
};

#ifndef TFFFT_ROW_THREADS
#define TFFFT_ROW_THREADS 128
#endif
#ifndef TFFFT_ROW_MINB
#define TFFFT_ROW_MINB 1
#endif
#ifndef TFFFT_C2R_MINB9
#define TFFFT_C2R_MINB9 5
#endif
#ifndef TFFFT_R2C_MINB9
#define TFFFT_R2C_MINB9 8
#endif
// (radix 16 x 8 x 8, E = 16, at 4 CTAs/SM of 128 threads -- 128 registers: r2c 2.88 -> 2.71 ms, c2r
// 3.04 -> 2.95 ms per 256x2048x2048 launch; 5 CTAs/SM spills: c2r 3.74 ms; profiles/r02s4/rows_2048.txt)
#ifndef TFFFT_C2R_MINB10
#define TFFFT_C2R_MINB10 4
#endif
#ifndef TFFFT_R2C_MINB10
#define TFFFT_R2C_MINB10 4
#endif
// r2c row schedule: float64 rows of n2 = 1024 run the radix-8 schedule
// (3 passes, E = 8, 6 CTAs/SM: 3.10 ms per 1024^3 launch vs 3.62 ms with radix
// 32x16); every other row / column transform uses the default schedule
#ifndef TFFFT_R2C_L9_F64_MB
#define TFFFT_R2C_L9_F64_MB 4
#endif
// n2 = 2048 (the rows of BASELINE config 4), per 8.6 GB-in / 8.6 GB-out launch
// (profiles/r02s4/rows_2048.txt): r2c 3.08 ms on the default radix 32 x 32,
// 2.97 ms on radix 16 x 8 x 8, 3.11 ms on 8 x 8 x 4 x 4; c2r 3.90 / 3.70 / 3.45 ms
#ifndef TFFFT_R2C_L10_F64_MB
#define TFFFT_R2C_L10_F64_MB 4
#endif
// (after the twiddle factorisation of finding 33: c2r 3.18 ms on 8 x 8 x 4 x 4, 3.02 ms on 16 x 8 x 8)
#ifndef TFFFT_C2R_L10_F64_MB
#define TFFFT_C2R_L10_F64_MB 4
#endif
__host__ __device__ constexpr int r2c_radix_bits(int L, int real_bytes) {
  return real_bytes == 8 ? (L == 9 ? TFFFT_R2C_L9_F64_MB : (L == 10 ? TFFFT_R2C_L10_F64_MB : 0)) : 0;
}
// c2r likewise: radix 8 at 6 CTAs/SM, 3.14 ms per 1024^3 launch vs 3.23 ms
// with radix 32x16 at 240 registers (profiles/r01s3/rows.txt)
#ifndef TFFFT_C2R_L9_F64_MB
#define TFFFT_C2R_L9_F64_MB 4
#endif
// (and for n2 = 512: radix 8 at 5 CTAs/SM, 0.392 -> 0.379 ms per 512^3 launch;
// the r2c rows there keep radix 16, profiles/r01s13/rows_512.txt)
__host__ __device__ constexpr int c2r_radix_bits(int L, int real_bytes) {
  return real_bytes == 8 ? (L == 9 ? TFFFT_C2R_L9_F64_MB : (L == 8 ? 3 : (L == 10 ? TFFFT_C2R_L10_F64_MB : 0))) : 0;
}

template <int L, int MB = 0> struct RowCfg {
  static constexpr int TPT = Shape<L, MB>::TPT;
  static constexpr int B = TFFFT_ROW_THREADS / TPT > 1 ? TFFFT_ROW_THREADS / TPT : 1;
  static constexpr int THREADS = TPT * B;
  static constexpr int PS = Shape<L, MB>::EB > 0 ? Shape<L, MB>::EB : 30;  // one pad slot per E elements
  static constexpr int N = Shape<L, MB>::N;
  static constexpr int S = N + (N >> (PS > 20 ? 30 : PS)) + 1 + 1;   // room for bin N in c2r
  // n2 = 1024 float64 row kernels on the radix-8 schedule: occupancy by
  // launch bounds, measured over 5 / 6 / 7 / 8 CTAs of 128 threads per SM
  // (profiles/r01s7/row_minb.txt): r2c best at 8 (64 registers, no spills,
  // 2.69 ms per 1024^3 launch), c2r -- with its consistency statistics and
  // pair loads -- at 5 (94 registers, 2.88 ms).  Other lengths keep the default.
  // (radix-8 schedule only, E = 8; the radix-32 schedule needs ~200 registers)
  static constexpr bool CAP = (L == 9 || L == 8) && THREADS == 128 && Shape<L, MB>::E == 8;
  // n2 = 2048 (E = 8 or 16, 128-thread CTAs): occupancy by launch bounds, TFFFT_R2C_MINB10 / TFFFT_C2R_MINB10
  static constexpr bool CAP10 = L == 10 && THREADS == 128 && (Shape<L, MB>::E == 8 || Shape<L, MB>::E == 16);
  static constexpr int MINB_C2R = CAP ? TFFFT_C2R_MINB9 : (CAP10 ? TFFFT_C2R_MINB10 : TFFFT_ROW_MINB);
  static constexpr int MINB_R2C = CAP ? TFFFT_R2C_MINB9 : (CAP10 ? TFFFT_R2C_MINB10 : TFFFT_ROW_MINB);
};

template <typename T, int L, bool WIDE = false>
__host__ __device__ constexpr size_t col_smem_bytes() {
  return ColCfg<T, L, WIDE>::P_BYTES + ColCfg<T, L, WIDE>::X_BYTES;
}
template <typename T, int L, int MB = 0>
__host__ __device__ constexpr size_t row_smem_bytes() {
  return sizeof(cx<T>) * RowCfg<L, MB>::B * RowCfg<L, MB>::S;
}

// ---------------------------------------------------------------------------
// batched column c2c (stages 1b, 3, 3', 1b') -- persistent, prefetching
// ---------------------------------------------------------------------------
// Each CTA walks tiles blockIdx.x, +gridDim.x, ...  While tile i is being
// transformed out of registers, tile i+1 streams into the thread-private
// prefetch slots with cp.async: every thread copies exactly the E elements it
// will feed into pass 0, so the hand-off needs no CTA barrier.
// TWO   : element offsets use the two-level STRIDED_INPLACE formula (p > 1,
//         stage 3); otherwise offset = e * inner_stride.
// RD    : 0 = in place; 1 = the epilogue writes peer bands to the exchange
//         staging buffer; 2 = peer bands are READ from the exchange landing
//         buffer (where the exchange delivered them contiguously) and every
//         element is written in place -- the strided "datatype" of the
//         reference's exchange (exchange.py:114-121) applied by the FFT's own
//         addressing, with no rearrangement pass.  Staging and landing share the
//         [band][i][j][k] chunk layout described by stg_band/stg_within/stg_grp.
// All element offsets are 32-bit (plan_create bounds the slab below 2^32
// elements); the 64-bit column base pointer is formed once per tile.
template <typename T, int L, bool INV, bool TWO, int RD, bool WIDE>
__global__ void __launch_bounds__(ColCfg<T, L, WIDE>::THREADS)
col_fft_kernel(const ColParams prm) {
  using CF = ColCfg<T, L, WIDE>;
  using SH = Shape<L>;
  using ST = Stockham<T, L, INV, CF::S, CF::PS, CF::SPLIT, (CF::GROUPS > 1 ? CF::GT : 0)>;
  constexpr int E = SH::E, TPT = SH::TPT, B = CF::B, NT = CF::THREADS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cx<T>* pf = reinterpret_cast<cx<T>*>(smem_raw);  // [E][NT] prefetch slots
  const cx<T>* tw = reinterpret_cast<const cx<T>*>(prm.tw);

  const int t = threadIdx.x;
  const int grp = t / CF::GT;              // independent column group
  const int bl = (t % CF::GT) % CF::GB;    // column within the group
  const int tt = (t % CF::GT) / CF::GB;    // thread within the column
  const int b = grp * CF::GB + bl;         // column within the tile
  void* xs = smem_raw + CF::P_BYTES + (size_t)grp * (CF::X_BYTES / CF::GROUPS);  // group's exchange buffer
  const unsigned is = (unsigned)prm.inner_stride;
  const unsigned bs = (unsigned)prm.block_stride;
  const unsigned ics = (unsigned)prm.ic_shift;
  const unsigned icm = (1u << ics) - 1u;
  constexpr int CL = CF::CL;
  const int cl_rank = CL > 1 ? (int)(blockIdx.x % CL) : 0;   // cluster dims (CL, 1, 1)
  const long long ntiles = (prm.ncols + CL * B - 1) / (CL * B);

  auto offset = [&](unsigned e) -> unsigned {
    if constexpr (TWO) return (e & icm) * is + (e >> ics) * bs;
    else return e * is;
  };
  struct Col { cx<T>* p; unsigned cq, cr; bool valid; };
  auto column = [&](long long tile) -> Col {
    const long long c_raw = tile * (CL * B) + cl_rank * B + b;
    const bool valid = c_raw < prm.ncols;
    const unsigned c = (unsigned)(valid ? c_raw : prm.ncols - 1);  // clamp: loads stay in bounds
    const unsigned cq = c / (unsigned)prm.cpb;
    const unsigned cr = c - cq * (unsigned)prm.cpb;
    return {reinterpret_cast<cx<T>*>(prm.data) + ((long long)cq * prm.grp_stride + cr), cq, cr, valid};
  };
  const unsigned bmask = (1u << prm.band_shift) - 1u;
  auto src = [&](const Col& col, unsigned e) -> const cx<T>* {
    if constexpr (RD == 2) {
      const int band = (int)(e >> prm.band_shift);
      if (band != prm.self_band)
        return reinterpret_cast<const cx<T>*>(prm.staging) + ((long long)col.cq * prm.stg_grp + col.cr + prm.stg_base) +
               (long long)band * prm.stg_band + (long long)(e & bmask) * prm.stg_within;
    }
    return col.p + offset(e);
  };
  cx<T>* lo = reinterpret_cast<cx<T>*>(xs);  // [LO_E][NT] leftover slots inside the exchange buffer
  auto prefetch = [&](const Col& col) {
#if TFFFT_PROBES
    if (prm.probe & 2) return;
#endif
#pragma unroll
    for (int kk = 0; kk < CF::PF_E; ++kk) cp_async<sizeof(cx<T>)>(pf + kk * NT + t, src(col, tt + TPT * kk));
    cp_commit();
  };
  auto prefetch_lo = [&](const Col& col) {
#if TFFFT_PROBES
    if (prm.probe & 2) return;
#endif
#pragma unroll
    for (int kk = CF::PF_E; kk < E; ++kk)
      cp_async<sizeof(cx<T>)>(lo + (kk - CF::PF_E) * NT + t, src(col, tt + TPT * kk));
    cp_commit();
  };

  long long tile = blockIdx.x / CL;
  const long long tstep = gridDim.x / CL;
  // Dynamic tile order (a ticket counter zeroed before each launch): the tiles
  // in flight stay within a window of ~gridDim consecutive tiles however far
  // the CTAs drift apart, so neighbouring tiles -- the rest of the same DRAM
  // pages -- are fetched together (1024^3 f64 stage 3: 3.68 -> 3.25 ms).
  // Needs the CTA barriers of the exchange in every iteration (P > 1).
  // (the host passes a counter only where it was measured faster: columns of 1024+)
  constexpr bool DYN_OK = TFFFT_COL_TICKET && CF::XCHG && CL == 1;
  const bool dyn = DYN_OK && prm.ticket != nullptr;
  // s_tk[0..1]: ping-pong next-tile slots; s_tk[2]: the first tile, in its own
  // slot so thread 0's first ping-pong write cannot race a late warp's read
  __shared__ long long s_tk[3];
  long long it = 0;
  if (dyn) {
    if (t == 0) {
      s_tk[2] = (long long)atomicAdd(prm.ticket, 1ull);
      s_tk[0] = (long long)atomicAdd(prm.ticket, 1ull);
    }
    __syncthreads();
    tile = s_tk[2];
  }
  if (tile >= ntiles) return;
  Col cur = column(tile);
  if (CF::PREFETCH) prefetch(cur);
  if (CF::LO_E > 0) prefetch_lo(cur);
  // tiles sharing one pf_bytes-wide row segment; each prefetches N/GT rows
  const int GT = prm.pf_ahead > 0 ? prm.pf_bytes / (B * (int)sizeof(cx<T>)) : 1;
  for (; tile < ntiles; tile = dyn ? tile : tile + tstep) {
    if constexpr (CL > 1 && TFFFT_COLCLUSTER_SYNC) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    }
    if (prm.pf_ahead > 0) {
      const long long tp = tile + prm.pf_ahead;
      const int rows = SH::N / GT;
      if (tp < ntiles && t < rows) {
        const long long c0 = (tp / GT) * GT * B;
        if (c0 + (long long)GT * B <= prm.ncols) {
          const unsigned e = (unsigned)((tp % GT) * rows + t);
          const cx<T>* p = reinterpret_cast<const cx<T>*>(prm.data) + c0 + offset(e);
          prefetch_l2(p, (unsigned)prm.pf_bytes);
        }
      }
    }
    cx<T> v[E];
    Col next = cur;
    long long nxt = tile + tstep;
    if (dyn) {
      nxt = s_tk[it & 1];
      if (t == 0) s_tk[(it + 1) & 1] = (long long)atomicAdd(prm.ticket, 1ull);  // read next iteration, after the barriers below
      ++it;
    }
    if constexpr (CF::PREFETCH) {
      cp_wait_all();
#pragma unroll
      for (int kk = 0; kk < E; ++kk)
        v[SH::in_slot(kk)] = kk < CF::PF_E ? pf[kk * NT + t] : lo[(kk - CF::PF_E) * NT + t];
      ST::first(v, tt, tw);  // consumes v: the slots are free for the next tile
      if (nxt < ntiles) {
        next = column(nxt);
        prefetch(next);
      }
      if constexpr (CF::LO_E > 0) {
        __syncthreads();  // every thread has its leftovers before the exchange reuses the buffer
        auto hook = [&] { if (nxt < ntiles) prefetch_lo(next); };
        ST::finish(xs, v, tt, bl, tw, hook);
      } else {
        ST::finish(xs, v, tt, bl, tw);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < E; ++kk) v[SH::in_slot(kk)] = *src(cur, tt + TPT * kk);
      ST::first(v, tt, tw);
      if (nxt < ntiles) next = column(nxt);
      ST::finish(xs, v, tt, bl, tw);
    }

#if TFFFT_PROBES
    if (prm.probe & 1) cur.valid = false;
#endif
    if (cur.valid) {
      if constexpr (RD == 1) {
        const long long cofs = (long long)cur.cq * prm.stg_grp + cur.cr + prm.stg_base;
        const unsigned sw = (unsigned)prm.stg_within;
#pragma unroll
        for (int u = 0; u < E / SH::RL; ++u)
#pragma unroll
          for (int m = 0; m < SH::RL; ++m) {
            const unsigned e = SH::out_elem(tt, u, m);
            const int band = (int)(e >> prm.band_shift);
            if (band != prm.self_band) {
              cx<T>* dst = reinterpret_cast<cx<T>*>(
                  __ldg(reinterpret_cast<const unsigned long long*>(prm.band_dst) + band));
              dst[cofs + (long long)(e & bmask) * sw] = v[u * SH::RL + m];
            } else {
              cur.p[offset(e)] = v[u * SH::RL + m];
            }
          }
      } else {
#pragma unroll
        for (int u = 0; u < E / SH::RL; ++u)
#pragma unroll
          for (int m = 0; m < SH::RL; ++m) cur.p[offset(SH::out_elem(tt, u, m))] = v[u * SH::RL + m];
      }
    }
    cur = next;
    if (dyn) tile = nxt;
  }
}

// ---------------------------------------------------------------------------
// r2c along n2 (packed: n2 reals -> N = n2/2 complex FFT -> n2/2+1 bins)
// ---------------------------------------------------------------------------
template <typename T, int L>
__global__ void __launch_bounds__(RowCfg<L, r2c_radix_bits(L, sizeof(T))>::THREADS,
                                  RowCfg<L, r2c_radix_bits(L, sizeof(T))>::MINB_R2C)
r2c_rows_kernel(const RowParams prm) {
  constexpr int MB = r2c_radix_bits(L, sizeof(T));
  using RC = RowCfg<L, MB>;
  using SH = Shape<L, MB>;
  using ST = Stockham<T, L, false, RC::S, RC::PS, false, 0, false, MB>;
  constexpr int N = SH::N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw);
  const cx<T>* tw = reinterpret_cast<const cx<T>*>(prm.tw);
  const cx<T>* twp = reinterpret_cast<const cx<T>*>(prm.tw_post);

  const int tt = threadIdx.x % SH::TPT;
  const int b = threadIdx.x / SH::TPT;
  const long long row = (long long)blockIdx.x * RC::B + b;
  const bool valid = row < prm.nrows;
  const cx<T>* in = reinterpret_cast<const cx<T>*>(reinterpret_cast<const T*>(prm.real) + (valid ? row : 0) * (2LL * N));

  cx<T> v[SH::E];
#pragma unroll
  for (int u = 0; u < SH::E / SH::R0; ++u)
#pragma unroll
    for (int m = 0; m < SH::R0; ++m) v[u * SH::R0 + m] = in[SH::in_elem(tt, u, m)];

  ST::run(sm, v, tt, b, tw);
  if constexpr (SH::P > 1) __syncthreads();  // last exchange reads done before reuse
  // natural-order outputs, UNPADDED: the post-processing reads contiguous runs
  // of k and of N - k, and a reversed run straddles the exchange layout's pad
  // slots (2-way bank conflicts on every read of N - k)
  cx<T>* zr = sm + b * RC::S;
#pragma unroll
  for (int u = 0; u < SH::E / SH::RL; ++u)
#pragma unroll
    for (int m = 0; m < SH::RL; ++m) zr[SH::out_elem(tt, u, m)] = v[u * SH::RL + m];
  __syncthreads();
  if (!valid) return;

  // Bins k and N - k come from the same pair (Z[k], Z[N-k]): with
  // S = Z[k] + conj(Z[N-k]), D = Z[k] - conj(Z[N-k]), T = D w^k (w = e^{-2 pi i / n2}),
  //   X[k]     = (S.x + T.y, S.y - T.x) / 2
  //   X[N - k] = (S.x - T.y, -(S.y + T.x)) / 2   (w^{N-k} = -conj(w^k))
  // so each thread reads every pair once and writes both bins.
  cx<T>* out = reinterpret_cast<cx<T>*>(prm.spec) + row * prm.n2c;
  const T half = T(0.5);
  // The twiddle of k = tt + TPT q factors as w^tt * exp(-2 pi i q / (2 E)): one
  // table load per thread and a rotation by a 16th (E = 8) or 32nd (E = 16)
  // root of unity that is a constant after unrolling (float64; the kernel is
  // bound by L1/TEX requests, profiles/r02s4/rows_full.txt).
  constexpr bool ROT = sizeof(T) == 8 && (SH::E == 8 || SH::E == 16);
  auto pair = [&](int k, cx<T> w) {
    const cx<T> A = zr[k];
    const cx<T> Bz = zr[N - k];
    const cx<T> S = {A.x + Bz.x, A.y - Bz.y};   // A + conj(B)
    const cx<T> D = {A.x - Bz.x, A.y + Bz.y};   // A - conj(B)
    const cx<T> Tt = cmul(D, w);
    out[k] = cx<T>{half * (S.x + Tt.y), half * (S.y - Tt.x)};
    if (N - k != k) out[N - k] = cx<T>{half * (S.x - Tt.y), -half * (S.y + Tt.x)};
  };
  cx<T> wb = {T(1), T(0)};
  if constexpr (ROT) wb = ldg_cx(twp + tt);
#pragma unroll
  for (int q = 0; q < (SH::E > 1 ? SH::E / 2 : 1); ++q) {
    const int k = tt + SH::TPT * q;  // k < N/2
    if (k == 0) {
      const cx<T> z0 = zr[0];
      out[0] = cx<T>{z0.x + z0.y, T(0)};
      out[N] = cx<T>{z0.x - z0.y, T(0)};
    } else if constexpr (ROT) {
      pair(k, SH::E == 8 ? mul_w16<false>(wb, q) : mul_w32<false>(wb, q));
    } else {
      pair(k, ldg_cx(twp + k));
    }
  }
  if (tt == 0 && N >= 2) pair(N / 2, ldg_cx(twp + N / 2));  // the self-paired middle bin
}

// ---------------------------------------------------------------------------
// c2r along n2 (packed inverse), scale folded in, consistency statistics
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ord(double x) { return __double_as_longlong(x); }

template <typename T, int L>
__global__ void __launch_bounds__(RowCfg<L, c2r_radix_bits(L, sizeof(T))>::THREADS,
                                  RowCfg<L, c2r_radix_bits(L, sizeof(T))>::MINB_C2R)
c2r_rows_kernel(const RowParams prm) {
  constexpr int MB = c2r_radix_bits(L, sizeof(T));
  using RC = RowCfg<L, MB>;
  using SH = Shape<L, MB>;
  using ST = Stockham<T, L, true, RC::S, RC::PS, false, 0, false, MB>;
  constexpr int N = SH::N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw);
  const cx<T>* tw = reinterpret_cast<const cx<T>*>(prm.tw);
  const cx<T>* twp = reinterpret_cast<const cx<T>*>(prm.tw_post);

  const int tt = threadIdx.x % SH::TPT;
  const int b = threadIdx.x / SH::TPT;
  const long long row = (long long)blockIdx.x * RC::B + b;
  const bool valid = row < prm.nrows;
  const cx<T>* in = reinterpret_cast<const cx<T>*>(prm.spec) + (valid ? row : 0) * prm.n2c;

  // Hermitian pre-processing: the thread's pass-0 operands k = in_elem(...)
  // and their partners N - k (contiguous forward / reversed runs per warp).
  // Statistics of the Hermitian check on the way: max |X|^2 over the row
  // (each k < N once, bin N by thread 0), |Im X_0|, |Im X_N| (thread 0).
  // Each row writes one plain 24-byte record (reduced per plane on request by
  // reduce_row_stats_kernel): atomics from the ~1000 rows of a plane in flight
  // would serialise on a few L2 addresses (measured +0.4 ms per 1024^3 launch).
  // float64: max |X|^2 is kept as the high word of the (non-negative) double,
  // compared as an integer, one IMNMX per element; the record stores the word
  // with an all-ones low half, an upper bound within 2^-20 relative of the
  // exact maximum (the tolerance is 1e-9 n max|X|).  float32: max(|Re X|,
  // |Im X|) compared as the float's bit pattern; the record 2 m^2 bounds
  // max |X|^2 from above (within 2x), well inside the float32 tolerance.
  constexpr int W = SH::TPT < 32 ? SH::TPT : 32;
  constexpr int SEGS = SH::TPT / W;  // warp segments per row
  __shared__ int seg_m2[RC::B][SEGS];
  int m2h = 0;
  double e0 = 0.0, eN = 0.0;
  auto m2hi = [](cx<T> X) {
    if constexpr (sizeof(T) == 4) return __float_as_int(fmaxf(fabsf(X.x), fabsf(X.y)));
    else return __double2hiint(fma((double)X.x, (double)X.x, (double)X.y * X.y));
  };
  // the pre-processed pass-0 operand from the bin pair (A = X_k, B = X_{N-k})
  auto pre = [&](cx<T> A, cx<T> Bx, int k) -> cx<T> {
    const cx<T> S = {A.x + Bx.x, A.y - Bx.y};  // A + conj(B)
    const cx<T> D = {A.x - Bx.x, A.y + Bx.y};  // A - conj(B)
    const cx<T> Tt = cmulc(D, ldg_cx(twp + k)); // exp(+2 pi i k / n2) * D
    return {S.x - Tt.y, S.y + Tt.x};
  };
  // The same with the twiddle factored: k = (tt + TPT u) + m N / R0, so
  // exp(2 pi i k / n2) = exp(2 pi i (tt + TPT u) / n2) * exp(2 pi i m / (2 R0)):
  // one table load per thread and u, and a rotation of D by a 16th (R0 = 8) or
  // 32nd (R0 = 16) root of unity that is a compile-time constant after
  // unrolling.  The kernel is bound by L1/TEX requests (85% busy,
  // profiles/r02s4/rows_full.txt): this drops one of the three 16-byte loads
  // per operand.
  constexpr bool ROT = sizeof(T) == 8 && (SH::R0 == 8 || SH::R0 == 16);
  auto pre_rot = [&](cx<T> A, cx<T> Bx, cx<T> wb, int m) -> cx<T> {
    const cx<T> S = {A.x + Bx.x, A.y - Bx.y};
    const cx<T> D = {A.x - Bx.x, A.y + Bx.y};
    const cx<T> Dm = SH::R0 == 8 ? mul_w16<true>(D, m) : mul_w32<true>(D, m);
    const cx<T> Tt = cmulc(Dm, wb);
    return {S.x - Tt.y, S.y + Tt.x};
  };
  cx<T> v[SH::E];
  if constexpr (sizeof(T) == 8) {
    // float64 (radix-8 schedule): pairs straight from global memory, 1024^3
    // launch 3.14 -> 2.97 ms against staging the row in shared memory
#pragma unroll
    for (int u = 0; u < SH::E / SH::R0; ++u) {
      cx<T> wb = {T(1), T(0)};
      if constexpr (ROT) wb = ldg_cx(twp + tt + SH::TPT * u);
#pragma unroll
      for (int m = 0; m < SH::R0; ++m) {
        const int k = SH::in_elem(tt, u, m);
        cx<T> A = ldg_cx(in + k);
        m2h = max(m2h, m2hi(A));
        cx<T> Bx;
        if (k == 0) {  // c2r uses only the real part of the DC / Nyquist bins
          Bx = ldg_cx(in + N);
          m2h = max(m2h, m2hi(Bx));
          e0 = fabs((double)A.y);
          eN = fabs((double)Bx.y);
          A.y = T(0);
          Bx.y = T(0);
        } else {
          Bx = ldg_cx(in + (N - k));
        }
        if constexpr (ROT) v[u * SH::R0 + m] = pre_rot(A, Bx, wb, m);
        else v[u * SH::R0 + m] = pre(A, Bx, k);
      }
    }
  } else {
    // float32 (radix-32 schedule): the row staged in shared memory in natural
    // order, UNPADDED (reversed runs N - k stay bank-conflict free); 1.43 ms
    // against 1.83 ms for the global pair reads
    cx<T>* xr = sm + b * RC::S;
#pragma unroll
    for (int q = 0; q < SH::E; ++q) {
      const int k = tt + SH::TPT * q;
      const cx<T> X = in[k];
      m2h = max(m2h, m2hi(X));
      xr[k] = X;
    }
    if (tt == 0) {
      cx<T> X0 = xr[0];
      cx<T> XN = in[N];
      m2h = max(m2h, m2hi(XN));
      e0 = fabs((double)X0.y);
      eN = fabs((double)XN.y);
      X0.y = T(0);  // c2r uses only the real part of the DC / Nyquist bins
      XN.y = T(0);
      xr[0] = X0;
      xr[N] = XN;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < SH::E / SH::R0; ++u)
#pragma unroll
      for (int m = 0; m < SH::R0; ++m) {
        const int k = SH::in_elem(tt, u, m);
        v[u * SH::R0 + m] = pre(xr[k], xr[N - k], k);
      }
  }
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) m2h = max(m2h, __shfl_xor_sync(0xffffffffu, m2h, o, W));
  if ((tt % W) == 0) seg_m2[b][tt / W] = m2h;
  __syncthreads();
  if (tt == 0 && valid && prm.row_stats != nullptr) {
#pragma unroll
    for (int g = 1; g < SEGS; ++g) m2h = max(m2h, seg_m2[b][g]);
    double* rec = prm.row_stats + 3 * row;
    if constexpr (sizeof(T) == 4) {
      const double m = (double)__int_as_float(m2h);
      rec[0] = 2.0 * m * m;
    } else {
      rec[0] = __hiloint2double(m2h, -1);
    }
    rec[1] = fmax(e0, eN);
    rec[2] = e0 + eN;
  }
  if constexpr (sizeof(T) == 4) __syncthreads();  // the staged row is consumed before the exchanges reuse it

  ST::run(sm, v, tt, b, tw);
  if (!valid) return;

  T* out = reinterpret_cast<T*>(prm.real) + row * (2LL * N);
  cx<T>* outc = reinterpret_cast<cx<T>*>(out);
  const T s = T(prm.scale);
#pragma unroll
  for (int u = 0; u < SH::E / SH::RL; ++u)
#pragma unroll
    for (int m = 0; m < SH::RL; ++m) {
      const cx<T> z = v[u * SH::RL + m];
      outc[SH::out_elem(tt, u, m)] = cx<T>{z.x * s, z.y * s};
    }
}

// per-plane maxima of the c2r row records (one CTA per plane), stored as the
// ordered-double words the host check reads (same format as the fused
// kernel's atomics)
static __global__ void __launch_bounds__(256) reduce_row_stats_kernel(const double* rec, int rows_per_plane,
                                                               unsigned long long* out) {
  const long long base = (long long)blockIdx.x * rows_per_plane;
  double m[3] = {0.0, 0.0, 0.0};
  for (int r = threadIdx.x; r < rows_per_plane; r += blockDim.x)
#pragma unroll
    for (int c = 0; c < 3; ++c) m[c] = fmax(m[c], rec[3 * (base + r) + c]);
  __shared__ double red[3][8];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m[c] = fmax(m[c], __shfl_xor_sync(0xffffffffu, m[c], o));
    if (threadIdx.x % 32 == 0) red[c][threadIdx.x / 32] = m[c];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) v = fmax(v, red[threadIdx.x][w]);
    out[3 * blockIdx.x + threadIdx.x] = ord(v);
  }
}

// Deferred Hermitian check: fold the per-plane statistics of one inverse into
// a device accumulator, with the host's test (kernels.py:222-238: |Im X_0|,
// |Im X_N| and the residue against rtol * n2 * max|X|), so a run of inverses
// needs no host synchronisation per call.  acc: [0] max residue, [1]
// violations, [2] first violating plane (field-major index), [3] worst
// max(edge, residue) / tol -- non-negative doubles compared as integers.
static __global__ void __launch_bounds__(256) consistency_fold_kernel(const unsigned long long* stats, int planes,
                                                                      double n2, double rtol,
                                                                      unsigned long long* acc) {
  for (int i = threadIdx.x; i < planes; i += blockDim.x) {
    const double m2 = __longlong_as_double((long long)stats[3 * i]);
    const double edge = __longlong_as_double((long long)stats[3 * i + 1]);
    const double r = __longlong_as_double((long long)stats[3 * i + 2]);
    const double tol = rtol * n2 * sqrt(m2);
    atomicMax(acc + 0, ord(r));
    if (edge > tol || r > tol) {
      atomicAdd(acc + 1, 1ull);
      atomicMin(acc + 2, (unsigned long long)i);
      atomicMax(acc + 3, ord(fmax(edge, r) / fmax(tol, 1e-300)));
    }
  }
}

// host-side launchers (defined in kernels_f64.cu / kernels_f32.cu)
// variant: 0 = single stride, 1 = single stride + redirect, 2 = two-level, 3 = two-level + redirect
// wide: stage-3 tiles (128-byte row visits for either precision); two: two-level
// element offsets; rd: 0 in place, 1 write peer bands to staging, 2 read peer bands from landing
template <typename T>
cudaError_t launch_col_fft(int L, bool inv, bool two, int rd, bool wide, const ColParams& p, cudaStream_t s);
template <typename T>
cudaError_t launch_r2c_rows(int L, const RowParams& p, cudaStream_t s);
template <typename T>
cudaError_t launch_c2r_rows(int L, const RowParams& p, cudaStream_t s);

}  // namespace tffft
