// Stage 1 / 1' fused per plane with the intermediate kept in L2 (sm_100a).
//
// The per-plane 2D transform (reference kernels.py:262-303, dfft.py:161-163
// and 205-209) needs every row of a plane before any column can start, and a
// float64 1024x513 half-spectrum plane (8.4 MB) does not fit in shared memory.
// Instead of two whole-slab passes through HBM, one persistent kernel walks
// the planes with an ordered ticket queue A(0), A(1), B(0), A(2), B(1), ...:
//
//   forward  A = R(i): r2c of BR rows of plane i  -> spectral rows (kept in L2)
//            B = C(i): c2c along n1 of BC columns of plane i, read from L2,
//                      self band written in place, peer bands to staging
//   inverse  A = C'(i): inverse c2c along n1 of BC columns (spectral slab from
//                      HBM -> written back, kept in L2)
//            B = R'(i): c2r of BR rows read from L2 -> real output, 1/N folded in
//
// A B task waits for all A tasks of its plane (release/acquire counters); the
// plane in flight between them lives in L2, so each direction moves the real
// slab once and the spectral slab once through HBM (SURVEY.md §8(d) traffic).
#pragma once
#include "fourstep.cuh"
#include "kernels.cuh"

namespace tffft {

constexpr int kS1Threads = 256;

struct Stage1Params {
  void* real;
  void* spec;
  void* staging;          // forward peer bands (p > 1) or null
  const void* tw_row;     // pass tables, length n2/2
  const void* tw_post;    // exp(-2 pi i k / n2), k < n2/2
  const void* tw_col;     // pass tables, length n1
  unsigned long long* stats;  // inverse consistency statistics per plane
  unsigned* counters;     // [0] ticket, [1, 1+n0p) doneA, [1+n0p, 1+2 n0p) doneB
  int n0p, n1, n2c;
  double scale;
  int band_shift, self_band;          // forward redirect: band = n1 index >> band_shift
  long long stg_band, stg_grp;        // staging + band*stg_band + i*stg_grp + (e & mask)*n2c + k
  int lookahead;                      // planes of A tasks handed out ahead of the B tasks
};

// Ticket order with lookahead D: A(0..D-1), then [A(q+D), B(q)] while q+D < ng,
// then B(q) alone.  Returns isA, group, index within the group's task list.
__device__ __forceinline__ void queue_decode(unsigned tk, int ng, int nA, int nB, int D, int& isA, int& g,
                                             int& w) {
  D = D < ng ? D : ng;
  const unsigned head = (unsigned)D * (unsigned)nA;
  if (tk < head) {
    isA = 1; g = (int)(tk / (unsigned)nA); w = (int)(tk % (unsigned)nA);
    return;
  }
  unsigned r = tk - head;
  const unsigned full = (unsigned)(ng - D) * (unsigned)(nA + nB);
  if (r < full) {
    const int q = (int)(r / (unsigned)(nA + nB));
    const int x = (int)(r % (unsigned)(nA + nB));
    if (x < nA) { isA = 1; g = q + D; w = x; }
    else { isA = 0; g = q; w = x - nA; }
    return;
  }
  r -= full;
  isA = 0; g = (ng - D) + (int)(r / (unsigned)nB); w = (int)(r % (unsigned)nB);
}

template <typename T, int LR, int LC>
struct S1Cfg {
  using SR = Shape<LR>;
  using SC = Shape<LC>;
  static constexpr int BR = kS1Threads / SR::TPT;  // rows per R task
  static constexpr int BC = kS1Threads / SC::TPT;  // columns per C task
  static constexpr int PSR = SR::EB > 0 ? SR::EB : 30;
  static constexpr int SRW = SR::N + (SR::N >> (PSR > 20 ? 30 : PSR)) + 2;  // row buffer stride (complex)
  static constexpr int PSC = SC::EB > 0 ? SC::EB : 30;
  static constexpr bool SPLIT = sizeof(T) == 8;
  static constexpr int QW = SPLIT ? 16 : 128 / (int)sizeof(cx<T>);
  static constexpr int RAWC = SC::N + (SC::N >> (PSC > 20 ? 30 : PSC));
  static constexpr int SCW = ((RAWC + QW - 1) / QW) * QW + (QW / BC > 0 ? QW / BC : 1);
  static constexpr size_t ROW_SMEM = sizeof(cx<T>) * (size_t)BR * SRW;
  static constexpr size_t COL_SMEM = (SPLIT ? 8 : sizeof(cx<T>)) * (size_t)BC * SCW;
  static constexpr size_t SMEM = ROW_SMEM > COL_SMEM ? ROW_SMEM : COL_SMEM;
};

template <typename T, int LR, int LC, bool FWD, bool REDIR>
__global__ void __launch_bounds__(kS1Threads, 2)
stage1_fused_kernel(const Stage1Params prm) {
  using CF = S1Cfg<T, LR, LC>;
  using SR = Shape<LR>;
  using SC = Shape<LC>;
  using STR = Stockham<T, LR, !FWD, CF::SRW, CF::PSR>;
  using STC = Stockham<T, LC, !FWD, CF::SCW, CF::PSC, CF::SPLIT>;
  constexpr int NR = SR::N;  // n2 / 2
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_isA, s_g, s_w, s_end;

  const int t = threadIdx.x;
  const int n1 = prm.n1, n2c = prm.n2c;
  const int ng = prm.n0p;
  const int nR = n1 / CF::BR;
  const int nC = (n2c + CF::BC - 1) / CF::BC;
  const int nA = FWD ? nR : nC, nB = FWD ? nC : nR;
  const unsigned total = (unsigned)ng * (unsigned)(nA + nB);
  unsigned* ticket = prm.counters;
  unsigned* doneA = prm.counters + 1;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  cx<T>* spec = reinterpret_cast<cx<T>*>(prm.spec);

  unsigned next_tk = 0;
  if (t == 0) next_tk = atomicAdd(ticket, 1u);
  for (;;) {
    if (t == 0) {
      const unsigned tk = next_tk;
      if (tk >= total) {
        s_end = 1;
      } else {
        int isA, g, w;
        queue_decode(tk, ng, nA, nB, prm.lookahead, isA, g, w);
        if (!isA)
          while (ld_acquire(doneA + g) < (unsigned)nA) __nanosleep(64);
        s_end = 0; s_isA = isA; s_g = g; s_w = w;
        next_tk = atomicAdd(ticket, 1u);
      }
    }
    __syncthreads();
    if (s_end) break;
    const bool isA = s_isA;
    const int plane = s_g, w = s_w;
    const bool row_task = FWD ? isA : !isA;

    if (row_task) {
      // ------------------------------------------------------------ rows
      cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw);
      const cx<T>* tw = reinterpret_cast<const cx<T>*>(prm.tw_row);
      const cx<T>* twp = reinterpret_cast<const cx<T>*>(prm.tw_post);
      const int tt = t % SR::TPT, b = t / SR::TPT;
      const long long row = (long long)plane * n1 + (long long)w * CF::BR + b;
      cx<T>* srow = spec + row * n2c;
      if constexpr (FWD) {
        const cx<T>* in = reinterpret_cast<const cx<T>*>(reinterpret_cast<const T*>(prm.real) + row * (2LL * NR));
        cx<T> v[SR::E];
#pragma unroll
        for (int u = 0; u < SR::E / SR::R0; ++u)
#pragma unroll
          for (int m = 0; m < SR::R0; ++m) v[u * SR::R0 + m] = ld_hint(in + SR::in_elem(tt, u, m), pol_stream);
        STR::run(sm, v, tt, b, tw);
        STR::store_natural(sm, v, tt, b);
        __syncthreads();
        const T half = T(0.5);
#pragma unroll
        for (int q = 0; q < SR::E; ++q) {
          const int k = tt + SR::TPT * q;
          cx<T> X;
          if (k == 0) {
            const cx<T> z0 = sm[STR::sidx(b, 0)];
            X = {z0.x + z0.y, T(0)};
            st_hint(srow + NR, cx<T>{z0.x - z0.y, T(0)}, pol_keep);
          } else {
            const cx<T> A = sm[STR::sidx(b, k)];
            const cx<T> Bz = sm[STR::sidx(b, NR - k)];
            const cx<T> S = {A.x + Bz.x, A.y - Bz.y};
            const cx<T> D = {A.x - Bz.x, A.y + Bz.y};
            const cx<T> Tt = cmul(D, ldg_cx(twp + k));
            X = {half * (S.x + Tt.y), half * (S.y - Tt.x)};
          }
          st_hint(srow + k, X, pol_keep);
        }
      } else {
        double m2 = 0.0, edge = 0.0, resid = 0.0;
#pragma unroll
        for (int q = 0; q <= SR::E; ++q) {
          const int k = tt + SR::TPT * q;
          if (k <= NR && (q < SR::E || tt == 0)) {
            cx<T> X = ldcg_cx(srow + k);
            m2 = fmax(m2, (double)X.x * X.x + (double)X.y * X.y);
            if (k == 0 || k == NR) {
              const double im = fabs((double)X.y);
              edge = fmax(edge, im);
              resid += im;
              X.y = T(0);
            }
            sm[STR::sidx(b, k)] = X;
          }
        }
        constexpr int WR = SR::TPT < 32 ? SR::TPT : 32;
#pragma unroll
        for (int o = WR / 2; o > 0; o >>= 1) {
          m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o, WR));
          edge = fmax(edge, __shfl_xor_sync(0xffffffffu, edge, o, WR));
          resid += __shfl_xor_sync(0xffffffffu, resid, o, WR);
        }
        if (prm.stats != nullptr && (tt % WR) == 0) {
          unsigned long long* st = prm.stats + 3 * plane;
          atomicMax(st + 0, ord(m2));
          if (tt == 0) {
            atomicMax(st + 1, ord(edge));
            atomicMax(st + 2, ord(resid));
          }
        }
        __syncthreads();
        // the spectral rows of this task are consumed (inverse clobbers its input,
        // dfft.py:182-184): drop their whole L2 lines without a write-back
        if (t < CF::BR * (int)(sizeof(cx<T>) * 2 * NR / 128 + 2)) {
          const char* lo = reinterpret_cast<const char*>(spec + ((long long)plane * n1 + (long long)w * CF::BR) * n2c);
          const char* hi = lo + (size_t)CF::BR * n2c * sizeof(cx<T>);
          const char* first = reinterpret_cast<const char*>((reinterpret_cast<uintptr_t>(lo) + 127) & ~(uintptr_t)127);
          const char* line = first + (size_t)t * 128;
          if (line + 128 <= hi) discard_l2(line);
        }
        const cx<T>* twpp = twp;
        cx<T> v[SR::E];
#pragma unroll
        for (int u = 0; u < SR::E / SR::R0; ++u)
#pragma unroll
          for (int m = 0; m < SR::R0; ++m) {
            const int k = SR::in_elem(tt, u, m);
            const cx<T> A = sm[STR::sidx(b, k)];
            const cx<T> Bx = sm[STR::sidx(b, NR - k)];
            const cx<T> S = {A.x + Bx.x, A.y - Bx.y};
            const cx<T> D = {A.x - Bx.x, A.y + Bx.y};
            const cx<T> Tt = cmulc(D, ldg_cx(twpp + k));
            v[u * SR::R0 + m] = {S.x - Tt.y, S.y + Tt.x};
          }
        __syncthreads();
        STR::run(sm, v, tt, b, tw);
        cx<T>* outc = reinterpret_cast<cx<T>*>(reinterpret_cast<T*>(prm.real) + row * (2LL * NR));
        const T s = T(prm.scale);
#pragma unroll
        for (int u = 0; u < SR::E / SR::RL; ++u)
#pragma unroll
          for (int m = 0; m < SR::RL; ++m) {
            const cx<T> z = v[u * SR::RL + m];
            st_hint(outc + SR::out_elem(tt, u, m), cx<T>{z.x * s, z.y * s}, pol_stream);
          }
      }
    } else {
      // ------------------------------------------------------------ columns (n1 axis)
      const cx<T>* tw = reinterpret_cast<const cx<T>*>(prm.tw_col);
      const int b = t % CF::BC, tt = t / CF::BC;
      const int k_raw = w * CF::BC + b;
      const bool valid = k_raw < n2c;
      const int k = valid ? k_raw : n2c - 1;
      cx<T>* col = spec + (long long)plane * n1 * n2c + k;
      cx<T> v[SC::E];
#pragma unroll
      for (int u = 0; u < SC::E / SC::R0; ++u)
#pragma unroll
        for (int m = 0; m < SC::R0; ++m) {
          const cx<T>* a = col + (unsigned)SC::in_elem(tt, u, m) * (unsigned)n2c;
          v[u * SC::R0 + m] = FWD ? ldcg_cx(a) : ld_hint(a, pol_stream);
        }
      STC::run(smem_raw, v, tt, b, tw);
      if (valid) {
        cx<T>* stg = reinterpret_cast<cx<T>*>(prm.staging);
        const unsigned bmask = (1u << prm.band_shift) - 1u;
#pragma unroll
        for (int u = 0; u < SC::E / SC::RL; ++u)
#pragma unroll
          for (int m = 0; m < SC::RL; ++m) {
            const unsigned e = (unsigned)SC::out_elem(tt, u, m);
            const cx<T> z = v[u * SC::RL + m];
            if constexpr (REDIR) {
              const int band = (int)(e >> prm.band_shift);
              if (band != prm.self_band) {
                st_hint(stg + (long long)band * prm.stg_band + (long long)plane * prm.stg_grp +
                            (long long)(e & bmask) * n2c + k, z, pol_stream);
                continue;
              }
            }
            st_hint(col + e * (unsigned)n2c, z, FWD ? pol_stream : pol_keep);
          }
      }
    }
    __syncthreads();
    if (t == 0 && isA) publish_add(doneA + plane);
  }
}

// (LR, LC) combinations with a fused kernel: n2/2 in [256, 2048], n1 = n2
__host__ __device__ constexpr bool stage1_fused_supported(int LR, int LC) {
  return LR >= 8 && LR <= 11 && LC == LR + 1;
}

template <typename T>
cudaError_t launch_stage1_fused(int LR, int LC, bool fwd, bool redir, const Stage1Params& p, cudaStream_t s);

}  // namespace tffft
