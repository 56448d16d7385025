// Stage 3 / 3' as an L2-resident four-step (sm_100a).
//
// The strided length-n0 column transform (reference kernels.py:176-200 over
// the STRIDED_INPLACE columns, layout.py:201-219) walks rows that are
// n1*n2c elements apart (8.4 MB at 1024^3 float64).  Measured on B200
// (tools/micro/stride_bw2.cu) such rows must be visited >= 256 bytes at a
// time to reach HBM bandwidth, but a CTA that owns whole columns can only
// afford 64-128 bytes per row.  So the column of length N = NA*NB is split:
//
//   pass A, task (group g, beta, block): rows r = NB*a + beta (a < NA) of W=64
//           adjacent columns -> NA-point FFT over a -> times w_N^(beta*alpha)
//           -> scratch[slot][alpha][beta][column]
//   pass B, task (group g, alpha, block): scratch[slot][alpha][*][column] ->
//           NB-point FFT over beta -> output rows k = alpha + NA*d
//
// Every HBM row visit is W*sizeof(cx) = 1 KB wide (float64).  The scratch of a
// group (N*G complex) stays in L2; groups advance through a 3-slot ring.  One
// persistent kernel runs both passes from an ordered ticket queue
// A(0), A(1), B(0), A(2), B(1), ...; a B task waits for its group's A tasks and
// an A task waits until the B tasks of the group that last used its ring slot
// have finished (global counters, release/acquire).  Tickets are handed out in
// order to resident CTAs, so every awaited task is already running: no
// deadlock.
#pragma once
#include "kernels.cuh"

namespace tffft {

constexpr int kFsThreads = 256;
constexpr int kFsSlots = 3;
constexpr int kFsMaxW = 256;    // group size G must be a multiple of every task width

// per-pass geometry: W columns per task = 256 / threads-per-column
template <typename T, int L>
struct FsPass {
  using SH = Shape<L>;
  static constexpr int N = SH::N;
  static constexpr int W = kFsThreads / SH::TPT;
  static constexpr int PS = SH::EB > 0 ? SH::EB : 30;
  // exchange column stride: S == 1 mod 16 words -> 16 adjacent columns per wavefront, no conflicts
  static constexpr int S = ((N + (N >> (PS > 20 ? 30 : PS)) + 15) / 16) * 16 + 1;
#ifndef TFFFT_FS_SPLIT
#define TFFFT_FS_SPLIT 1
#endif
  static constexpr bool SPLIT = sizeof(T) == 8 && TFFFT_FS_SPLIT;
  static constexpr size_t SMEM = (SPLIT ? 8 : sizeof(cx<T>)) * (size_t)W * S;
};

struct FourStepParams {
  void* data;             // spectral slab (in place)
  void* staging;          // inverse redirect target (p > 1) or null
  void* scratch;          // kFsSlots * N * G complex
  const void* twA;        // pass tables, length NA
  const void* twB;        // pass tables, length NB
  const void* twN;        // exp(-2 pi i t / N), t < N
  unsigned* counters;     // [0] ticket, [1, 1+ng) doneA, [1+ng, 1+2ng) doneB; zeroed per launch
  long long ncols;        // columns c in [0, ncols)
  int G;                  // columns per group (multiple of kFsMaxW)
  int ngroups;
  // element r of column c lives at c + (r & icm) * inner_stride + (r >> ic_shift) * block_stride
  int ic_shift;
  long long inner_stride, block_stride;
  // inverse redirect of block s != self_band: staging + s*stg_band + (r & bmask)*stg_within + c
  int band_shift, self_band;
  long long stg_band, stg_within;
};

// Poll a completion counter.  A relaxed (not acquire) load: ld.acquire.gpu
// compiles to CCTL.IVALL, which would invalidate this SM's whole L1 (and the
// twiddle tables in it) on every poll.  Every read of the data a counter
// publishes bypasses L1 (ld.global.cg or TMA) and the producer publishes with
// a fence + atomic after its writes completed, so L2 already holds the data.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Publish a finished task: release-ordered add.  Unlike __threadfence() +
// atomicAdd (a gpu-scope fence, CCTL.IVALL in SASS) it does not invalidate
// the SM's L1.  Called by one thread after a CTA barrier, so the release
// covers the whole CTA's writes (cumulativity).
__device__ __forceinline__ void publish_add(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

template <typename T>
__device__ __forceinline__ cx<T> ldcg_cx(const cx<T>* p) {
  auto v = __ldcg(reinterpret_cast<const typename vec2<T>::type*>(p));
  return {v.x, v.y};
}
// L2 eviction-priority policies: HBM streaming data evict_first, the scratch
// ring evict_last (it must survive from pass A to pass B)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ cx<double> ld_hint(const cx<double>* a, uint64_t pol) {
  cx<double> z;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(z.x), "=d"(z.y) : "l"(a), "l"(pol));
  return z;
}
__device__ __forceinline__ cx<float> ld_hint(const cx<float>* a, uint64_t pol) {
  cx<float> z;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
               : "=f"(z.x), "=f"(z.y) : "l"(a), "l"(pol));
  return z;
}
__device__ __forceinline__ void st_hint(cx<double>* a, cx<double> z, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(z.x), "d"(z.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(cx<float>* a, cx<float> z, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(a), "f"(z.x), "f"(z.y), "l"(pol)
               : "memory");
}
// drop an L2 line without writing it back (its scratch contents are consumed)
__device__ __forceinline__ void discard_l2(const void* a) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}

#ifndef TFFFT_FS_MINB
#define TFFFT_FS_MINB 3
#endif
template <typename T, int LA, int LB, bool INV, bool TWO, bool REDIR>
__global__ void __launch_bounds__(kFsThreads, TFFFT_FS_MINB)
fourstep_kernel(const FourStepParams prm) {
  using PA = FsPass<T, LA>;
  using PB = FsPass<T, LB>;
  using SA = Shape<LA>;
  using SB = Shape<LB>;
  constexpr int NA = SA::N, NB = SB::N, N = NA * NB;
  using STA = Stockham<T, LA, INV, PA::S, PA::PS, PA::SPLIT>;
  using STB = Stockham<T, LB, INV, PB::S, PB::PS, PB::SPLIT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_isA, s_g, s_w, s_end;

  const int t = threadIdx.x;
  cx<T>* data = reinterpret_cast<cx<T>*>(prm.data);
  cx<T>* scr = reinterpret_cast<cx<T>*>(prm.scratch);
  const cx<T>* twN = reinterpret_cast<const cx<T>*>(prm.twN);
  const unsigned is = (unsigned)prm.inner_stride, bs = (unsigned)prm.block_stride;
  const unsigned ics = (unsigned)prm.ic_shift, icm = (1u << ics) - 1u;
  auto offset = [&](unsigned r) -> unsigned {
    if constexpr (TWO) return (r & icm) * is + (r >> ics) * bs;
    else return r * is;
  };
  const int ng = prm.ngroups;
  const int blocksA = prm.G / PA::W, blocksB = prm.G / PB::W;
  const int nA = NB * blocksA, nB = NA * blocksB;
  const unsigned total = (unsigned)ng * (unsigned)(nA + nB);
  unsigned* ticket = prm.counters;
  unsigned* doneA = prm.counters + 1;
  unsigned* doneB = prm.counters + 1 + ng;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();

  // thread 0 owns the queue: it always holds the NEXT ticket, fetched while the
  // CTA works on the current task, so the atomic's round trip is hidden
  unsigned next_tk = 0;
  if (t == 0) next_tk = atomicAdd(ticket, 1u);
  for (;;) {
    if (t == 0) {
      const unsigned tk = next_tk;
      if (tk >= total) {
        s_end = 1;
      } else {
        // decode: A(0), [A(q+1), B(q)] for q < ng-1, B(ng-1)
        int isA, g, w;
        if (tk < (unsigned)nA) {
          isA = 1; g = 0; w = (int)tk;
        } else {
          const unsigned r = tk - (unsigned)nA;
          const int q = (int)(r / (unsigned)(nA + nB));
          const int x = (int)(r % (unsigned)(nA + nB));
          if (q < ng - 1 && x < nA) { isA = 1; g = q + 1; w = x; }
          else { isA = 0; g = q; w = q < ng - 1 ? x - nA : x; }
        }
        if (isA) {
          if (g >= kFsSlots)
            while (ld_acquire(doneB + (g - kFsSlots)) < (unsigned)nB) __nanosleep(64);
        } else {
          while (ld_acquire(doneA + g) < (unsigned)nA) __nanosleep(64);
        }
        s_end = 0; s_isA = isA; s_g = g; s_w = w;
        next_tk = atomicAdd(ticket, 1u);
      }
    }
    __syncthreads();
    if (s_end) break;
    const bool isA = s_isA;
    const int g = s_g, w = s_w;
    cx<T>* gscr = scr + (size_t)(g % kFsSlots) * N * prm.G;
    if (isA) {
      constexpr int W = PA::W;
      const int b = t % W, tt = t / W;
      const int beta = w / blocksA, blk = w % blocksA;
      const int lc = blk * W + b;
      const long long c_raw = (long long)g * prm.G + lc;
      const unsigned c = (unsigned)(c_raw < prm.ncols ? c_raw : prm.ncols - 1);
      cx<T> v[SA::E];
#pragma unroll
      for (int u = 0; u < SA::E / SA::R0; ++u)
#pragma unroll
        for (int m = 0; m < SA::R0; ++m)
          v[u * SA::R0 + m] = ld_hint(data + c + offset((unsigned)(NB * SA::in_elem(tt, u, m) + beta)), pol_stream);
      STA::run(smem_raw, v, tt, b, reinterpret_cast<const cx<T>*>(prm.twA));
#pragma unroll
      for (int u = 0; u < SA::E / SA::RL; ++u)
#pragma unroll
        for (int m = 0; m < SA::RL; ++m) {
          const int alpha = SA::out_elem(tt, u, m);
          const cx<T> z = ctw<INV>(v[u * SA::RL + m], ldg_cx(twN + ((beta * alpha) & (N - 1))));
          st_hint(gscr + ((size_t)alpha * NB + beta) * prm.G + lc, z, pol_keep);
        }
    } else {
      constexpr int W = PB::W;
      const int b = t % W, tt = t / W;
      const int alpha = w / blocksB, blk = w % blocksB;
      const int lc = blk * W + b;
      const long long c_raw = (long long)g * prm.G + lc;
      const bool valid = c_raw < prm.ncols;
      const unsigned c = (unsigned)(valid ? c_raw : prm.ncols - 1);
      cx<T> v[SB::E];
#pragma unroll
      for (int u = 0; u < SB::E / SB::R0; ++u)
#pragma unroll
        for (int m = 0; m < SB::R0; ++m)
          v[u * SB::R0 + m] = ldcg_cx(gscr + ((size_t)alpha * NB + SB::in_elem(tt, u, m)) * prm.G + lc);
      STB::run(smem_raw, v, tt, b, reinterpret_cast<const cx<T>*>(prm.twB));
      // the task's scratch lines (NB rows x W columns) are consumed: drop them
      // from L2 without a write-back
      __syncthreads();
      {
        constexpr int LPR = W * (int)sizeof(cx<T>) / 128;  // lines per scratch row segment
        for (int li = t; li < NB * LPR; li += kFsThreads) {
          const int beta = li / LPR, part = li % LPR;
          discard_l2(reinterpret_cast<const char*>(gscr + ((size_t)alpha * NB + beta) * prm.G + blk * W) +
                     part * 128);
        }
      }
      if (valid) {
        cx<T>* stg = reinterpret_cast<cx<T>*>(prm.staging);
        const unsigned bmask = (1u << prm.band_shift) - 1u;
#pragma unroll
        for (int u = 0; u < SB::E / SB::RL; ++u)
#pragma unroll
          for (int m = 0; m < SB::RL; ++m) {
            const unsigned r = (unsigned)(alpha + NA * SB::out_elem(tt, u, m));
            const cx<T> z = v[u * SB::RL + m];
            if constexpr (REDIR) {
              const int band = (int)(r >> prm.band_shift);
              if (band != prm.self_band) {
                st_hint(stg + (long long)band * prm.stg_band + (long long)(r & bmask) * prm.stg_within + c, z,
                        pol_stream);
                continue;
              }
            }
            st_hint(data + c + offset(r), z, pol_stream);
          }
      }
    }
    __syncthreads();  // every thread's stores issued before the completion count
    if (t == 0) publish_add(isA ? doneA + g : doneB + g);
  }
}

template <typename T, int LA, int LB>
__host__ __device__ constexpr size_t fourstep_smem_bytes() {
  return FsPass<T, LA>::SMEM > FsPass<T, LB>::SMEM ? FsPass<T, LA>::SMEM : FsPass<T, LB>::SMEM;
}

// log2 NA of the four-step split of log2 n0; 0 when n0 takes the direct kernel
__host__ __device__ constexpr int fourstep_la(int L) { return L >= 9 && L <= 12 ? (L + 1) / 2 : 0; }

template <typename T>
cudaError_t launch_fourstep(int L, bool inv, int variant, const FourStepParams& p, cudaStream_t s);

}  // namespace tffft
