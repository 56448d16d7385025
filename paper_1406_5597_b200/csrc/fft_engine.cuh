// Register/shared-memory Stockham FFT engine for sm_100a.
//
// One length-N complex transform (N = 2^L, L <= 12) is owned by TPT = N/E
// threads; each thread keeps E complex values in registers.  A transform runs
// as P = ceil(L/4) radix passes (radix <= 16).  Pass 0 reads its operands
// straight from global memory and the last pass writes its results straight
// to global memory; the P-1 exchanges in between go through shared memory.
//
// Stockham autosort indexing (pass with radix R, Ns = product of earlier
// radices, butterfly j in [0, N/R), k = j mod Ns):
//   in : x[j + m*N/R]                        m = 0..R-1
//   tw : v[m] *= exp(-+2*pi*i*m*k/(Ns*R))
//   out: y[(j/Ns)*Ns*R + k + m*Ns]  = DFT_R(v)[m]
// The first pass has Ns = 1 (no twiddles) and the last Ns*R = N, so its
// outputs land in natural order at x[j + m*N/R].
//
// This replaces the reference's radix-2 bit-reversal DIT loop
// (reference pkg/src/slabfft/kernels.py:134-161): same unnormalised DFT,
// same sign convention (forward exp(-2*pi*i...), kernels.py:41-45).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tffft {

// ---------------------------------------------------------------------------
// radix schedule (shared by host table builder and device code)
// ---------------------------------------------------------------------------
constexpr int kMaxRadixBits = 4;
constexpr int kMaxLog = 12;
#ifndef TFFFT_L10_RADIX_BITS
#define TFFFT_L10_RADIX_BITS 5
#endif
// largest radix (bits) of a length-2^L schedule; E = 2^(first radix bits)
// operands per thread
#ifndef TFFFT_L9_RADIX_BITS
#define TFFFT_L9_RADIX_BITS 5
#endif
__host__ __device__ constexpr int max_radix_bits(int L) {
  return L == 10 ? TFFFT_L10_RADIX_BITS : L == 9 ? TFFFT_L9_RADIX_BITS : kMaxRadixBits;
}

// Every schedule function takes an optional mb = largest radix in bits
// (default: max_radix_bits(L)); a kernel may run its own schedule, see
// r2c_radix_bits in kernels.cuh.  The host table builder uses the same functions.
__host__ __device__ constexpr int sched_bits(int L, int mb) { return mb > 0 ? mb : max_radix_bits(L); }
__host__ __device__ constexpr int num_passes(int L, int mb = 0) {
  return L == 0 ? 0 : (L + sched_bits(L, mb) - 1) / sched_bits(L, mb);
}
__host__ __device__ constexpr int pass_bits(int L, int p, int mb = 0) {
  return (L / num_passes(L, mb)) + (p < (L % num_passes(L, mb)) ? 1 : 0);
}
__host__ __device__ constexpr int ept_bits(int L, int mb = 0) { return L == 0 ? 0 : pass_bits(L, 0, mb); }
__host__ __device__ constexpr int ns_bits(int L, int p, int mb = 0) {
  return p == 0 ? 0 : ns_bits(L, p - 1, mb) + pass_bits(L, p - 1, mb);
}
// offset of pass p's twiddle block (passes >= 1 only); block p holds the Ns
// roots exp(-2 pi i k / (Ns R)), k < Ns; powers m = 2..R-1 are formed in registers
__host__ __device__ constexpr int tw_offset(int L, int p, int mb = 0) {
  return p <= 1 ? 0 : tw_offset(L, p - 1, mb) + (1 << ns_bits(L, p - 1, mb));
}
__host__ __device__ constexpr int tw_total(int L, int mb = 0) {
  return num_passes(L, mb) <= 1 ? 0
                                : tw_offset(L, num_passes(L, mb) - 1, mb) + (1 << ns_bits(L, num_passes(L, mb) - 1, mb));
}

// ---------------------------------------------------------------------------
// complex arithmetic
// ---------------------------------------------------------------------------
template <typename T> struct vec2;
template <> struct vec2<double> { using type = double2; };
template <> struct vec2<float> { using type = float2; };

template <typename T>
struct __align__(2 * sizeof(T)) cx {
  T x, y;
};

template <typename T>
__device__ __forceinline__ cx<T> cadd(cx<T> a, cx<T> b) { return {a.x + b.x, a.y + b.y}; }
template <typename T>
__device__ __forceinline__ cx<T> csub(cx<T> a, cx<T> b) { return {a.x - b.x, a.y - b.y}; }
// a * w
template <typename T>
__device__ __forceinline__ cx<T> cmul(cx<T> a, cx<T> w) {
  return {fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x)};
}
// a * conj(w)
template <typename T>
__device__ __forceinline__ cx<T> cmulc(cx<T> a, cx<T> w) {
  return {fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y)};
}
// multiply by the direction's twiddle: forward w, inverse conj(w)
template <bool INV, typename T>
__device__ __forceinline__ cx<T> ctw(cx<T> a, cx<T> w) {
  if constexpr (INV) return cmulc(a, w); else return cmul(a, w);
}

template <typename T>
__device__ __forceinline__ cx<T> ldg_cx(const cx<T>* p) {
  auto v = __ldg(reinterpret_cast<const typename vec2<T>::type*>(p));
  return {v.x, v.y};
}
// twiddle fetch from global (read-only path) or, with TWS, from a shared-memory copy
template <bool TWS, typename T>
__device__ __forceinline__ cx<T> tw_cx(const cx<T>* p) {
  if constexpr (TWS) return *p; else return ldg_cx(p);
}

// w^m for m = 1..R-1 by a balanced product tree (depth <= log2 R), from one
// table load instead of R-1: trades L1 wavefronts for idle FP64 issue slots.
__host__ __device__ constexpr int hibit(int m) { return m < 2 ? m : 2 * hibit(m / 2); }

template <int M, int R, typename T>
__device__ __forceinline__ void twiddle_powers_from(cx<T>* pw) {
  if constexpr (M < R) {
    constexpr int HI = hibit(M);
    if constexpr (M == HI) pw[M] = cmul(pw[M / 2], pw[M / 2]);
    else pw[M] = cmul(pw[HI], pw[M - HI]);
    twiddle_powers_from<M + 1, R>(pw);
  }
}
template <int R, typename T>
__device__ __forceinline__ void twiddle_powers(cx<T> w, cx<T>* pw) {
  pw[1] = w;
  twiddle_powers_from<2, R>(pw);
}

// ---------------------------------------------------------------------------
// small DFTs in registers: a[0..R-1] -> DFT_R(a), natural order
// ---------------------------------------------------------------------------
// exp(-2*pi*i*t/16) for the forward direction; INV conjugates.
template <bool INV, typename T>
__device__ __forceinline__ cx<T> mul_w16(cx<T> a, int t) {
  const T c1 = T(0.923879532511286756128183189396788933);
  const T s1 = T(0.382683432365089771728459984030398866);
  const T h = T(0.707106781186547524400844362104849039);
  // forward: w = cos - i sin; multiply a by w
  T c, s;
  switch (t & 15) {
    case 0: return a;
    case 4: return INV ? cx<T>{-a.y, a.x} : cx<T>{a.y, -a.x};
    case 8: return {-a.x, -a.y};
    case 12: return INV ? cx<T>{a.y, -a.x} : cx<T>{-a.y, a.x};
    case 2: c = h; s = h; break;
    case 6: c = -h; s = h; break;
    case 10: c = -h; s = -h; break;
    case 14: c = h; s = -h; break;
    case 1: c = c1; s = s1; break;
    case 3: c = s1; s = c1; break;
    case 5: c = -s1; s = c1; break;
    case 7: c = -c1; s = s1; break;
    case 9: c = -c1; s = -s1; break;
    case 11: c = -s1; s = -c1; break;
    case 13: c = s1; s = -c1; break;
    default: c = c1; s = -s1; break;  // 15
  }
  if (INV) s = -s;
  // (a.x + i a.y)(c - i s)
  return {fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s)};
}

// exp(-2*pi*i*t/32), t < 16 (even t via mul_w16)
template <bool INV, typename T>
__device__ __forceinline__ cx<T> mul_w32(cx<T> a, int t) {
  if ((t & 1) == 0) return mul_w16<INV>(a, t >> 1);
  const T k1 = T(0.980785280403230449126182236134239037);
  const T k3 = T(0.831469612302545237078788377617905756);
  const T k5 = T(0.555570233019602224742830813948532874);
  const T k7 = T(0.195090322016128267848284868477022240);
  T c, s;
  switch (t & 15) {
    case 1: c = k1; s = k7; break;
    case 3: c = k3; s = k5; break;
    case 5: c = k5; s = k3; break;
    case 7: c = k7; s = k1; break;
    case 9: c = -k7; s = k1; break;
    case 11: c = -k5; s = k3; break;
    case 13: c = -k3; s = k5; break;
    default: c = -k1; s = k7; break;  // 15
  }
  if (INV) s = -s;
  return {fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s)};
}

template <int R, bool INV, typename T>
struct DFT {
  static __device__ __forceinline__ void run(cx<T>* a) {
    static_assert(R <= 32, "radix above 32");
    constexpr int H = R / 2;
    cx<T> e[H], o[H];
#pragma unroll
    for (int i = 0; i < H; ++i) { e[i] = a[2 * i]; o[i] = a[2 * i + 1]; }
    DFT<H, INV, T>::run(e);
    DFT<H, INV, T>::run(o);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      cx<T> t = mul_w32<INV>(o[k], k * (32 / R));
      a[k] = cadd(e[k], t);
      a[k + H] = csub(e[k], t);
    }
  }
};
template <bool INV, typename T>
struct DFT<1, INV, T> {
  static __device__ __forceinline__ void run(cx<T>*) {}
};
template <bool INV, typename T>
struct DFT<2, INV, T> {
  static __device__ __forceinline__ void run(cx<T>* a) {
    cx<T> t = a[0];
    a[0] = cadd(t, a[1]);
    a[1] = csub(t, a[1]);
  }
};
template <bool INV, typename T>
struct DFT<4, INV, T> {
  static __device__ __forceinline__ void run(cx<T>* a) {
    cx<T> t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
    cx<T> t2 = cadd(a[1], a[3]), d = csub(a[1], a[3]);
    // forward: -i*d ; inverse: +i*d
    cx<T> t3 = INV ? cx<T>{-d.y, d.x} : cx<T>{d.y, -d.x};
    a[0] = cadd(t0, t2);
    a[2] = csub(t0, t2);
    a[1] = cadd(t1, t3);
    a[3] = csub(t1, t3);
  }
};

// ---------------------------------------------------------------------------
// async copy helpers (LDGSTS)
// ---------------------------------------------------------------------------
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}
// bulk L2 prefetch (TMA unit): bytes multiple of 16, address 16-byte aligned
__device__ __forceinline__ void prefetch_l2(const void* gmem, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// Stockham pass machinery
// ---------------------------------------------------------------------------
template <int L, int MB = 0>
struct Shape {
  static constexpr int N = 1 << L;
  static constexpr int P = num_passes(L, MB);
  static constexpr int EB = ept_bits(L, MB);
  static constexpr int E = 1 << EB;
  static constexpr int TPT = N / E;  // threads per transform
  static constexpr int R0 = L == 0 ? 1 : (1 << pass_bits(L, 0, MB));
  static constexpr int RL = L == 0 ? 1 : (1 << pass_bits(L, P - 1, MB));
  static constexpr int TW = tw_total(L, MB);
  // element index held in v[u*R0+m] before pass 0 / in v[u*RL+m] after the last pass
  static __device__ __forceinline__ int in_elem(int tt, int u, int m) { return tt + TPT * u + m * (N / R0); }
  static __device__ __forceinline__ int out_elem(int tt, int u, int m) { return tt + TPT * u + m * (N / RL); }
  // register slot of pass-0 input element tt + TPT*k (k < E)
  static __device__ __forceinline__ constexpr int in_slot(int k) { return (k % (E / R0)) * R0 + k / (E / R0); }
};

// Exchange buffer: element a of transform b at b*S + a + (a >> PS).  With
// SPLIT (float64) the exchange runs in two rounds of 8-byte words (real parts,
// then imaginary parts), halving the buffer; otherwise whole complex values.
// SYNC: 0 = __syncthreads; 32 = __syncwarp (every transform inside one warp);
// otherwise the CTA is split into independent groups of SYNC threads and group
// g = tid / SYNC synchronises on named barrier 1 + g.
template <typename T, int L, bool INV, int S, int PS, bool SPLIT = false, int SYNC = 0, bool TWS = false, int MB = 0>
struct Stockham {
  static __device__ __forceinline__ void sync() {
    if constexpr (SYNC == 0) __syncthreads();
    else if constexpr (SYNC == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.x / SYNC), "n"(SYNC) : "memory");
  }
  using SH = Shape<L, MB>;
  static constexpr int N = SH::N, E = SH::E, TPT = SH::TPT, P = SH::P;

  static __device__ __forceinline__ int sidx(int b, int a) { return b * S + a + (a >> PS); }

  template <int p>
  static __device__ __forceinline__ void compute(cx<T>* v, int tt, const cx<T>* __restrict__ tw) {
    constexpr int R = 1 << pass_bits(L, p, MB);
    constexpr int NS = 1 << ns_bits(L, p, MB);
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      if constexpr (p > 0) {
        const int j = tt + TPT * u;
        const int k = j & (NS - 1);
        cx<T> pw[R];
        twiddle_powers<R>(tw_cx<TWS>(tw + tw_offset(L, p, MB) + k), pw);
#pragma unroll
        for (int m = 1; m < R; ++m) v[u * R + m] = ctw<INV>(v[u * R + m], pw[m]);
      }
      DFT<R, INV, T>::run(v + u * R);
    }
  }

  // COMP: 0 = real part, 1 = imaginary part, 2 = whole complex value
  template <int COMP>
  static __device__ __forceinline__ void put(void* sm, int i, const cx<T>& x) {
    if constexpr (COMP == 2) reinterpret_cast<cx<T>*>(sm)[i] = x;
    else reinterpret_cast<T*>(sm)[i] = COMP == 0 ? x.x : x.y;
  }
  template <int COMP>
  static __device__ __forceinline__ void get(const void* sm, int i, cx<T>& x) {
    if constexpr (COMP == 2) x = reinterpret_cast<const cx<T>*>(sm)[i];
    else if constexpr (COMP == 0) x.x = reinterpret_cast<const T*>(sm)[i];
    else x.y = reinterpret_cast<const T*>(sm)[i];
  }

  template <int p, int COMP>
  static __device__ __forceinline__ void store(void* sm, const cx<T>* v, int tt, int b) {
    constexpr int R = 1 << pass_bits(L, p, MB);
    constexpr int NS = 1 << ns_bits(L, p, MB);
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      const int j = tt + TPT * u;
      const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
      for (int m = 0; m < R; ++m) put<COMP>(sm, sidx(b, base + m * NS), v[u * R + m]);
    }
  }

  template <int p, int COMP>
  static __device__ __forceinline__ void load(const void* sm, cx<T>* v, int tt, int b) {
    constexpr int R = 1 << pass_bits(L, p, MB);
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      const int j = tt + TPT * u;
#pragma unroll
      for (int m = 0; m < R; ++m) get<COMP>(sm, sidx(b, j + m * (N / R)), v[u * R + m]);
    }
  }

  template <int p>
  static __device__ __forceinline__ void exchange(void* sm, cx<T>* v, int tt, int b) {
    if constexpr (SPLIT) {
      store<p - 1, 0>(sm, v, tt, b);
      sync();
      load<p, 0>(sm, v, tt, b);
      sync();
      store<p - 1, 1>(sm, v, tt, b);
      sync();
      load<p, 1>(sm, v, tt, b);
      sync();
    } else {
      store<p - 1, 2>(sm, v, tt, b);
      sync();
      load<p, 2>(sm, v, tt, b);
      sync();
    }
  }

  // hook() runs once the last exchange has drained the buffer (every thread
  // has loaded its operands of the last pass), before that pass computes
  template <int p, class Hook>
  static __device__ __forceinline__ void rest(void* sm, cx<T>* v, int tt, int b, const cx<T>* __restrict__ tw,
                                              Hook& hook) {
    if constexpr (p < P) {
      exchange<p>(sm, v, tt, b);
      if constexpr (p == P - 1) hook();
      compute<p>(v, tt, tw);
      rest<p + 1>(sm, v, tt, b, tw, hook);
    }
  }
  struct NoHook {
    __device__ __forceinline__ void operator()() const {}
  };

  // v holds pass-0 inputs (element in_elem(tt,u,m) in v[u*R0+m]); on return
  // v[u*RL+m] holds output element out_elem(tt,u,m).  All threads of the CTA
  // must call this (it synchronises when P > 1).  run = first() + finish().
  static __device__ __forceinline__ void first(cx<T>* v, int tt, const cx<T>* __restrict__ tw) {
    if constexpr (P > 0) compute<0>(v, tt, tw);
  }
  static __device__ __forceinline__ void finish(void* sm, cx<T>* v, int tt, int b, const cx<T>* __restrict__ tw) {
    NoHook h;
    if constexpr (P > 0) rest<1>(sm, v, tt, b, tw, h);
  }
  template <class Hook>
  static __device__ __forceinline__ void finish(void* sm, cx<T>* v, int tt, int b, const cx<T>* __restrict__ tw,
                                                Hook& hook) {
    if constexpr (P > 0) rest<1>(sm, v, tt, b, tw, hook);
  }
  static __device__ __forceinline__ void run(void* sm, cx<T>* v, int tt, int b, const cx<T>* __restrict__ tw) {
    first(v, tt, tw);
    finish(sm, v, tt, b, tw);
  }

  // write the final outputs into smem at their natural index (for the real
  // transforms' post-processing that pairs bins k and N-k); whole complex values
  static __device__ __forceinline__ void store_natural(cx<T>* sm, const cx<T>* v, int tt, int b) {
    constexpr int RL = SH::RL;
#pragma unroll
    for (int u = 0; u < E / RL; ++u)
#pragma unroll
      for (int m = 0; m < RL; ++m) sm[sidx(b, SH::out_elem(tt, u, m))] = v[u * RL + m];
  }
};

}  // namespace tffft
