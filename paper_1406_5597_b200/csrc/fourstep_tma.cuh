// Stage 3 / 3' (p = 1) as a TMA-fed, warp-specialised four-step (sm_100a).
//
// Same decomposition as fourstep.cuh (N = NA*NB; pass A over rows NB*a+beta,
// twiddle, L2 scratch ring; pass B over the scratch, rows alpha+NA*d), but
// every task's 32 KB tile moves with ONE tensor-memory-access instruction
// instead of per-element loads and stores:
//
//   warp 8  (producer): ticket queue + dependency waits, then
//           cp.async.bulk.tensor load of the task's box into a 2-stage ring,
//           completion on the stage's "full" mbarrier (expect_tx)
//   warps 0-7 (consumers): shared -> registers -> NA/NB-point Stockham FFT
//           (exchanges on named barrier 1) -> twiddle -> results written back
//           into the same stage -> "ready" mbarrier
//   warp 9  (store): cp.async.bulk.tensor store of the stage, waits for the
//           smem reads ("empty" -> producer may refill) and for completion of
//           the writes, then publishes the task on the group's done counter
//
// HBM row visits are W*16 = 1 KB wide; the global address arithmetic lives in
// the tensor maps, so the consumers execute only shared-memory and FP64 work.
#pragma once
#include <cuda.h>

#include "fourstep.cuh"
#include "stage1_fused.cuh"

namespace tffft {

constexpr int kFtConsumers = 256;
constexpr int kFtThreads = kFtConsumers + 64;
constexpr int kFtStages = 2;

struct FsTmaParams {
  const void* twA;
  const void* twB;
  const void* twN;
  unsigned* counters;  // [0] ticket, [1, 1+ng) doneA, [1+ng, 1+2ng) doneB
  const void* scratch; // for discarding consumed scratch lines
  int ngroups, G;
};

// ---------------------------------------------------------------------------
// mbarrier / TMA primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}
// TMA tile moves with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                          uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, int c0, int c1, int c2, const void* src,
                                           uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;"
               ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_store4(const CUtensorMap* map, int c0, int c1, int c2, int c3, const void* src,
                                           uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], [%5], %6;"
               ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, unsigned parity) {
  unsigned done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait1() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kFtConsumers) : "memory"); }

template <typename T, int LA, int LB>
struct FtCfg {
  using PA = FsPass<T, LA>;
  using PB = FsPass<T, LB>;
  static constexpr int NA = 1 << LA, NB = 1 << LB;
  static_assert(PA::W == PB::W, "one column width for both passes");
  static constexpr int W = PA::W;
  static constexpr size_t STAGE = sizeof(cx<T>) * (size_t)W * (NA > NB ? NA : NB);
  static constexpr size_t XCHG = PA::SMEM > PB::SMEM ? PA::SMEM : PB::SMEM;
  // twiddles copied into shared memory per CTA: pass tables of both lengths + w_N^t, t < N
  static constexpr int TWA = Shape<LA>::TW > 0 ? Shape<LA>::TW : 1, TWB = Shape<LB>::TW > 0 ? Shape<LB>::TW : 1;
  static constexpr size_t TWBYTES = sizeof(cx<T>) * (size_t)(TWA + TWB + NA * NB);
  static constexpr size_t SMEM = kFtStages * STAGE + XCHG + TWBYTES + 1024;  // + barriers / descriptors
};

template <typename T, int LA, int LB, bool INV>
__global__ void __launch_bounds__(kFtThreads)
fourstep_tma_kernel(const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_out,
                    const __grid_constant__ CUtensorMap map_scr_a, const __grid_constant__ CUtensorMap map_scr_b,
                    const FsTmaParams prm) {
  using CF = FtCfg<T, LA, LB>;
  using SA = Shape<LA>;
  using SB = Shape<LB>;
  using PA = FsPass<T, LA>;
  using PB = FsPass<T, LB>;
  constexpr int NA = CF::NA, NB = CF::NB, N = NA * NB, W = CF::W;
  using STA = Stockham<T, LA, INV, PA::S, PA::PS, PA::SPLIT, kFtConsumers, true>;
  using STB = Stockham<T, LB, INV, PB::S, PB::PS, PB::SPLIT, kFtConsumers, true>;

  extern __shared__ __align__(1024) unsigned char smem_tma[];
  cx<T>* stage0 = reinterpret_cast<cx<T>*>(smem_tma);
  unsigned char* xbuf = smem_tma + kFtStages * CF::STAGE;
  cx<T>* s_twA = reinterpret_cast<cx<T>*>(xbuf + CF::XCHG);
  cx<T>* s_twB = s_twA + CF::TWA;
  cx<T>* s_twN = s_twB + CF::TWB;
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(s_twA) + CF::TWBYTES);
  uint64_t* empty = full + kFtStages;
  uint64_t* ready = empty + kFtStages;
  int* desc = reinterpret_cast<int*>(ready + kFtStages);  // [stage][4]: end, isA, g, w

  const int t = threadIdx.x;
  const int warp = t / 32, lane = t % 32;
  const int ng = prm.ngroups;
  const int blocks = prm.G / W;
  const int nA = NB * blocks, nB = NA * blocks;
  const unsigned total = (unsigned)ng * (unsigned)(nA + nB);
  unsigned* doneA = prm.counters + 1;
  unsigned* doneB = prm.counters + 1 + ng;

  if (t == 0) {
    for (int s = 0; s < kFtStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
      mbar_init(ready + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {  // twiddles -> shared memory (an L1 invalidation by a completion fence cannot evict them)
    const cx<T>* ga = reinterpret_cast<const cx<T>*>(prm.twA);
    const cx<T>* gb = reinterpret_cast<const cx<T>*>(prm.twB);
    const cx<T>* gn = reinterpret_cast<const cx<T>*>(prm.twN);
    for (int k = t; k < CF::TWA; k += kFtThreads) s_twA[k] = ga[k];
    for (int k = t; k < CF::TWB; k += kFtThreads) s_twB[k] = gb[k];
    for (int k = t; k < N; k += kFtThreads) s_twN[k] = gn[k];
  }
  __syncthreads();

  if (warp == kFtConsumers / 32) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_norm = policy_evict_last();
      unsigned next_tk = atomicAdd(prm.counters, 1u);  // one ticket ahead: the atomic's latency is hidden
      for (unsigned i = 0;; ++i) {
        const int s = i % kFtStages;
        const unsigned tk = next_tk;
        if (tk < total) next_tk = atomicAdd(prm.counters, 1u);
        mbar_wait(empty + s, ((i / kFtStages) & 1) ^ 1);
        int* d = desc + 4 * s;
        if (tk >= total) {
          d[0] = 1;
          mbar_arrive(full + s);
          break;
        }
        int isA, g, w;
        queue_decode(tk, ng, nA, nB, 1, isA, g, w);  // A(g+1) interleaves with B(g); A(g) needs B(g-3): 3 ring slots
        if (isA) {
          if (g >= kFsSlots)
            while (ld_acquire(doneB + (g - kFsSlots)) < (unsigned)nB) __nanosleep(64);
        } else {
          while (ld_acquire(doneA + g) < (unsigned)nA) __nanosleep(64);
        }
        d[0] = 0; d[1] = isA; d[2] = g; d[3] = w;
        mbar_arrive_tx(full + s, (unsigned)((isA ? NA : NB) * W * sizeof(cx<T>)));
        cx<T>* dst = stage0 + (size_t)s * (CF::STAGE / sizeof(cx<T>));
        if (isA) {
          const int beta = w / blocks, blk = w % blocks;
          tma_load3(dst, &map_in, 2 * (g * prm.G + blk * W), 0, beta, full + s, pol_stream);
        } else {
          const int alpha = w / blocks, blk = w % blocks;
          tma_load4(dst, &map_scr_b, 2 * blk * W, alpha, 0, g % kFsSlots, full + s, pol_norm);
        }
      }
    }
    return;
  }
  if (warp == kFtConsumers / 32 + 1) {
    // ------------------------------------------------------------ store
    // Up to two stores in flight; a task is published (done counter) once its
    // writes are complete.  When no further task is ready the warp flushes, so
    // a producer waiting on a done counter never waits on an idle store warp.
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      int pend_isA = -1, pend_g = 0;  // stored, not yet published
      auto publish = [&](int isA, int g) {
        fence_async_global();
        publish_add(isA ? doneA + g : doneB + g);
      };
      for (unsigned i = 0;; ++i) {
        const int s = i % kFtStages;
        const unsigned par = (i / kFtStages) & 1;
        if (pend_isA >= 0 && !mbar_test(ready + s, par)) {
          bulk_wait0();
          publish(pend_isA, pend_g);
          pend_isA = -1;
        }
        mbar_wait(ready + s, par);
        const int* d = desc + 4 * s;
        if (d[0]) break;
        const int isA = d[1], g = d[2], w = d[3];
        const cx<T>* src = stage0 + (size_t)s * (CF::STAGE / sizeof(cx<T>));
        if (isA) {
          const int beta = w / blocks, blk = w % blocks;
          tma_store4(&map_scr_a, 2 * blk * W, 0, beta, g % kFsSlots, src, pol_keep);
        } else {
          const int alpha = w / blocks, blk = w % blocks;
          tma_store3(&map_out, 2 * (g * prm.G + blk * W), 0, alpha, src, pol_stream);
        }
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(empty + s);  // the producer may refill the stage
        if (pend_isA >= 0) {
          bulk_wait1();  // the previous store's writes are complete
          publish(pend_isA, pend_g);
        }
        pend_isA = isA;
        pend_g = g;
      }
      if (pend_isA >= 0) {
        bulk_wait0();
        publish(pend_isA, pend_g);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const cx<T>* twN = s_twN;
  const int b = t % W, tt = t / W;
  for (unsigned i = 0;; ++i) {
    const int s = i % kFtStages;
    mbar_wait(full + s, (i / kFtStages) & 1);
    const int* d = desc + 4 * s;
    if (d[0]) {
      if (t == 0) mbar_arrive(ready + s);  // let the store warp see the end marker
      break;
    }
    const int isA = d[1], w = d[3];
    cx<T>* st = stage0 + (size_t)s * (CF::STAGE / sizeof(cx<T>));
    if (isA) {
      const int beta = w / blocks;
      cx<T> tw8[SA::E];  // epilogue twiddles issued before the FFT so their latency hides behind it
#pragma unroll
      for (int u = 0; u < SA::E / SA::RL; ++u)
#pragma unroll
        for (int m = 0; m < SA::RL; ++m)
          tw8[u * SA::RL + m] = twN[(beta * SA::out_elem(tt, u, m)) & (N - 1)];
      cx<T> v[SA::E];
#pragma unroll
      for (int u = 0; u < SA::E / SA::R0; ++u)
#pragma unroll
        for (int m = 0; m < SA::R0; ++m) v[u * SA::R0 + m] = st[SA::in_elem(tt, u, m) * W + b];
      STA::run(xbuf, v, tt, b, s_twA);
      consumer_bar();  // every thread's stage reads are done before it is overwritten
#pragma unroll
      for (int u = 0; u < SA::E / SA::RL; ++u)
#pragma unroll
        for (int m = 0; m < SA::RL; ++m) {
          const int alpha = SA::out_elem(tt, u, m);
          st[alpha * W + b] = ctw<INV>(v[u * SA::RL + m], tw8[u * SA::RL + m]);
        }
    } else {
      {  // the task's scratch tile has landed in shared memory: drop it from L2 unwritten
        const int g = d[2], alpha = w / blocks, blk = w % blocks;
        constexpr int LPR = W * (int)sizeof(cx<T>) / 128;
        const char* base = reinterpret_cast<const char*>(prm.scratch) +
                           ((((size_t)(g % kFsSlots) * N + (size_t)alpha * NB) * prm.G) + (size_t)blk * W) * sizeof(cx<T>);
        for (int li = t; li < NB * LPR; li += kFtConsumers)
          discard_l2(base + (size_t)(li / LPR) * prm.G * sizeof(cx<T>) + (li % LPR) * 128);
      }
      cx<T> v[SB::E];
#pragma unroll
      for (int u = 0; u < SB::E / SB::R0; ++u)
#pragma unroll
        for (int m = 0; m < SB::R0; ++m) v[u * SB::R0 + m] = st[SB::in_elem(tt, u, m) * W + b];
      STB::run(xbuf, v, tt, b, s_twB);
      consumer_bar();
#pragma unroll
      for (int u = 0; u < SB::E / SB::RL; ++u)
#pragma unroll
        for (int m = 0; m < SB::RL; ++m) st[SB::out_elem(tt, u, m) * W + b] = v[u * SB::RL + m];
    }
    fence_async_shared();  // generic-proxy smem writes -> visible to the TMA store
    consumer_bar();
    if (t == 0) mbar_arrive(ready + s);
  }
}

// four-step TMA path available for log2 n0 in [9, 12] when both passes share a column width
__host__ __device__ constexpr bool fourstep_tma_supported(int L) { return L == 10 || L == 12; }

template <typename T>
cudaError_t launch_fourstep_tma(int L, bool inv, const CUtensorMap* maps, const FsTmaParams& p, cudaStream_t s);

}  // namespace tffft
