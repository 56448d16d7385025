// Copy bandwidth of the column-kernel access pattern versus row-visit width and
// bytes in flight.  One persistent CTA per SM: a producer thread streams 32 KB
// TMA boxes (W float64 x 4096/W rows of a matrix with row stride S) into a
// K-stage shared ring; 128 threads write each box back in place with 16-byte
// stores, as the column kernel's epilogue does.  S = 8.4 MB (stage 3 at
// 1024^3) or 8208 B (stage 1b).  Prints GB/s (read + write).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void mb_tx(uint64_t* b, unsigned tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned par) {
  unsigned done = 0;
  while (!done) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(su(b)), "r"(par) : "memory");
}

template <int K>
__global__ void __launch_bounds__(160, 1) stream(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap wide,
                                                 char* base, long long rowb, int tiles, int W, int R, int nq, int pf) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + K * 32768);
  uint64_t* empty = full + K;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < K; ++s) { mb_init(full + s, 1); mb_init(empty + s, 128); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int mine = tiles > (int)blockIdx.x ? (tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (t >= 128) {  // producer warp
    if (t == 128) {
      for (int i = 0; i < mine; ++i) {
        const int s = i % K;
        mb_wait(empty + s, ((i / K) & 1) ^ 1);
        const int tile = blockIdx.x + i * gridDim.x, cb = tile / nq, q = tile % nq;
        if (pf && (cb & 1) == 0)  // L2 prefetch of the 2W-wide segment this tile and its neighbour share
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&wide), "r"(cb * W), "r"(q * R) : "memory");
        mb_tx(full + s, 32768);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su(sm + s * 32768)), "l"(&map), "r"(cb * W), "r"(q * R), "r"(su(full + s)) : "memory");
      }
    }
    return;
  }
  const int cpr = W / 2;  // 16-byte chunks per box row
  for (int i = 0; i < mine; ++i) {
    const int s = i % K;
    mb_wait(full + s, (i / K) & 1);
    const int tile = blockIdx.x + i * gridDim.x, cb = tile / nq, q = tile % nq;
    const int4* src = reinterpret_cast<const int4*>(sm + s * 32768);
#pragma unroll 4
    for (int c = t; c < 2048; c += 128) {
      const int r = c / cpr, k = c % cpr;
      *reinterpret_cast<int4*>(base + (long long)(q * R + r) * rowb + (long long)cb * W * 8 + k * 16) = src[c];
    }
    mb_arrive(empty + s);
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int K>
int run(const CUtensorMap& map, const CUtensorMap& wide, char* buf, long long rowb, long long rows, int W, int nsm, int pf) {
  auto k = stream<K>;
  const int smem = K * 32768 + 2 * K * 8 + 64;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int R = 4096 / W, nq = (int)(rows / R), ncb = (int)(rowb / (W * 8));
  const int tiles = ncb * nq;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<nsm, 160, smem>>>(map, wide, buf, rowb, tiles, W, R, nq, pf);
  cudaEventRecord(a);
  for (int it = 0; it < 3; ++it) k<<<nsm, 160, smem>>>(map, wide, buf, rowb, tiles, W, R, nq, pf);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = 3.0 * 2.0 * (double)tiles * 32768;
  printf("stride %8lld B, box %4d B x %3d rows, K=%d (%3d KB in flight/SM)%s: %7.1f GB/s\n", rowb, W * 8, R, K, K * 32,
         pf ? " + 2x-wide L2 prefetch" : "", bytes / ms / 1e6);
  return 0;
}

int main() {
  const long long total = 8404992LL * 1024;  // the 1024^3 float64 spectral slab
  char* buf;
  CK(cudaMalloc(&buf, total));
  CK(cudaMemset(buf, 0, total));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  Enc enc = reinterpret_cast<Enc>(fn);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (long long rb : {8404992LL, 8208LL}) {
    const long long nrows = total / rb;
    for (int W : {16, 32}) {  // doubles per box row: 128 B, 256 B
      CUtensorMap map, wide;
      cuuint64_t dims[2] = {(cuuint64_t)(rb / 8), (cuuint64_t)nrows};
      cuuint64_t strides[1] = {(cuuint64_t)rb};
      cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)(4096 / W)}, boxw[2] = {(cuuint32_t)(2 * W), (cuuint32_t)(4096 / W)};
      cuuint32_t es[2] = {1, 1};
      if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
          enc(&wide, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, boxw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
      }
      run<2>(map, wide, buf, rb, nrows, W, nsm, 0);
      run<2>(map, wide, buf, rb, nrows, W, nsm, 1);
      run<4>(map, wide, buf, rb, nrows, W, nsm, 1);
    }
  }
  return 0;
}
