// Is the L2 faster than HBM for the column-kernel access pattern?  In-place
// read+write of 128-byte x R-row tiles with row stride S, over (a) a footprint
// far larger than L2 (HBM) and (b) the same launch with every tile index
// folded into a small window (footprint `win` bytes, L2-resident).  Also a
// contiguous in-place sweep over both footprints.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tile_rw(char* buf, long long S, int R, int tiles_x, long long fold) {
  long long blk = blockIdx.x;
  if (fold > 0) blk %= fold;
  const int tx = (int)(blk % tiles_x), ty = (int)(blk / tiles_x);
  const int lane = threadIdx.x % 8, r0 = threadIdx.x / 8, rpp = blockDim.x / 8;
  char* base = buf + (long long)ty * R * S + (long long)tx * 128 + lane * 16;
  int4 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = *reinterpret_cast<int4*>(base + (long long)(r0 + i * rpp) * S);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) { v[i].x += 1; *reinterpret_cast<int4*>(base + (long long)(r0 + i * rpp) * S) = v[i]; }
}

__global__ void contig_rw(int4* buf, long long n, long long fold) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long j = fold > 0 ? i % fold : i;
    int4 v = buf[j];
    v.x += 1;
    buf[j] = v;
  }
}

int main() {
  const long long total = 8LL << 30;
  char* buf;
  if (cudaMalloc(&buf, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    launch(); launch();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms;
  };
  for (long long S : {8208LL, 8404992LL}) {
    const int R = 256 * 16 / 8;  // 256 threads, 8 lanes of 16 B per row, 16 rows per thread
    const long long rows = total / S;
    const int tiles_x = (int)(S / 128), tiles_y = (int)(rows / R);
    const long long blocks = (long long)tiles_x * tiles_y;
    const double bytes = 2.0 * blocks * R * 128;
    for (long long win : {0LL, 8LL << 20, 32LL << 20, 64LL << 20}) {
      long long fold = 0;
      if (win) fold = (win / (R * S)) * tiles_x > 0 ? (win / (R * S)) * tiles_x : (win / (R * 128));
      if (win && fold > blocks) fold = blocks;
      float ms = timeit([&] { tile_rw<<<blocks, 256>>>(buf, S, R, tiles_x, fold); });
      printf("tiles 128B x %d rows, stride %9lld, footprint %s%4lld MB: %8.1f GB/s (%s)\n", R, S, win ? "" : "all ",
             win ? win >> 20 : total >> 20, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  const long long n = total / 16;
  for (long long win : {0LL, 8LL << 20, 32LL << 20, 64LL << 20}) {
    const long long fold = win / 16;
    float ms = timeit([&] { contig_rw<<<148 * 8, 512>>>(reinterpret_cast<int4*>(buf), n, fold); });
    printf("contiguous in-place, footprint %4lld MB: %8.1f GB/s\n", win ? win >> 20 : total >> 20, 2.0 * total / ms / 1e6);
  }
  return 0;
}
