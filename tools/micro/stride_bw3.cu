// Row-visit width vs row stride: in-place read+write of W-byte x R-row tiles
// over ~8.6 GB, for strides below / above the 2 MB GPU page.  If 128-byte
// visits lose only when every row of a tile sits in a different page, the
// stage-3 limit is address translation rather than DRAM row locality.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tile_rw(char* buf, long long S, long long rows, int R, int W, long long tiles_x) {
  const long long tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int lanes = W / 16, rpp = blockDim.x / lanes;
  const int lane = threadIdx.x % lanes, r0 = threadIdx.x / lanes;
  char* base = buf + ty * R * S + tx * W + lane * 16;
  int4 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = *reinterpret_cast<int4*>(base + (long long)(r0 + i * rpp) * S);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) { v[i].x += 1; *reinterpret_cast<int4*>(base + (long long)(r0 + i * rpp) * S) = v[i]; }
}

int main() {
  const long long total = 8404992LL * 1024;
  char* buf;
  if (cudaMalloc(&buf, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const long long strides[] = {8192, 65536, 262144, 1048576, 2097152, 4194304, 8404992};
  for (long long S : strides) {
    for (int W : {64, 128, 256}) {
      const int threads = 512, R = threads * 16 / (W / 16);  // rows per CTA
      const long long rows = total / S;
      const long long tiles_x = S / W, tiles_y = rows / R;
      const long long blocks = tiles_x * tiles_y;
      const double bytes = 2.0 * (double)blocks * R * W;
      for (int it = 0; it < 2; ++it) tile_rw<<<(unsigned)blocks, threads>>>(buf, S, rows, R, W, tiles_x);
      cudaEventRecord(a);
      tile_rw<<<(unsigned)blocks, threads>>>(buf, S, rows, R, W, tiles_x);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("stride %8lld B  W=%4d  rows/CTA=%4d : %7.1f GB/s  (%s)\n", S, W, R, bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
