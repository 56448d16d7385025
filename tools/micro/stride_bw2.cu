// In-place read+write of W-byte-wide, R-row tiles of a (rows x S) array: the
// stage-3 access pattern (S = 8.4 MB plane stride at 1024^3 float64).
#include <cstdio>
#include <cuda_runtime.h>

template <int VPT>
__global__ void tile_rw(char* buf, long long S, int R, int W, int tiles_x) {
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int lanes = W / 16, rpp = blockDim.x / lanes;
  const int lane = threadIdx.x % lanes, r0 = threadIdx.x / lanes;
  char* base = buf + (long long)ty * R * S + (long long)tx * W + lane * 16;
  int4 v[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) v[i] = *reinterpret_cast<int4*>(base + (long long)(r0 + i * rpp) * S);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < VPT; ++i) { v[i].x += 1; *reinterpret_cast<int4*>(base + (long long)(r0 + i * rpp) * S) = v[i]; }
}

int main() {
  const long long S = 8404992, ROWS = 1024;  // 1024^3 float64 spectral plane stride
  const long long total = S * ROWS;
  char* buf;
  if (cudaMalloc(&buf, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  struct Cfg { int W, R, threads; };
  // VPT fixed at 16: rows per CTA R = threads*16*16/W
  Cfg cfgs[] = {{32, 0, 64}, {32, 0, 256}, {64, 0, 256}, {64, 0, 128}, {64, 0, 512}, {128, 0, 512},
                {128, 0, 256}, {256, 0, 512}, {256, 0, 256}, {512, 0, 512}, {1024, 0, 512}};
  printf("setup: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  for (auto c : cfgs) {
    c.R = c.threads * 16 / c.W * 16;
    const int tiles_x = (int)(S / c.W), tiles_y = (int)(ROWS / c.R);
    const long long blocks = (long long)tiles_x * tiles_y;
    for (int it = 0; it < 2; ++it) tile_rw<16><<<blocks, c.threads>>>(buf, S, c.R, c.W, tiles_x);
    cudaEventRecord(a);
    tile_rw<16><<<blocks, c.threads>>>(buf, S, c.R, c.W, tiles_x);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("W=%5d rows/CTA=%5d threads=%4d : %7.1f GB/s  (%s)\n", c.W, c.R, c.threads, 2.0 * total / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
