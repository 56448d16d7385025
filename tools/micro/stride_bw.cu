// Microbenchmark: in-place read+write of column tiles (W bytes wide, R rows at
// stride S bytes), the access pattern of the strided column-FFT kernels.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int VPT>
__global__ void tile_rw(char* buf, long long stride, int rows, int wbytes, long long tiles_per_row_band,
                        long long ntiles) {
  // one CTA per tile; tile t covers columns [ (t % tpr) * W, +W ) of rows [(t / tpr) * rows, +rows)
  long long t = blockIdx.x;
  if (t >= ntiles) return;
  long long band = t / tiles_per_row_band, col = (t % tiles_per_row_band) * wbytes;
  const int lanes_per_row = wbytes / 16;
  const int rows_per_pass = blockDim.x / lanes_per_row;
  int4 v[VPT];
  const int lane = threadIdx.x % lanes_per_row, r0 = threadIdx.x / lanes_per_row;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    long long r = band * rows + r0 + (long long)i * rows_per_pass;
    v[i] = *reinterpret_cast<int4*>(buf + r * stride + col + lane * 16);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    long long r = band * rows + r0 + (long long)i * rows_per_pass;
    int4 x = v[i];
    x.x += 1;
    *reinterpret_cast<int4*>(buf + r * stride + col + lane * 16) = x;
  }
}

int main(int argc, char** argv) {
  const long long total = 8LL << 30;  // 8 GiB
  char* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int threads = 256;
  // tile of 64 KB per CTA (16 int4 per thread): rows = 64KB / W
  long long strides[] = {8208, 8208LL * 1024};
  for (long long S : strides) {
    for (int W : {32, 64, 128, 256, 512, 1024}) {
      const int VPT = 16;
      int rows = threads * VPT * 16 / W;
      long long nrow_total = total / S;
      long long bands = nrow_total / rows;
      long long tpr = S / W;  // tiles per row band (S multiple of 16)
      long long ntiles = bands * tpr;
      if (ntiles > 2000000000LL) ntiles = 2000000000LL;
      for (int it = 0; it < 2; ++it) tile_rw<16><<<ntiles, threads>>>(buf, S, rows, W, tpr, ntiles);
      cudaEventRecord(a);
      tile_rw<16><<<ntiles, threads>>>(buf, S, rows, W, tpr, ntiles);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double bytes = 2.0 * ntiles * threads * VPT * 16;
      printf("S=%10lld W=%5d rows/tile=%5d : %8.1f GB/s (%.3f ms) %s\n", S, W, rows, bytes / ms / 1e6, ms,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
