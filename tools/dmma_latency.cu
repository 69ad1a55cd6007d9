// DMMA m8n8k4 latency / throughput probe: cycles per DMMA vs (warps per SM, chains per warp).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double d[CH][2];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-9 + c;
  double a = 1e-3 * (threadIdx.x & 31), b = 2e-3 * (threadIdx.x & 7);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH> void run(int warps) {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 148 * 8);
  int iters = 2000;
  k<CH><<<148, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  k<CH><<<148, warps * 32>>>(out, cyc, iters);
  long long h[148]; cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
  double c = (double)h[0] / (iters * CH);   // cycles per DMMA per warp
  printf("warps/SM %2d chains %2d : %6.2f cyc per DMMA per warp -> SM rate %.3f DMMA/cyc (peak 0.25)\n", warps, CH, c, warps / c);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {1, 2, 4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
  return 0;
}
