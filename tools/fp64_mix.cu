// Do DMMA (tensor pipe) and DFMA (fp64 pipe) run concurrently on B200?  Half the warps of
// every CTA issue m8n8k4 DMMA chains, the other half DFMA chains; compare with each alone.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, int mode) {  // mode 0: dmma only, 1: dfma only, 2: mixed
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double d[4][2];
  for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-9 + c;
  double a = 1e-3 * (threadIdx.x & 31), b = 2e-3 * (threadIdx.x & 7);
  double f[8];
  for (int c = 0; c < 8; ++c) f[c] = threadIdx.x * 1e-7 + c;
  if (do_mma) {
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  } else {
    for (int i = 0; i < iters * 8; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) f[c] = fma(f[c], 1.0000001, 1e-9);
  }
  double s = 0; for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1]; for (int c = 0; c < 8; ++c) s += f[c];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000, blocks = 148 * 4, threads = 256;
  for (int mode = 0; mode < 3; ++mode) {
    k<<<blocks, threads>>>(out, 10, mode);
    cudaEventRecord(e0); k<<<blocks, threads>>>(out, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = blocks * threads / 32.0;
    double mma_w = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0), fma_w = mode == 1 ? warps : (mode == 2 ? warps / 2 : 0);
    double mma_tf = mma_w * iters * 4 * 256 * 2 / (ms * 1e-3) / 1e12;
    double fma_tf = fma_w * 32 * iters * 8 * 8 * 2 / (ms * 1e-3) / 1e12;
    printf("mode %d: %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", mode, ms, mma_tf, fma_tf, mma_tf + fma_tf);
  }
  return 0;
}
