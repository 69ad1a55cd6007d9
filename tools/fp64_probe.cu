// FP64 throughput / fragment-layout probe for B200 (sm_100a).
// Measures DFMA and DMMA (mma.sync f64 shapes) issue throughput and checks the
// fragment layouts assumed by the transform kernels. Prints one JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double b, double c) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double (&d)[4], const double (&a)[2], double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE>
__global__ void dmma_kernel(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  double acc[4][4];
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) acc[t][q] = 0.0;
  double a[8], b[4];
  for (int q = 0; q < 8; ++q) a[q] = 1e-3 * (lane + q);
  for (int q = 0; q < 4; ++q) b[q] = 1e-3 * (lane - q);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (SHAPE == 0) { double d2[2] = {acc[t][0], acc[t][1]}; mma884(d2, a[t], b[t]); acc[t][0] = d2[0]; acc[t][1] = d2[1]; }
      if (SHAPE == 1) { double d4[4] = {acc[t][0], acc[t][1], acc[t][2], acc[t][3]}; double aa[2] = {a[0], a[1]};
                        mma1684(d4, aa, b[t]); for (int q = 0; q < 4; ++q) acc[t][q] = d4[q]; }
      if (SHAPE == 2) { double d4[4] = {acc[t][0], acc[t][1], acc[t][2], acc[t][3]}; double aa[4] = {a[0], a[1], a[2], a[3]};
                        double bb[2] = {b[0], b[1]}; mma1688(d4, aa, bb); for (int q = 0; q < 4; ++q) acc[t][q] = d4[q]; }
      if (SHAPE == 3) { double d4[4] = {acc[t][0], acc[t][1], acc[t][2], acc[t][3]}; double aa[8];
                        for (int q = 0; q < 8; ++q) aa[q] = a[q]; double bb[4] = {b[0], b[1], b[2], b[3]};
                        mma16816(d4, aa, bb); for (int q = 0; q < 4; ++q) acc[t][q] = d4[q]; }
    }
  }
  double s = 0; for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) s += acc[t][q];
  if (s == 12345.678) out[0] = s;
}

// Layout check: one warp computes D = A(MxK) * B(KxN) with the assumed fragment maps.
template <int SHAPE>
__global__ void layout_kernel(const double* A, const double* B, double* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  if (SHAPE == 0) {  // m8n8k4
    double d[2] = {0, 0};
    mma884(d, A[g * 4 + t], B[t * 8 + g]);
    D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1];
  } else if (SHAPE == 1) {  // m16n8k4
    double d[4] = {0, 0, 0, 0}; double a[2] = {A[g * 4 + t], A[(g + 8) * 4 + t]};
    mma1684(d, a, B[t * 8 + g]);
    D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1]; D[(g + 8) * 8 + 2 * t] = d[2]; D[(g + 8) * 8 + 2 * t + 1] = d[3];
  } else if (SHAPE == 2) {  // m16n8k8
    double d[4] = {0, 0, 0, 0};
    double a[4] = {A[g * 8 + t], A[(g + 8) * 8 + t], A[g * 8 + t + 4], A[(g + 8) * 8 + t + 4]};
    double b[2] = {B[t * 8 + g], B[(t + 4) * 8 + g]};
    mma1688(d, a, b);
    D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1]; D[(g + 8) * 8 + 2 * t] = d[2]; D[(g + 8) * 8 + 2 * t + 1] = d[3];
  } else {  // m16n8k16
    double d[4] = {0, 0, 0, 0}; double a[8]; double b[4];
    for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i % 2)) * 16 + t + 4 * (i / 2)];
    for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
    mma16816(d, a, b);
    D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1]; D[(g + 8) * 8 + 2 * t] = d[2]; D[(g + 8) * 8 + 2 * t + 1] = d[3];
  }
}

template <int SHAPE>
double check_layout() {
  const int M = SHAPE == 0 ? 8 : 16, N = 8, K = SHAPE == 0 ? 4 : SHAPE == 1 ? 4 : SHAPE == 2 ? 8 : 16;
  std::vector<double> A(M * K), B(K * N), D(M * N), R(M * N, 0.0);
  for (int i = 0; i < M * K; ++i) A[i] = std::sin(1.0 + i);
  for (int i = 0; i < K * N; ++i) B[i] = std::cos(2.0 + 3 * i);
  for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) for (int k = 0; k < K; ++k) R[i * N + j] += A[i * K + k] * B[k * N + j];
  double *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  layout_kernel<SHAPE><<<1, 32>>>(dA, dB, dD);
  CK(cudaGetLastError());
  CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
  double err = 0; for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(D[i] - R[i]));
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return err;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  const int iters = 4096, threads = 256, blocks = sms * 8;
  dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  double dfma_tf = 2.0 * 32.0 * iters * (double)threads * blocks / (ms * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"dfma_tflops\": %.2f", sms, dfma_tf);
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double fmas[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  for (int s = 0; s < 4; ++s) {
    auto launch = [&](int it) {
      if (s == 0) dmma_kernel<0><<<blocks, threads>>>(out, it);
      if (s == 1) dmma_kernel<1><<<blocks, threads>>>(out, it);
      if (s == 2) dmma_kernel<2><<<blocks, threads>>>(out, it);
      if (s == 3) dmma_kernel<3><<<blocks, threads>>>(out, it);
    };
    int it = 2048;
    launch(8);
    cudaEventRecord(e0); launch(it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double warps = (double)blocks * threads / 32;
    double tf = 2.0 * fmas[s] * 4 * it * warps / (ms * 1e-3) / 1e12;
    printf(", \"dmma_%s_tflops\": %.2f", names[s], tf);
  }
  printf(", \"layout_err\": [%.3g, %.3g, %.3g, %.3g]", check_layout<0>(), check_layout<1>(), check_layout<2>(), check_layout<3>());
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf(", \"clock_khz\": %d}\n", clk);
  CK(cudaGetLastError());
  return 0;
}
