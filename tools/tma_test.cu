// Standalone TMA f64 box-load probe: variant chosen by argv[1] (each run is its own context).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2508_07193_b200/csrc/tma.cuh"
using namespace fmp;

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          s_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(s_u32(bar))
      : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int rank, int bytes, int cx, int c0, int n) {
  extern __shared__ __align__(1024) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 8192);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, bytes);
    if (rank % 100 == 44) tma_load_4d(sm, &tm, cx, c0, (rank / 100) % 10, rank / 1000, bar);
    else if (rank == 4) tma_load_4d(sm, &tm, cx, c0, 0, 0, bar);
    else tma2d(sm, &tm, cx, c0, bar);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sm[i];
}

namespace fmp { void set_error(const char* fmt, ...) { printf("error: %s\n", fmt); } }

int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int bx = 16, by = 16, bz = 16;
  double *x, *out;
  cudaMalloc(&x, 3 * bx * by * bz * 8);
  cudaMalloc(&out, 65536);
  double* h = new double[3 * bx * by * bz];
  for (int i = 0; i < 3 * bx * by * bz; ++i) h[i] = i + 1;
  cudaMemcpy(x, h, 3 * bx * by * bz * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  int rank = 4, bxw = 66, c0 = -1;
  if (variant == 1) c0 = 0;               // non-negative start
  if (variant == 2) { bxw = 64; c0 = 0; } // box 64 wide
  if (variant == 3) rank = 2;
  if (variant == 4) { rank = 2; bxw = 16; c0 = 0; }
  const uint64_t dims[4] = {bx, by, bz, 3};
  const uint64_t strides[3] = {bx * 8, bx * by * 8, (uint64_t)bx * by * bz * 8};
  const uint32_t box[4] = {(uint32_t)bxw, 10, 1, 3};
  const uint64_t dims2[2] = {bx, (uint64_t)by * bz * 3};
  int e;
  if (variant >= 10) {   // box probes: argv = variant bw bh bc cx cy cz cc
    const int bw = atoi(argv[2]), bh = atoi(argv[3]), bc = atoi(argv[4]);
    const int cx = atoi(argv[5]), cy = atoi(argv[6]), cz = atoi(argv[7]), cc = atoi(argv[8]);
    const uint64_t d10[4] = {bx, by, bz, 3};
    const uint32_t b10[4] = {(uint32_t)bw, (uint32_t)bh, 1, (uint32_t)bc};
    e = encode_tensor_map_f64(&tm, x, 4, d10, strides, b10);
    printf("box {%d,%d,1,%d} at (%d,%d,%d,%d) encode %d\n", bw, bh, bc, cx, cy, cz, cc, e);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8 + 128);
    k<<<1, 128, 8192 * 8 + 128>>>(tm, out, 44 + 100 * cz + 1000 * cc, bw * bh * bc * 8, cx, cy, bw * bh * bc);
    cudaError_t err = cudaDeviceSynchronize();
    printf("  -> %s\n", cudaGetErrorString(err));
    return err ? 1 : 0;
  }
  if (variant >= 5) {   // same bytes as 32-bit or 64-bit integer elements
    const int dt = variant == 5 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : variant == 6 ? CU_TENSOR_MAP_DATA_TYPE_INT64
                                                                                 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
    const int f = (variant == 6) ? 1 : 2;
    const uint64_t d5[4] = {(uint64_t)bx * f, by, bz, 3};
    const uint32_t b5[4] = {(uint32_t)(66 * f), 10, 1, 3};
    e = encode_tensor_map(&tm, dt, x, 4, d5, strides, b5);
    c0 = -1;
  } else {
    e = rank == 4 ? encode_tensor_map_f64(&tm, x, 4, dims, strides, box)
                  : encode_tensor_map_f64(&tm, x, 2, dims2, strides, box);
  }
  const int n = rank == 4 ? bxw * 10 * 3 : bxw * 10;
  printf("variant %d rank %d box %d c0 %d encode %d\n", variant, rank, bxw, c0, e);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8 + 128);
  k<<<1, 128, 8192 * 8 + 128>>>(tm, out, rank, n * 8, (variant == 5 || variant == 7) ? 2 * c0 : c0, c0, n);
  cudaError_t err = cudaDeviceSynchronize();
  printf("  -> %s\n", cudaGetErrorString(err));
  if (err) return 1;
  double* ho = new double[n];
  cudaMemcpy(ho, out, n * 8, cudaMemcpyDeviceToHost);
  printf("  row0: %g %g %g  row1: %g %g\n", ho[0], ho[1], ho[2], ho[bxw], ho[bxw + 1]);
  return 0;
}
