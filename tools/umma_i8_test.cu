// Minimal tcgen05 INT8 GEMM check (kind::i8, cta_group::1, SWIZZLE_NONE K-major operands):
// D[128 x N] (int32, TMEM) = A[128 x K] * B[N x K]^T.  Validates the smem/instruction descriptor
// encodings and the TMEM load path used by the Ozaki Woodbury GEMM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version 1 (sm_100)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__global__ void k(const int8_t* A, const int8_t* B, int* D) {
  __shared__ __align__(1024) int8_t sA[M * K];
  __shared__ __align__(1024) int8_t sB[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  // core-matrix layout per 32-byte K chunk c: [c][kh][rowgroup][8 rows][16 B]
  for (int q = tid; q < M * K / 16; q += blockDim.x) {  // 16-byte pieces
    const int r = q / (K / 16), kb = q % (K / 16);       // row, 16-byte K block
    const int c = kb / 2, kh = kb % 2;
    int8_t* dst = sA + c * (M * 32) + kh * (M * 16) + (r / 8) * 128 + (r % 8) * 16;
    for (int e = 0; e < 16; ++e) dst[e] = A[r * K + kb * 16 + e];
  }
  for (int q = tid; q < N * K / 16; q += blockDim.x) {
    const int r = q / (K / 16), kb = q % (K / 16);
    const int c = kb / 2, kh = kb % 2;
    int8_t* dst = sB + c * (N * 32) + kh * (N * 16) + (r / 8) * 128 + (r % 8) * 16;
    for (int e = 0; e < 16; ++e) dst[e] = B[r * K + kb * 16 + e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  // instruction descriptor: S32 accum, signed A/B, K-major both, N>>3, M>>4
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    for (int c = 0; c < K / 32; ++c) {
      const uint64_t da = make_desc(smem_u32(sA + c * M * 32), M * 16, 128);
      const uint64_t db = make_desc(smem_u32(sB + c * N * 32), N * 16, 128);
      const uint32_t acc = c > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // TMEM -> registers: warp w owns lanes 32w..32w+31 (rows), 16 columns per load
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    const int row = warp * 32 + (tid & 31);
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(64));
}

int main() {
  std::vector<int8_t> A(M * K), B(N * K);
  srand(1);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  k<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int ref = 0;
      for (int q = 0; q < K; ++q) ref += (int)A[i * K + q] * (int)B[j * K + q];
      if (ref != D[i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): got %d want %d\n", i, j, D[i * N + j], ref);
        ++bad;
      }
    }
  printf("cuda: %s, mismatches: %ld of %d\n", cudaGetErrorString(e), bad, M * N);
  return 0;
}
