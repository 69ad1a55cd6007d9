// tcgen05.mma kind::i8 probe of the Ozaki GEMM's per-K-chunk MMA sequence (M=128, K=32):
// cycles per chunk for the real pattern (7 A slices, stacked B, N = pad16((8-p) W) split at 256)
// and variants that isolate the cost: one shared A address, SWIZZLE_32B operand layout,
// uniform N=256 MMAs.  Operands cycle through 4 stage buffers in shared memory (no loads).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_chunk tools/umma_chunk.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ bool g_elect;   // set per launch: issue from the whole warp with elect.sync inside the asm
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(t),
      "l"(a), "l"(b), "r"(idesc), "r"(1));
}

constexpr int STAGE = 7 * 4096 + 512 * 32;   // 45056
constexpr int NST = 4;

// variant: 0 real (NONE layout), 1 same A, 2 real SW32, 3 N=256 x 8 distinct A, 4 real with only
// p<=4 (N>=256 part), 5 each p as separate N<=W MMAs (one per level: 28 MMAs of N=W)
__global__ void k(int W, int variant, int chunks, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < NST * STAGE; i += blockDim.x) sm[i] = (uint8_t)(i * 37 + 11);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tb;
  const uint32_t ID0 = (2u << 4) | (1u << 7) | (1u << 10) | (8u << 24);
  const bool sw = variant == 2;
  const uint32_t lay = sw ? 6u : 0u;
  const int R = (7 * W + 15) / 16 * 16;
  // NONE: A lbo = 128*16 (K halves), sbo = 128 (8-row core matrices); B lbo = R*16
  // SW32: rows of 32 B contiguous, sbo = 256 (8 rows), lbo unused (16)
  const uint32_t lboA = sw ? 16 : 2048, sboA = sw ? 256 : 128, lboB = sw ? 16 : R * 16, sboB = sw ? 256 : 128;
  long long t0 = 0;
  int flip = 0;
  if (threadIdx.x < 32) {
    t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
      const uint32_t st = su(sm + (c % NST) * STAGE);
      if (variant == 3) {
        for (int p = 0; p < 8; ++p)
          mma(tmem + (p & 1) * 256, desc(st + (p % 7) * 4096, lboA, sboA, lay), desc(st + 28672, lboB, sboB, lay),
              ID0 | (32u << 17));
      } else if (variant >= 10) {   // isolated N = variant: 8 MMAs alternating TMEM halves
        for (int p = 0; p < 8; ++p)
          mma(tmem + (p & 1) * 256, desc(st + (p % 7) * 4096, lboA, sboA, lay), desc(st + 28672, lboB, sboB, lay),
              ID0 | ((uint32_t)(variant >> 3) << 17));
      } else if (variant == 5) {
        for (int p = 1; p <= 7; ++p)
          for (int q = 1; q <= 8 - p; ++q)
            mma(tmem + (p + q - 2) * W, desc(st + (p - 1) * 4096, lboA, sboA, lay),
                desc(st + 28672 + (q - 1) * W * (sw ? 32 : 16), lboB, sboB, lay), ID0 | ((uint32_t)(W >> 3) << 17));
      } else {
        for (int p = 1; p <= 7; ++p) {
          if (variant == 4 && p > 4) break;
          const uint32_t a = st + (variant == 1 ? 0 : (p - 1) * 4096);
          const int N = ((8 - p) * W + 15) / 16 * 16;
          for (int r0 = 0; r0 < N; r0 += 256) {
            const int nn = N - r0 < 256 ? N - r0 : 256;
            flip ^= 1;
            mma(variant == 6 ? tmem + flip * 256 : tmem + (p - 1) * W + r0, desc(a, lboA, sboA, lay), desc(st + 28672 + r0 * (sw ? 32 : 16), lboB, sboB, lay),
                ID0 | ((uint32_t)(nn >> 3) << 17));
          }
        }
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(su(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(su(&bar)));
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE);
  const int chunks = 512;
  const char* names[7] = {"real_none", "same_a", "real_sw32", "n256x8", "p1to4", "per_level", "real_alt_dst"};
  printf("{\"probe\": \"umma_chunk\", \"results\": [\n");
  bool first = true;
  for (int n = 16; n <= 256; n += 16) {
    k<<<148, 128, NST * STAGE>>>(72, n, 16, d);
    k<<<148, 128, NST * STAGE>>>(72, n, chunks, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%s {\"N\": %d, \"clk_per_mma\": %.1f, \"err\": \"%s\"}", first ? "" : ",\n", n, mx / chunks / 8,
           cudaGetErrorString(e));
    first = false;
  }
  int ws[3] = {72, 64, 48};
  for (int wi = 0; wi < 3; ++wi)
    for (int v = 0; v < 7; ++v) {
      if (v == 5 && ws[wi] % 16) continue;
      k<<<148, 128, NST * STAGE>>>(ws[wi], v, 16, d);
      k<<<148, 128, NST * STAGE>>>(ws[wi], v, chunks, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%s {\"W\": %d, \"variant\": \"%s\", \"clk_per_chunk\": %.1f, \"err\": \"%s\"}", first ? "" : ",\n", ws[wi],
             names[v], mx / chunks, cudaGetErrorString(e));
      first = false;
    }
  printf("\n]}\n");
  return 0;
}
