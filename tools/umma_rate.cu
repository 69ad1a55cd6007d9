// tcgen05.mma kind::i8 issue-rate probe: cycles per MMA (M=128, K=32) for several N and smem
// layouts (SWIZZLE_NONE vs SWIZZLE_32B/64B/128B), operands resident in smem, one CTA per SM.
// Prints MAC/clk/SM so the Ozaki GEMM can be held against the real per-SM int8 tensor rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

__global__ void k(int n, int layout, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* A = sm;              // 128 x 128 B
  uint8_t* B = sm + 16384;      // 256 x 128 B
  for (int i = threadIdx.x; i < 16384 + 32768; i += blockDim.x) sm[i] = (uint8_t)(i * 37 + 11);
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
  // layout 0: no swizzle (LBO = K-half stride, SBO = 128);  swizzled: SBO = 8 rows x atom bytes
  uint32_t lboA = 128 * 16, sboA = 128, lboB = 256 * 16, sboB = 128;
  if (layout == 6) { lboA = lboB = 16; sboA = sboB = 256; }    // 32B swizzle: 8 rows x 32 B
  if (layout == 4) { lboA = lboB = 16; sboA = sboB = 512; }    // 64B
  if (layout == 2) { lboA = lboB = 16; sboA = sboB = 1024; }   // 128B
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t da = desc(su(A), lboA, sboA, layout), db = desc(su(B), lboB, sboB, layout);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (uint32_t)((i & 1) * 256)),
          "l"(da), "l"(db), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(su(&bar)));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024);
  const int iters = 4096;
  printf("{\"probe\": \"umma_i8_rate\", \"results\": [\n");
  int layouts[4] = {0, 6, 4, 2};
  int ns[6] = {16, 32, 64, 128, 192, 256};
  bool first = true;
  for (int li = 0; li < 4; ++li)
    for (int ni = 0; ni < 6; ++ni) {
      k<<<148, 128, 49152>>>(ns[ni], layouts[li], 64, d);   // warm-up
      k<<<148, 128, 49152>>>(ns[ni], layouts[li], iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double cyc = mx / iters;
      printf("%s {\"layout\": %d, \"n\": %d, \"clk_per_mma\": %.2f, \"mac_per_clk\": %.0f, \"err\": \"%s\"}",
             first ? "" : ",\n", layouts[li], ns[ni], cyc, 128.0 * ns[ni] * 32 / cyc, cudaGetErrorString(e));
      first = false;
    }
  printf("\n]}\n");
  return 0;
}
