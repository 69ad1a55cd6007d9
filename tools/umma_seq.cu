// tcgen05.mma kind::i8 probe (M=128, K=32): cycles per "chunk" of an arbitrary MMA sequence, to
// isolate what limits the Ozaki GEMM's per-chunk sequence (B operand address changes, N mix,
// accumulator overlap, A reuse).  Each sequence entry: A slot (4 KB blocks), B row offset (16-byte
// rows of the stacked B), TMEM column, N.  Operands cycle through 4 stage buffers (no loads).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_seq tools/umma_seq.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <string>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(t),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

constexpr int STAGE = 7 * 4096 + 512 * 32;   // 7 A slices + 512 stacked B rows
constexpr int NST = 4;
struct Op { int a, brow, d, n; };
__constant__ Op c_ops[64];

constexpr int SCR = 44 * 1024;   // scratch region written by the concurrent bulk-copy warp
__constant__ int c_flags;
__constant__ int c_setoff;   // flag 64: chunk c accumulates at D + (c & 1) * c_setoff   // 1: commit per chunk, 2: fence::after_thread_sync per chunk, 4: rotate D by 64 cols per chunk (sets of 7)
__global__ void k(int nops, int chunks, int lboB_rows, long long* out, const uint8_t* gsrc, int copy_mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar, cbar, ebar[4];
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < NST * STAGE; i += blockDim.x) sm[i] = (uint8_t)(i * 37 + 11);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&cbar)));
    stop = 0;
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&ebar[i])));
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tb;
  const uint32_t ID0 = (2u << 4) | (1u << 7) | (1u << 10) | (8u << 24);
  const uint32_t lboA = 2048, sboA = 128, lboB = lboB_rows * 16, sboB = 128;
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
      const uint32_t st = su(sm + (c % NST) * STAGE);
      const int fl = c_flags;
      if (fl & 2) asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t dset = (fl & 4) ? (uint32_t)((c % 7) * 64) : (fl & 64) ? (uint32_t)((c & 1) * c_setoff) : 0u;
      for (int i = 0; i < nops; ++i) {
        const Op o = c_ops[i];
        mma(tmem + o.d + dset, desc(st + o.a * 4096, lboA, sboA), desc(st + 28672 + o.brow * 16, lboB, sboB),
            ID0 | ((uint32_t)(o.n >> 3) << 17), 1);
      }
      const int every = (fl & 8) ? 2 : (fl & 16) ? 4 : (fl & 32) ? 8 : 1;
      if ((fl & 1) && (c % every) == every - 1)
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(su(&ebar[c % 4])));
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(su(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(su(&bar)));
    if (threadIdx.x == 0) {
      out[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (threadIdx.x == 32 && copy_mode) {
    // concurrent bulk copies global (L2-resident) -> shared scratch, as fast as they complete
    long long bytes = 0, c0 = clock64();
    uint32_t ph = 0;
    uint8_t* dst = sm + NST * STAGE;
    int it = 0;
    while (!stop) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(&cbar)), "r"(SCR) : "memory");
      for (int j = 0; j < 4; ++j)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         su(dst + j * (SCR / 4))), "l"(gsrc + ((size_t)(it * 4 + j) % 64) * (SCR / 4)), "r"(SCR / 4), "r"(su(&cbar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(su(&cbar)), "r"(ph) : "memory");
      ph ^= 1;
      bytes += SCR;
      ++it;
    }
    out[148 + blockIdx.x] = bytes * 1000 / (clock64() - c0);   // milli-bytes per clock
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

static long long* g_d;
static bool g_first = true;
static uint8_t* g_src;
static int g_copy = 0;
static void run(const char* name, const std::vector<Op>& ops, int lbo_rows = 512, int ctas = 148) {
  cudaMemcpyToSymbol(c_ops, ops.data(), sizeof(Op) * ops.size());
  const int chunks = 256;
  k<<<ctas, 128, NST * STAGE + SCR>>>((int)ops.size(), 8, lbo_rows, g_d, g_src, g_copy);
  k<<<ctas, 128, NST * STAGE + SCR>>>((int)ops.size(), chunks, lbo_rows, g_d, g_src, g_copy);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, g_d, sizeof(long long) * 296, cudaMemcpyDeviceToHost);
  double cb = 0;
  for (int i = 0; i < ctas; ++i) cb += h[148 + i] / 1000.0 / ctas;
  double mx = 0;
  for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
  long long ncols = 0;
  for (auto& o : ops) ncols += o.n;
  printf("%s {\"name\": \"%s\", \"mmas\": %zu, \"sum_n\": %lld, \"clk_per_chunk\": %.1f, \"clk_per_n\": %.3f, \"copy\": %d, \"copy_B_per_clk\": %.1f, \"err\": \"%s\"}",
         g_first ? "" : ",\n", name, ops.size(), ncols, mx / chunks, mx / chunks / ncols, g_copy, g_copy ? cb : 0.0, cudaGetErrorString(e));
  g_first = false;
  fflush(stdout);
}

// the kernel's per-chunk sequence for width W: A slice p against stacked B rows [0, N_p), N_p =
// pad16((8-p) W), split into near-equal parts of <= 256
static std::vector<Op> sparse_seq(int W, int p0) {   // the kernel's REV order, slices p0+1..7 only
  std::vector<Op> v;
  for (int p = 7; p > p0; --p) {
    const int N = ((8 - p) * W + 15) / 16 * 16;
    const int parts = (N + 255) / 256, step = ((N + parts - 1) / parts + 15) / 16 * 16;
    for (int r0 = 0; r0 < N; r0 += step) {
      const int nn = N - r0 < step ? N - r0 : step;
      v.push_back(Op{p - 1, r0, (p - 1) * W + r0, nn});
    }
  }
  return v;
}
static std::vector<Op> real_seq(int W, bool fixed_b, bool alt_d, bool same_a) {
  std::vector<Op> v;
  int flip = 0;
  for (int p = 1; p <= 7; ++p) {
    const int N = ((8 - p) * W + 15) / 16 * 16;
    const int parts = (N + 255) / 256, step = ((N + parts - 1) / parts + 15) / 16 * 16;
    for (int r0 = 0; r0 < N; r0 += step) {
      const int nn = N - r0 < step ? N - r0 : step;
      v.push_back(Op{same_a ? 0 : p - 1, fixed_b ? 0 : r0, alt_d ? (flip ^= 1) * 256 : (p - 1) * W + r0, nn});
    }
  }
  return v;
}

int main() {
  cudaMalloc(&g_d, 296 * sizeof(long long));
  cudaMemset(g_d, 0, 296 * sizeof(long long));
  cudaMalloc(&g_src, 64 * (SCR / 4));
  cudaMemset(g_src, 1, 64 * (SCR / 4));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE + SCR);
  for (g_copy = 1; g_copy >= 0; --g_copy) {
    std::vector<Op> v8;
    for (int i = 0; i < 8; ++i) v8.push_back(Op{i % 7, 0, (i & 1) * 256, 256});
    run(g_copy ? "n256_fixB_copy" : "n256_fixB", v8);
    run(g_copy ? "real_w72_copy" : "real_w72", real_seq(72, false, false, false));
    run(g_copy ? "real_w64_copy" : "real_w64", real_seq(64, false, false, false));
    run(g_copy ? "real_w8_copy" : "real_w8", real_seq(8, false, false, false));
  }
  g_copy = 0;
  for (int f : {1, 3}) {
    cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
    char nm[64];
    snprintf(nm, 64, "real_w72_flags%d", f); run(nm, real_seq(72, false, false, false));
    snprintf(nm, 64, "real_w8_flags%d", f); run(nm, real_seq(8, false, false, false));
  }
  for (int f : {9, 17, 33}) {
    cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
    char nm[64];
    snprintf(nm, 64, "real_w72_commit_every%d", (f & 8) ? 2 : (f & 16) ? 4 : 8); run(nm, real_seq(72, false, false, false));
    snprintf(nm, 64, "real_w64_commit_every%d", (f & 8) ? 2 : (f & 16) ? 4 : 8); run(nm, real_seq(64, false, false, false));
  }
  {
    int f = 4;
    cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
    run("real_w8_rot7sets", real_seq(8, false, false, false));
    f = 5;
    cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
    run("real_w8_rot7sets_commit", real_seq(8, false, false, false));
    f = 0;
    cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
  }
  for (int p0 : {0, 2, 3, 4, 5}) {
    for (int f : {0, 1}) {
      cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
      char nm[64];
      snprintf(nm, 64, "sparse_w72_p0_%d_commit%d", p0, f);
      run(nm, sparse_seq(72, p0));
    }
  }
  {
    int f = 0;
    cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
    for (int n : {32, 64}) {   // 8 distinct D ranges of 64 columns fit the 512 allocated
      std::vector<Op> v;
      char nm[64];
      v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, 0, 0, n}); snprintf(nm, 64, "n%d_x8_sameD", n); run(nm, v);
      v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, 0, i * 64, n}); snprintf(nm, 64, "n%d_x8_distinctD", n); run(nm, v);
      v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, i * 32, i * 64, n}); snprintf(nm, 64, "n%d_x8_distinctD_distinctB", n); run(nm, v);
    }
  }
  for (int W : {32, 24}) {
    int off = 7 * W + 16;
    cudaMemcpyToSymbol(c_setoff, &off, sizeof(int));
    for (int p0 : {0, 2, 3, 4, 5}) {
      for (int f : {1, 65}) {
        cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
        char nm[64];
        snprintf(nm, 64, "sparse_w%d_p0_%d_%s", W, p0, f & 64 ? "altsets" : "oneset");
        run(nm, sparse_seq(W, p0));
      }
    }
  }
  {
    int f = 0;
    cudaMemcpyToSymbol(c_flags, &f, sizeof(int));
  }
  printf("{\"probe\": \"umma_seq\", \"results\": [\n");
  std::vector<Op> v;
  // N = 256 x 8 variations
  v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, 0, (i & 1) * 256, 256}); run("n256_fixB_distA_altD", v);
  v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, (i & 1) * 256, (i & 1) * 256, 256}); run("n256_altB_distA_altD", v);
  v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{0, (i & 1) * 256, (i & 1) * 256, 256}); run("n256_altB_sameA_altD", v);
  v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, 0, 0, 256}); run("n256_fixB_distA_sameD", v);
  v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, (i & 1) * 256, 0, 256}); run("n256_altB_distA_sameD", v);
  v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, (i & 1) * 16, (i & 1) * 256, 256}); run("n256_B+16rows_distA_altD", v);
  // N = 128 x 16
  v.clear(); for (int i = 0; i < 16; ++i) v.push_back(Op{i % 7, 0, (i & 3) * 128, 128}); run("n128_fixB_distA", v);
  v.clear(); for (int i = 0; i < 16; ++i) v.push_back(Op{i % 7, (i & 3) * 128, (i & 3) * 128, 128}); run("n128_4B_distA", v);
  v.clear(); for (int i = 0; i < 16; ++i) v.push_back(Op{i % 7, (i & 3) * 128, 0, 128}); run("n128_4B_distA_sameD", v);
  // B-operand row stride (LBO) effect, fixed B
  v.clear(); for (int i = 0; i < 8; ++i) v.push_back(Op{i % 7, 0, (i & 1) * 256, 256}); run("n256_fixB_lbo256", v, 256);
  // the kernel's sequences
  for (int W : {72, 64, 48, 32}) {
    char nm[64];
    snprintf(nm, 64, "real_w%d", W); run(nm, real_seq(W, false, false, false));
    snprintf(nm, 64, "real_w%d_fixB", W); run(nm, real_seq(W, true, false, false));
    snprintf(nm, 64, "real_w%d_altD", W); run(nm, real_seq(W, false, true, false));
    snprintf(nm, 64, "real_w%d_fixB_altD", W); run(nm, real_seq(W, true, true, false));
    snprintf(nm, 64, "real_w%d_sameA", W); run(nm, real_seq(W, false, false, true));
  }
  // per-level pairs with N = 2W stacked (two levels per MMA?) and uniform 8 MMAs of the same total N
  printf("\n]}\n");
  return 0;
}
