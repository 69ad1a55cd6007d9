// Woodbury GEMM Z = C^-1 Y in FP64 accuracy on the INT8 tensor cores (tcgen05.mma kind::i8),
// by the Ozaki splitting scheme.
//
// FP64 has no tcgen05 kind; DMMA (mma.sync f64) and DFMA share one FP64 datapath (~37 TF/s,
// tools/fp64_mix.cu), which the transform kernels already saturate.  The GEMM -- 2 m^2 n_s
// flops per shape, the largest single block of the preconditioner -- is instead moved to the
// INT8 tensor pipe:
//   rows of A = C^-1 and of B = Y^T are scaled by powers of two (exponents eA_i, eB_n) into
//   (-1, 1) and cut into S base-128 digits ("slices") a_p, b_q in [-127, 127];
//   A B^T = 2^(eA_i + eB_n) * sum_L 2^(-7L) D_L,   D_L = sum_{p+q=L} a_p b_q^T   (L = 2 .. S+1),
// each D_L an exact int32 sum (|a b| <= 127^2, K <= 2^15).  Truncating at L <= S+1 bounds the
// error by ~2^(-7S) of the row/column scales (S = 6: 2^-42; tests/test_ozaki_gpu.py).
//
// Layout: slices are stored pre-tiled in the UMMA canonical K-major SWIZZLE_NONE layout --
// for each (128-row tile, 32-byte K chunk) the S slices are one contiguous block of
// S x [2 K-halves][16 row groups][8 rows][16 B] -- so a pipeline stage is two bulk copies
// (cp.async.bulk, mbarrier complete_tx), no tensor maps.  One CTA per SM, persistent over
// (shape, row tile, column tile); warp 4 streams operands, warp 5 issues the S(S+1)/2 MMAs
// per K chunk into S TMEM accumulators (one per level), warps 0-3 drain TMEM, combine the
// levels in FP64 and store Z.
#include <cstdint>
#include "common.cuh"

namespace fmp {

constexpr int OZ_S = 6;                 // slices per operand
constexpr int OZ_M = 128;               // rows per tile (TMEM lanes)
constexpr int OZ_N = 80;                // columns per tile: OZ_S * OZ_N <= 512 TMEM columns
constexpr int OZ_KC = 32;               // K bytes per MMA / stage
constexpr int OZ_ABLK = OZ_M * OZ_KC;   // bytes of one A slice block
constexpr int OZ_BBLK = OZ_N * OZ_KC;   // bytes of one B slice block
constexpr int OZ_STAGE = OZ_S * (OZ_ABLK + OZ_BBLK);
constexpr int OZ_STAGES = 4;
constexpr int OZ_THREADS = 192;         // warps 0-3 epilogue, 4 producer, 5 MMA
constexpr int OZ_TMEM_COLS = 512;

struct OzShape {
  const int8_t* A;      // tiled slices of C^-1: [mtile][kchunk][S][OZ_ABLK]
  const int* eA;        // [m] row exponents
  const int8_t* B;      // tiled slices of Y: [ntile][kchunk][S][OZ_BBLK]
  const int* eB;        // [n] column exponents
  double* Z;            // [n][ld]
  int m, n, ld, kchunks;
};
struct OzTile {
  int shape, mt, nt, pad;
};

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);   // version 1, SWIZZLE_NONE
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(s_u32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   s_u32(dst)),
               "l"(src), "r"(bytes), "r"(s_u32(bar))
               : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(s_u32(b))
               : "memory");
}
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_ozaki(const OzShape* __restrict__ shapes, const OzTile* __restrict__ tiles, int n_tiles) {
  extern __shared__ __align__(1024) uint8_t osm[];
  __shared__ __align__(8) uint64_t full_bar[OZ_STAGES], empty_bar[OZ_STAGES], tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(s_u32(&tmem_base)),
                 "r"(OZ_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;

  if (warp == 4) {
    // ---------------- producer: two bulk copies per stage
    if (lane == 0) {
      int it = 0;
      for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
        const OzTile tl = tiles[ti];
        const OzShape sh = shapes[tl.shape];
        const int8_t* a = sh.A + (size_t)tl.mt * sh.kchunks * OZ_S * OZ_ABLK;
        const int8_t* b = sh.B + (size_t)tl.nt * sh.kchunks * OZ_S * OZ_BBLK;
        for (int kc = 0; kc < sh.kchunks; ++kc, ++it) {
          const int s = it % OZ_STAGES;
          const uint32_t ph = (it / OZ_STAGES) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = osm + s * OZ_STAGE;
          mbar_expect_tx(&full_bar[s], OZ_STAGE);
          bulk_g2s(st, a + (size_t)kc * OZ_S * OZ_ABLK, OZ_S * OZ_ABLK, &full_bar[s]);
          bulk_g2s(st + OZ_S * OZ_ABLK, b + (size_t)kc * OZ_S * OZ_BBLK, OZ_S * OZ_BBLK, &full_bar[s]);
        }
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer: S(S+1)/2 MMAs per K chunk, level L -> TMEM columns [(L-2)*N, ...)
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_N >> 3) << 17) |
                           ((uint32_t)(OZ_M >> 4) << 24);
    int it = 0, tcount = 0;
    for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x, ++tcount) {
      const OzShape sh = shapes[tiles[ti].shape];
      if (tcount > 0) {   // the epilogue must have drained the accumulators of the previous tile
        mbar_wait(&tempty_bar, (tcount - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
      }
      for (int kc = 0; kc < sh.kchunks; ++kc, ++it) {
        const int s = it % OZ_STAGES;
        const uint32_t ph = (it / OZ_STAGES) & 1;
        mbar_wait(&full_bar[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (lane == 0) {
          const uint32_t sa = s_u32(osm + s * OZ_STAGE);
          const uint32_t sb = sa + OZ_S * OZ_ABLK;
#pragma unroll
          for (int L = 2; L <= OZ_S + 1; ++L) {
            const uint32_t dt = tmem + (uint32_t)((L - 2) * OZ_N);
#pragma unroll
            for (int p = 1; p < L; ++p) {
              const int q = L - p;
              if (q > OZ_S) continue;
              const uint64_t da = umma_desc(sa + (p - 1) * OZ_ABLK, OZ_M * 16, 128);
              const uint64_t db = umma_desc(sb + (q - 1) * OZ_BBLK, OZ_N * 16, 128);
              umma_i8(dt, da, db, idesc, (kc > 0 || p > 1) ? 1u : 0u);
            }
          }
          umma_commit(&empty_bar[s]);                         // stage free once these MMAs retire
          if (kc == sh.kchunks - 1) umma_commit(&tfull_bar);  // accumulators complete
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue warps 0-3: lane quadrant = warp, one row per thread
    int tcount = 0;
    for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x, ++tcount) {
      const OzTile tl = tiles[ti];
      const OzShape sh = shapes[tl.shape];
      mbar_wait(&tfull_bar, tcount & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int row = tl.mt * OZ_M + warp * 32 + lane;
      const int ea = row < sh.m ? sh.eA[row] : 0;
      for (int c0 = 0; c0 < OZ_N; c0 += 16) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
        for (int L = OZ_S + 1; L >= 2; --L) {   // smallest terms first
          uint32_t v[16];
          const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((L - 2) * OZ_N + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
              "[%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15])
              : "r"(addr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double w = ldexp(1.0, -7 * L);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = fma((double)(int)v[j], w, acc[j]);
        }
        if (row < sh.m) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = tl.nt * OZ_N + c0 + j;
            if (n < sh.n) sh.Z[(size_t)n * sh.ld + row] = ldexp(acc[j], ea + sh.eB[n]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      mbar_arrive(&tempty_bar);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(OZ_TMEM_COLS));
}

// ---------------------------------------------------------------- slicing
// One warp per row r of src [rows][ld] (K = kvalid entries): exponent e = max |x| exponent,
// digits of x * 2^-e in base 128, written into the tiled UMMA layout with tile height T.
template <int T>
__global__ void k_ozaki_slice(const double* __restrict__ src, int rows, int ld, int kvalid, int kchunks,
                              int8_t* __restrict__ dst, int* __restrict__ exps) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int tiles_rows = (rows + T - 1) / T * T;
  if (warp >= tiles_rows) return;
  const int r = warp;
  const bool valid = r < rows;
  double mx = 0.0;
  if (valid)
    for (int k = lane; k < kvalid; k += 32) mx = fmax(mx, fabs(src[(size_t)r * ld + k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);   // mx = f 2^e, f in [0.5, 1): |x| 2^-e < 1
  if (lane == 0 && valid) exps[r] = e;
  const int rt = r / T, rr = r % T;
  const size_t blk = (size_t)T * OZ_KC;
  for (int k = lane; k < kchunks * OZ_KC; k += 32) {
    double x = (valid && k < kvalid) ? ldexp(src[(size_t)r * ld + k], -e) : 0.0;
    const int kc = k / OZ_KC, kb = k % OZ_KC, kh = kb / 16, kk = kb % 16;
    int8_t* base = dst + ((size_t)rt * kchunks + kc) * OZ_S * blk + kh * (T * 16) + (rr / 8) * 128 + (rr % 8) * 16 + kk;
#pragma unroll
    for (int p = 0; p < OZ_S; ++p) {
      x *= 128.0;
      const double d = trunc(x);   // |d| <= 127, same sign as x; x - d exact
      x -= d;
      base[p * blk] = (int8_t)d;
    }
  }
}

int ozaki_slice_a(const double* cinv, int m, int ld, int kchunks, int8_t* dst, int* exps, cudaStream_t st) {
  const int rows = (m + OZ_M - 1) / OZ_M * OZ_M;
  k_ozaki_slice<OZ_M><<<(rows * 32 + 255) / 256, 256, 0, st>>>(cinv, m, ld, m, kchunks, dst, exps);
  FMP_CHECK_LAUNCH();
  return 0;
}

int ozaki_slice_b(const double* y, int n, int m, int ld, int kchunks, int8_t* dst, int* exps, cudaStream_t st) {
  const int rows = (n + OZ_N - 1) / OZ_N * OZ_N;
  k_ozaki_slice<OZ_N><<<(rows * 32 + 255) / 256, 256, 0, st>>>(y, n, ld, m, kchunks, dst, exps);
  FMP_CHECK_LAUNCH();
  return 0;
}

size_t ozaki_a_bytes(int m, int kchunks) { return (size_t)((m + OZ_M - 1) / OZ_M) * kchunks * OZ_S * OZ_ABLK; }
size_t ozaki_b_bytes(int n, int kchunks) { return (size_t)((n + OZ_N - 1) / OZ_N) * kchunks * OZ_S * OZ_BBLK; }
int ozaki_kchunks(int m) { return (m + OZ_KC - 1) / OZ_KC; }
int ozaki_tile_m() { return OZ_M; }
int ozaki_tile_n() { return OZ_N; }

int ozaki_setup() {
  FMP_CHECK_CUDA(cudaFuncSetAttribute(k_ozaki, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      OZ_STAGES * OZ_STAGE));
  return 0;
}

int ozaki_launch(const OzShape* shapes, const OzTile* tiles, int n_tiles, int sms, cudaStream_t st) {
  if (n_tiles <= 0) return 0;
  const int grid = n_tiles < sms ? n_tiles : sms;
  k_ozaki<<<grid, OZ_THREADS, OZ_STAGES * OZ_STAGE, st>>>(shapes, tiles, n_tiles);
  FMP_CHECK_LAUNCH();
  return 0;
}

}  // namespace fmp
