// Grouped FP64 GEMM for the Woodbury correction (K4): Z_s = C_s^-1 Y_s for every extended
// shape s of a plan, on DMMA (mma.sync m8n8k4 f64) tensor cores.
//
// ref:subdomain.py:280 applies z = C^-1 e0[rows] one subdomain at a time (a DGEMV that
// re-reads the 293-374 MB C^-1 for every subdomain).  Batched over the n_s subdomains of a
// shape it is one m x m x n_s GEMM that streams C^-1 once per column tile: compute-bound
// for n_s >= ~24.  Operands (row-major, leading dimension ld = m rounded up to 4, zero padded):
//   A = C^-1 [m][ld],  B = Y [n_s][ld] (column j = subdomain j),  C = Z [n_s][ld].
// CTA tile MT x NT over the full K = m, K-chunks of 16 streamed by cp.async through a
// STAGES-deep ring; warps own WM x WN 8x8 DMMA tiles (WM*WN independent accumulator chains).
#include "common.cuh"

namespace fmp {

struct GemmShape {
  const double* A;
  const double* B;
  double* C;
  int m, n, ld;
};
struct GemmTile {
  int shape, i0, n0, pad;
};

constexpr int KC = 32;        // K chunk per stage
constexpr int GS = KC + 4;    // smem row stride (== 4 mod 8: conflict-free fragment loads)

template <int WM, int WN, int NWM, int NWN, int STAGES>
struct GemmCfg {
  static constexpr int MT = 8 * WM * NWM, NT = 8 * WN * NWN, WARPS = NWM * NWN;
  static constexpr int A_ST = MT * GS, B_ST = NT * GS;
  static constexpr size_t smem = (size_t)STAGES * (A_ST + B_ST) * sizeof(double);
};

__device__ __forceinline__ void cp16(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}

template <int WM, int WN, int NWM, int NWN, int STAGES>
__global__ void __launch_bounds__(32 * NWM * NWN)
    k_gemm(const GemmShape* __restrict__ shapes, const GemmTile* __restrict__ tiles, int n_tiles) {
  using L = GemmCfg<WM, WN, NWM, NWN, STAGES>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * L::A_ST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp % NWM, wn = warp / NWM;
  for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    const GemmTile tl = tiles[ti];
    const GemmShape sh = shapes[tl.shape];
    const int nk = (sh.m + KC - 1) / KC;
    auto issue = [&](int kt) {
      const int s = kt % STAGES, k0 = kt * KC;
      double* a = sA + s * L::A_ST;
      double* b = sB + s * L::B_ST;
      for (int q = tid; q < (L::MT + L::NT) * (KC / 2); q += 32 * L::WARPS) {
        const int r = q / (KC / 2), ch = q % (KC / 2), k = k0 + 2 * ch;
        if (r < L::MT) {
          const int i = tl.i0 + r;
          const bool v = i < sh.m && k < sh.ld;
          cp16(a + r * GS + 2 * ch, v ? sh.A + (int64_t)i * sh.ld + k : sh.A, v);
        } else {
          const int rr = r - L::MT, n = tl.n0 + rr;
          const bool v = n < sh.n && k < sh.ld;
          cp16(b + rr * GS + 2 * ch, v ? sh.B + (int64_t)n * sh.ld + k : sh.B, v);
        }
      }
    };
    double acc[WM][WN][2];
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    __syncthreads();   // previous tile's last stage fully consumed
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nk) issue(s);
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (kt + STAGES - 1 < nk) issue(kt + STAGES - 1);
      cp_async_commit();
      const double* a = sA + (kt % STAGES) * L::A_ST + (wm * WM * 8 + g) * GS + t;
      const double* b = sB + (kt % STAGES) * L::B_ST + (wn * WN * 8 + g) * GS + t;
#pragma unroll
      for (int kk = 0; kk < KC / 4; ++kk) {
        double af[WM], bf[WN];
#pragma unroll
        for (int i = 0; i < WM; ++i) af[i] = a[i * 8 * GS + kk * 4];
#pragma unroll
        for (int j = 0; j < WN; ++j) bf[j] = b[j * 8 * GS + kk * 4];
#pragma unroll
        for (int i = 0; i < WM; ++i)
#pragma unroll
          for (int j = 0; j < WN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    cp_async_wait<0>();
    // C[n][i]: lanes of equal t cover 8 consecutive i -> 64-byte segments
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const int row = tl.i0 + wm * WM * 8 + i * 8 + g;
      if (row >= sh.m) continue;
#pragma unroll
      for (int j = 0; j < WN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = tl.n0 + wn * WN * 8 + j * 8 + 2 * t + h;
          if (n < sh.n) sh.C[(int64_t)n * sh.ld + row] = acc[i][j][h];
        }
    }
  }
}

// tile configurations: wide (n >= 48): 96 x 72 CTAs, two per SM; narrow (16 < n < 48) and
// skinny (n <= 16) are C^-1-streaming (memory-bound) products: one-warp 32-row CTAs so that
// every SM streams several row panels at once.
using CfgWide = GemmCfg<4, 3, 3, 3, 3>;    //  96 x 72, 9 warps
using CfgNarrow = GemmCfg<4, 3, 1, 1, 4>;  //  32 x 24, 1 warp
using CfgSkinny = GemmCfg<4, 1, 1, 1, 4>;  //  32 x  8, 1 warp
constexpr int kCtasPerSm[3] = {1, 8, 8};

int gemm_setup() {
  FMP_CHECK_CUDA(cudaFuncSetAttribute(k_gemm<4, 3, 3, 3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)CfgWide::smem));
  FMP_CHECK_CUDA(cudaFuncSetAttribute(k_gemm<4, 3, 1, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)CfgNarrow::smem));
  FMP_CHECK_CUDA(cudaFuncSetAttribute(k_gemm<4, 1, 1, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)CfgSkinny::smem));
  return 0;
}

int gemm_config_of(int n) { return n >= 48 ? 0 : (n > 16 ? 1 : 2); }
int gemm_tile_m(int cfg) { return cfg == 0 ? CfgWide::MT : (cfg == 1 ? CfgNarrow::MT : CfgSkinny::MT); }
int gemm_tile_n(int cfg) { return cfg == 0 ? CfgWide::NT : (cfg == 1 ? CfgNarrow::NT : CfgSkinny::NT); }

// shapes/tiles are device arrays; tiles of one launch all use configuration `cfg`
int gemm_launch(int cfg, const GemmShape* shapes, const GemmTile* tiles, int n_tiles, int sms, cudaStream_t st) {
  if (n_tiles <= 0) return 0;
  const int slots = kCtasPerSm[cfg] * sms;
  const int grid = n_tiles < slots ? n_tiles : slots;
  if (cfg == 0)
    k_gemm<4, 3, 3, 3, 3><<<grid, 32 * CfgWide::WARPS, CfgWide::smem, st>>>(shapes, tiles, n_tiles);
  else if (cfg == 1)
    k_gemm<4, 3, 1, 1, 4><<<grid, 32 * CfgNarrow::WARPS, CfgNarrow::smem, st>>>(shapes, tiles, n_tiles);
  else
    k_gemm<4, 1, 1, 1, 4><<<grid, 32 * CfgSkinny::WARPS, CfgSkinny::smem, st>>>(shapes, tiles, n_tiles);
  FMP_CHECK_LAUNCH();
  return 0;
}

}  // namespace fmp
