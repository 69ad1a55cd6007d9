// Woodbury GEMM Z = C^-1 Y in FP64 accuracy on the INT8 tensor cores (tcgen05.mma kind::i8),
// by the Ozaki splitting scheme.
//
// FP64 has no tcgen05 kind; DMMA (mma.sync f64) and DFMA share one FP64 datapath (~37 TF/s,
// tools/fp64_mix.cu), which the transform kernels already saturate.  The GEMM -- 2 m^2 n_s
// flops per shape, the largest single block of the preconditioner -- is instead moved to the
// INT8 tensor pipe:
//   rows of A = C^-1 and of B = Y^T are scaled by powers of two (exponents eA_i, eB_n) into
//   (-1, 1), rounded to 8S-2 bits and cut into S balanced base-256 digits ("slices")
//   a_p, b_q in [-128, 127]:   x = 2^(e+2) sum_p d_p 2^(-8p)  (error <= 2^(e-8S+1));
//   A B^T = 2^(eA_i + eB_n + 4) * sum_L 2^(-8L) D_L,   D_L = sum_{p+q=L} a_p b_q^T  (L = 2 .. S+1),
// each D_L an exact int32 sum (|a b| <= 2^14, K <= 16384 per level with <= S pairs).  S = 7 keeps
// 54 bits per operand -- FP64-level agreement with DGEMM (tests/test_ozaki_gpu.py); dropping
// the levels above S+1 costs ~2^-72.
//
// Layout: slices are stored pre-tiled in the UMMA canonical K-major SWIZZLE_NONE layout --
// for each (128-row tile, 32-byte K chunk) the S slices are one contiguous block of
// S x [2 K-halves][16 row groups][8 rows][16 B] -- so a pipeline stage is two bulk copies
// (cp.async.bulk, mbarrier complete_tx), no tensor maps.  One CTA per SM, persistent over
// (shape, row tile, column tile); warp 4 streams operands, warp 5 issues the S(S+1)/2 MMAs
// per K chunk into S TMEM accumulators (one per level), warps 0-3 drain TMEM, combine the
// levels in FP64 and store Z.
#include <algorithm>
#include <cstdint>
#include <vector>
#include "common.cuh"
#include "ozaki.cuh"
#include "tma.cuh"

namespace fmp {

constexpr int OZ_S = 7;                 // slices per operand
constexpr int OZ_M = 128;               // rows per tile (TMEM lanes)
constexpr int OZ_WMAX = 64;             // column-tile width cap (multiple of 16): OZ_S * w <= 512 TMEM columns
constexpr int OZ_MAX_K = 16384;         // int32 headroom: S pairs x 2^14 x K < 2^31 (per K part)
constexpr int OZ_KC = 32;               // K bytes per MMA / stage
constexpr int OZ_PART = OZ_MAX_K / OZ_KC;   // K chunks per part: larger K is split into parts whose
                                             // FP64 results the epilogue adds (same CTA, in order)
constexpr int OZ_ABLK = OZ_M * OZ_KC;   // bytes of one A slice block
constexpr int OZ_STAGE = OZ_S * (OZ_ABLK + OZ_WMAX * OZ_KC);
constexpr int OZ_STAGES = 5;
constexpr int OZ_THREADS = 192;         // warps 0-3 epilogue, 4 producer, 5 MMA
constexpr int OZ_TMEM_COLS = 512;
static_assert(OZ_S * OZ_WMAX <= OZ_TMEM_COLS, "levels x width exceed TMEM");

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);   // version 1, SWIZZLE_NONE
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

// One K chunk of a tile of width W: for each A slice p, MMAs of N <= 256 against the stacked B
// slices 1..S+1-p (levels p+1..S+1).  W is a template constant so every descriptor and TMEM
// offset folds to an immediate: the issue loop is ~4 instructions per MMA.
template <int W>
__device__ __forceinline__ void issue_chunk(uint64_t da0, uint64_t db0, uint32_t tmem, bool first) {
  constexpr uint32_t IDESC0 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_M >> 4) << 24);
#pragma unroll
  for (int p = 1; p <= OZ_S; ++p) {
    const uint64_t da = da0 + (uint64_t)(((p - 1) * OZ_ABLK) >> 4);
    const uint32_t acc = (first && p == 1) ? 0u : 1u;
#pragma unroll
    for (int r0 = 0; r0 < (OZ_S + 1 - p) * W; r0 += 256) {
      const int nn = ((OZ_S + 1 - p) * W - r0) < 256 ? ((OZ_S + 1 - p) * W - r0) : 256;
      umma_i8(tmem + (uint32_t)((p - 1) * W + r0), da, db0 + (uint64_t)((r0 * 16) >> 4),
              IDESC0 | ((uint32_t)(nn >> 3) << 17), acc);
    }
  }
}

__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_ozaki(const OzShape* __restrict__ shapes, const OzTile* __restrict__ tiles, const int* __restrict__ offs,
            long long* __restrict__ prof) {
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
      for (int ti = offs[blockIdx.x]; ti < offs[blockIdx.x + 1]; ++ti) {
        const OzTile tl = tiles[ti];
        const OzShape sh = shapes[tl.shape];
        const int8_t* a = sh.A + (size_t)tl.mt * sh.kchunks * OZ_S * OZ_ABLK;
        const uint32_t bblk = (uint32_t)sh.w * OZ_KC;
        const int8_t* b = sh.B + (size_t)tl.nt * sh.kchunks * OZ_S * bblk;
        const int k0 = tl.kpart * OZ_PART, k1 = min(sh.kchunks, k0 + OZ_PART);
        for (int kc = k0; kc < k1; ++kc, ++it) {
          const int s = it % OZ_STAGES;
          const uint32_t ph = (it / OZ_STAGES) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = osm + s * OZ_STAGE;
          mbar_expect_tx(&full_bar[s], OZ_S * (OZ_ABLK + bblk));
          bulk_g2s(st, a + (size_t)kc * OZ_S * OZ_ABLK, OZ_S * OZ_ABLK, &full_bar[s]);
          bulk_g2s(st + OZ_S * OZ_ABLK, b + (size_t)kc * OZ_S * bblk, OZ_S * bblk, &full_bar[s]);
        }
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer.  Level L = p + q accumulates in TMEM columns [(L-2) w, (L-1) w).
    // The B slices of a stage are stacked along N ([K half][q][w rows]), so for a fixed A slice p
    // ONE MMA of N = (S+1-p) w against B slices 1..S+1-p feeds levels p+1..S+1 at once (split at
    // N = 256): S+3 MMAs per K chunk instead of S(S+1)/2, each A block read from smem once per p.
    int it = 0, tcount = 0;
    long long t0 = clock64(), w_full = 0, w_empty = 0, t1;
    for (int ti = offs[blockIdx.x]; ti < offs[blockIdx.x + 1]; ++ti, ++tcount) {
      const OzTile tl = tiles[ti];
      const OzShape sh = shapes[tl.shape];
      const int w = sh.w;
      const int k0 = tl.kpart * OZ_PART, k1 = min(sh.kchunks, k0 + OZ_PART);
      const uint32_t lbo_b = (uint32_t)OZ_S * w * 16;
      if (tcount > 0) {   // the epilogue must have drained the accumulators of the previous tile
        if (prof) t1 = clock64();
        mbar_wait(&tempty_bar, (tcount - 1) & 1);
        if (prof) w_empty += clock64() - t1;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
      }
      for (int kc = k0; kc < k1; ++kc, ++it) {
        const int s = it % OZ_STAGES;
        const uint32_t ph = (it / OZ_STAGES) & 1;
        if (prof) t1 = clock64();
        mbar_wait(&full_bar[s], ph);
        if (prof) w_full += clock64() - t1;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (lane == 0) {
          const uint32_t sa = s_u32(osm + s * OZ_STAGE);
          const uint64_t da0 = umma_desc(sa, OZ_M * 16, 128);
          const uint64_t db0 = umma_desc(sa + OZ_S * OZ_ABLK, lbo_b, 128);
          const bool first = kc == k0;
          switch (w) {
            case 16: issue_chunk<16>(da0, db0, tmem, first); break;
            case 32: issue_chunk<32>(da0, db0, tmem, first); break;
            case 48: issue_chunk<48>(da0, db0, tmem, first); break;
            default: issue_chunk<64>(da0, db0, tmem, first); break;
          }
          umma_commit(&empty_bar[s]);                         // stage free once these MMAs retire
          if (kc == k1 - 1) umma_commit(&tfull_bar);  // accumulators complete
        }
        __syncwarp();
      }
    }
    if (prof && lane == 0) {   // FMP_OZ_PROF: MMA-warp cycles waiting for operands / for the epilogue
      prof[blockIdx.x * 4 + 0] = clock64() - t0;
      prof[blockIdx.x * 4 + 1] = w_full;
      prof[blockIdx.x * 4 + 2] = w_empty;
      prof[blockIdx.x * 4 + 3] = tcount;
    }
  } else {
    // ---------------- epilogue warps 0-3: lane quadrant = warp, one row per thread
    int tcount = 0;
    for (int ti = offs[blockIdx.x]; ti < offs[blockIdx.x + 1]; ++ti, ++tcount) {
      const OzTile tl = tiles[ti];
      const OzShape sh = shapes[tl.shape];
      mbar_wait(&tfull_bar, tcount & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int row = tl.mt * OZ_M + warp * 32 + lane;
      const int ea = row < sh.m ? sh.eA[row] : 0;
      for (int c0 = 0; c0 < sh.w; c0 += 16) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
        for (int L = OZ_S + 1; L >= 2; --L) {   // smallest terms first
          uint32_t v[16];
          const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((L - 2) * sh.w + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
              "[%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15])
              : "r"(addr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double wgt = ldexp(1.0, -8 * L);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = fma((double)(int)v[j], wgt, acc[j]);
        }
        if (row < sh.m) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = tl.nt * sh.w + c0 + j;
            if (n < sh.n) {
              double* z = sh.Z + (size_t)n * sh.ld + row;
              const double v = ldexp(acc[j], ea + sh.eB[n] + 4);
              *z = tl.kpart == 0 ? v : *z + v;   // later K parts: this CTA wrote the earlier ones
            }
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
// Batched over operands (OzSlice table): one CTA per padded row computes the row exponent e
// (max|x| < 2^e) and writes the row's S digit bytes per 16-byte K group into the tiled UMMA layout.

// S balanced base-256 digits of one 16-byte K group of row r, written into the tiled UMMA layout
// of tile height T ([tile][kchunk][S][2 K halves][T/8][8 rows][16 B]; B slices stacked along N)
__device__ __forceinline__ void ozaki_write_digits(const OzSlice& o, int r, int gk, int e, bool valid) {
  uint32_t w[OZ_S][4];
#pragma unroll
  for (int p = 0; p < OZ_S; ++p) w[p][0] = w[p][1] = w[p][2] = w[p][3] = 0u;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = gk * 16 + j;
    const double x = (valid && k < o.kvalid) ? o.src[(size_t)r * o.ld + k] : 0.0;
    long long V = llrint(ldexp(x, 8 * OZ_S - 2 - e));   // |V| <= 2^(8S-2)
#pragma unroll
    for (int p = OZ_S - 1; p >= 0; --p) {                // balanced base-256 digits, least significant first
      const int d = (int)(((V + 128) & 255) - 128);
      V = (V - d) >> 8;
      w[p][j >> 2] |= (uint32_t)(uint8_t)(int8_t)d << (8 * (j & 3));
    }
  }
  const int rt = r / o.T, rr = r % o.T, kc = gk / 2, kh = gk % 2;
  const size_t slice_stride = o.stacked ? (size_t)o.T * 16 : (size_t)o.T * OZ_KC;
  const size_t half_stride = o.stacked ? (size_t)OZ_S * o.T * 16 : (size_t)o.T * 16;
  uint8_t* base = reinterpret_cast<uint8_t*>(o.dst) + ((size_t)rt * o.kchunks + kc) * OZ_S * (o.T * OZ_KC) +
                  kh * half_stride + (rr / 8) * 128 + (rr % 8) * 16;
#pragma unroll
  for (int p = 0; p < OZ_S; ++p)
    *reinterpret_cast<uint4*>(base + p * slice_stride) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// One CTA per (padded) row: the row's exponent (max |x|), then its digits -- one launch, the row
// re-read from L1/L2.  Padding rows of the last tile get zero digits.
__global__ void __launch_bounds__(256) k_ozaki_slice_rows(const OzSlice* __restrict__ sl, int count) {
  __shared__ double red[8];
  __shared__ int e_sh;
  int si = 0;
  while (si + 1 < count && sl[si + 1].prow0 <= (int64_t)blockIdx.x) ++si;
  const OzSlice o = sl[si];
  const int r = (int)(blockIdx.x - o.prow0);
  const bool valid = r < o.rows;
  double mx = 0.0;
  if (valid) {
    const double* src = o.src + (size_t)r * o.ld;
    for (int k = threadIdx.x; k < o.kvalid; k += blockDim.x) mx = fmax(mx, fabs(src[k]));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    if (valid) o.exps[r] = e;
    e_sh = e;
  }
  __syncthreads();
  const int e = e_sh, groups = o.kchunks * (OZ_KC / 16);
  for (int gk = threadIdx.x; gk < groups; gk += blockDim.x) ozaki_write_digits(o, r, gk, e, valid);
}

void ozaki_plan_slices(OzSlice* s, int count, int64_t* rows, int64_t* threads) {
  int64_t r = 0, q = 0, pr = 0;
  for (int i = 0; i < count; ++i) {
    s[i].row0 = r;
    s[i].q0 = q;
    s[i].prow0 = pr;
    const int64_t padded = (s[i].rows + s[i].T - 1) / s[i].T * s[i].T;
    r += s[i].rows;
    q += padded * s[i].kchunks * (OZ_KC / 16);
    pr += padded;
  }
  *rows = r;
  *threads = pr;   // the slicing grid: one CTA per padded row
}

int ozaki_slice(const OzSlice* d_slices, int count, int64_t rows, int64_t padded_rows, cudaStream_t st) {
  if (count <= 0 || rows <= 0) return 0;
  k_ozaki_slice_rows<<<(unsigned)padded_rows, 256, 0, st>>>(d_slices, count);
  FMP_CHECK_LAUNCH();
  return 0;
}

int ozaki_width(int n) {
  const int nt = (n + OZ_WMAX - 1) / OZ_WMAX;
  const int w = nt > 0 ? (n + nt - 1) / nt : 1;
  return (w + 15) / 16 * 16;
}
size_t ozaki_a_bytes(int m, int kchunks) { return (size_t)((m + OZ_M - 1) / OZ_M) * kchunks * OZ_S * OZ_ABLK; }
size_t ozaki_b_bytes(int n, int kchunks) {
  const int w = ozaki_width(n);
  return (size_t)((n + w - 1) / w) * kchunks * OZ_S * w * OZ_KC;
}
int ozaki_kchunks(int m) { return (m + OZ_KC - 1) / OZ_KC; }
int ozaki_kparts(int kchunks) { return (kchunks + OZ_PART - 1) / OZ_PART; }
int ozaki_tile_m() { return OZ_M; }

int ozaki_setup() {
  FMP_CHECK_CUDA(cudaFuncSetAttribute(k_ozaki, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      OZ_STAGES * OZ_STAGE));
  return 0;
}

static long long* g_oz_prof = nullptr;   // FMP_OZ_PROF=1: per-CTA MMA-warp wait cycles (tools)

int ozaki_launch(const OzShape* shapes, const OzTile* tiles, const int* offs, int grid, cudaStream_t st) {
  if (grid <= 0) return 0;
  if (!g_oz_prof && getenv_flag("FMP_OZ_PROF")) FMP_CHECK_CUDA(cudaMalloc(&g_oz_prof, 4096 * 4 * sizeof(long long)));
  k_ozaki<<<grid, OZ_THREADS, OZ_STAGES * OZ_STAGE, st>>>(shapes, tiles, offs, g_oz_prof);
  FMP_CHECK_LAUNCH();
  return 0;
}

// Tensor-pipe cycles of one K chunk of a column tile of width w: per A slice p, one MMA per
// <= 256 columns of the stacked B slices, each >= ~46 cycles (tools/umma_rate.cu)
static double chunk_cycles(int w) {
  double c = 0.0;
  for (int p = 1; p <= OZ_S; ++p)
    for (int n = (OZ_S + 1 - p) * w; n > 0; n -= 256) c += std::max(46.0, std::min(n, 256) / 2.0);
  return c;
}

void ozaki_schedule(const std::vector<OzShape>& shapes, std::vector<OzTile>& tiles, int grid, std::vector<int>& offs) {
  // longest-processing-time-first assignment of tiles to the persistent CTAs; equal-cost tiles
  // keep their (shape, row tile, column tile) order, so CTAs working at the same time still
  // share C^-1 row tiles in L2.  Each CTA then walks its list in the original order.
  std::vector<double> cost(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) {
    const OzShape& sh = shapes[tiles[i].shape];
    const int k0 = tiles[i].kpart * OZ_PART;
    cost[i] = std::min(OZ_PART, sh.kchunks - k0) * chunk_cycles(sh.w);
  }
  // the K parts of one (shape, row tile, column tile) are one unit: same CTA, original order
  std::vector<int> unit_of(tiles.size());
  std::vector<double> ucost;
  for (size_t i = 0; i < tiles.size(); ++i) {
    const bool same = i > 0 && tiles[i].shape == tiles[i - 1].shape && tiles[i].mt == tiles[i - 1].mt &&
                      tiles[i].nt == tiles[i - 1].nt;
    if (!same) ucost.push_back(0.0);
    unit_of[i] = (int)ucost.size() - 1;
    ucost.back() += cost[i];
  }
  std::vector<int> order(ucost.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ucost[a] > ucost[b]; });
  std::vector<double> load(grid, 0.0);
  std::vector<int> cta_of_unit(ucost.size());
  for (int u : order) {
    const int c = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    load[c] += ucost[u];
    cta_of_unit[u] = c;
  }
  std::vector<std::vector<int>> lists(grid);
  for (size_t i = 0; i < tiles.size(); ++i) lists[cta_of_unit[unit_of[i]]].push_back((int)i);
  std::vector<OzTile> out;
  offs.assign(1, 0);
  for (auto& l : lists) {
    std::sort(l.begin(), l.end());
    for (int i : l) out.push_back(tiles[i]);
    offs.push_back((int)out.size());
  }
  tiles.swap(out);
}

}  // namespace fmp

// Diagnostics (tools/oz_prof.py): the last Ozaki launch's per-CTA MMA-warp cycles
// [total, waiting for operand stages, waiting for the epilogue, tiles], FMP_OZ_PROF=1 only.
extern "C" int fmp_debug_ozaki_prof(long long* out, int n) {
  if (!fmp::g_oz_prof) return -1;
  FMP_CHECK_CUDA(cudaMemcpy(out, fmp::g_oz_prof, (size_t)n * 4 * sizeof(long long), cudaMemcpyDeviceToHost));
  return 0;
}
