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
// (shape, row tile, column tile); warp 8 streams operands, warp 9 issues the S(S+1)/2 MMAs
// per K chunk into S TMEM accumulators (one per level), warps 0-7 drain TMEM (two per lane
// quadrant, alternate 8-column groups), combine the
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
constexpr int OZ_WMAX = 72;             // column-tile width cap (multiple of 8): 7 levels x 72 = 504 TMEM columns
constexpr int OZ_RMAX = 512;            // stacked B rows: pad16(S w) <= 512
constexpr int OZ_MAX_K = 16384;         // int32 headroom: S pairs x 2^14 x K < 2^31 (per K segment)
constexpr int OZ_KC = 32;               // K bytes per MMA / stage
constexpr int OZ_PART = OZ_MAX_K / OZ_KC;   // max K chunks of one segment
constexpr int OZ_ABLK = OZ_M * OZ_KC;   // bytes of one A slice block
constexpr int OZ_STAGE = OZ_S * OZ_ABLK + OZ_RMAX * OZ_KC;
constexpr int OZ_STAGES = 5;
constexpr int OZ_EPI = 8;               // epilogue warps: two per TMEM lane quadrant, each half the column groups
constexpr int OZ_THREADS = (OZ_EPI + 2) * 32;   // warps 0-7 epilogue, 8 producer, 9 MMA
constexpr int OZ_TMEM_COLS = 512;
constexpr int OZ_SLOT = OZ_WMAX * OZ_M; // doubles of one partial slot ([column][row])
static_assert(OZ_S * OZ_WMAX + 8 <= OZ_TMEM_COLS, "levels x width exceed TMEM");
static_assert(OZ_STAGES * OZ_STAGE <= 227 * 1024, "stages exceed shared memory");

__host__ __device__ constexpr int oz_pad16(int x) { return (x + 15) / 16 * 16; }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);   // version 1, SWIZZLE_NONE
}

// The MMA warp runs its loop with all 32 lanes converged; each tcgen05 instruction is issued by
// the lane elect.sync picks inside the same asm block.  (Issuing under `if (lane == 0)` made
// ptxas wrap every MMA in an ELECT / BRA.U.ANY loop with an R2UR per operand: ~50 extra cycles
// per MMA, tools/umma_chunk.cu.)  elect.sync picks the same lane every time, so the commits
// track the MMAs of the thread that issued them.
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(s_u32(b))
      : "memory");
}
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// One K chunk of a tile of width W: for each A slice p, MMAs (N <= 256, multiples of 16) against
// the stacked B slices 1..S+1-p (levels p+1..S+1), N = pad16((S+1-p) W).  Level L = p + q sits in
// TMEM columns [(L-2) W, (L-1) W); the pad16 tail of an MMA reads the next stacked slice (or the
// zero rows past the last one) and lands in columns >= 7 W, which no level uses.  W is a template
// constant so every descriptor and TMEM offset folds to an immediate.
template <int W, bool REV>
__device__ __forceinline__ void issue_chunk_order(uint64_t da0, uint64_t db0, uint32_t tmem, bool first, int p0) {
  constexpr uint32_t IDESC0 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_M >> 4) << 24);
#pragma unroll
  for (int pi = 1; pi <= OZ_S; ++pi) {
    const int p = REV ? OZ_S + 1 - pi : pi;
    if (p <= p0) continue;   // leading all-zero slices of this chunk: their products are zero
    const uint64_t da = da0 + (uint64_t)(((p - 1) * OZ_ABLK) >> 4);
    const uint32_t acc = (first && p == 1) ? 0u : 1u;
    const int N = oz_pad16((OZ_S + 1 - p) * W);
    // N > 256 is split into near-equal parts (multiples of 16): an MMA costs max(N/2, ~50) cycles,
    // so 288 -> 144 + 144 beats 256 + 32 (tools/umma_chunk.cu)
    constexpr int kMax = 256;
    const int parts = (N + kMax - 1) / kMax;
    const int step = oz_pad16((N + parts - 1) / parts);
#pragma unroll
    for (int r0 = 0; r0 < N; r0 += step) {
      const int nn = (N - r0) < step ? (N - r0) : step;
      umma_i8(tmem + (uint32_t)((p - 1) * W + r0), da, db0 + (uint64_t)((r0 * 16) >> 4),
              IDESC0 | ((uint32_t)(nn >> 3) << 17), acc);
    }
  }
}
// One asm block for a whole non-first chunk of a 72-column tile, p = 7 .. 1 (REV): a single elect,
// every MMA predicated on p > p0, the descriptors and TMEM columns formed by immediate adds, so
// ptxas moves da0 / db0 / tmem into uniform registers once per chunk instead of once per MMA.
// (Generated from the same N splits as issue_chunk_order<72, true>.)
__device__ __forceinline__ void issue_chunk72_rev(uint64_t da0, uint64_t db0, uint32_t tmem, int p0) {
  asm volatile(
      "{\n\t.reg .pred e, q, en;\n\t.reg .b32 d, id;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 en, 1, 0;\n\t"
      "setp.lt.s32 q, %3, 7;\n\tand.pred q, q, e;\n\tadd.s64 a, %1, 1536;\n\t"
      "add.u32 d, %0, 432;\n\tadd.s64 b, %2, 0;\n\tmov.b32 id, 135529632;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "setp.lt.s32 q, %3, 6;\n\tand.pred q, q, e;\n\tadd.s64 a, %1, 1280;\n\t"
      "add.u32 d, %0, 360;\n\tadd.s64 b, %2, 0;\n\tmov.b32 id, 136578208;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "setp.lt.s32 q, %3, 5;\n\tand.pred q, q, e;\n\tadd.s64 a, %1, 1024;\n\t"
      "add.u32 d, %0, 288;\n\tadd.s64 b, %2, 0;\n\tmov.b32 id, 137888928;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "setp.lt.s32 q, %3, 4;\n\tand.pred q, q, e;\n\tadd.s64 a, %1, 768;\n\t"
      "add.u32 d, %0, 216;\n\tadd.s64 b, %2, 0;\n\tmov.b32 id, 136578208;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "add.u32 d, %0, 360;\n\tadd.s64 b, %2, 144;\n\tmov.b32 id, 136578208;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "setp.lt.s32 q, %3, 3;\n\tand.pred q, q, e;\n\tadd.s64 a, %1, 512;\n\t"
      "add.u32 d, %0, 144;\n\tadd.s64 b, %2, 0;\n\tmov.b32 id, 137364640;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "add.u32 d, %0, 336;\n\tadd.s64 b, %2, 192;\n\tmov.b32 id, 137102496;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "setp.lt.s32 q, %3, 2;\n\tand.pred q, q, e;\n\tadd.s64 a, %1, 256;\n\t"
      "add.u32 d, %0, 72;\n\tadd.s64 b, %2, 0;\n\tmov.b32 id, 137888928;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "add.u32 d, %0, 296;\n\tadd.s64 b, %2, 224;\n\tmov.b32 id, 137626784;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "setp.lt.s32 q, %3, 1;\n\tand.pred q, q, e;\n\tadd.s64 a, %1, 0;\n\t"
      "add.u32 d, %0, 0;\n\tadd.s64 b, %2, 0;\n\tmov.b32 id, 138413216;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "add.u32 d, %0, 256;\n\tadd.s64 b, %2, 256;\n\tmov.b32 id, 138413216;\n\t@q tcgen05.mma.cta_group::1.kind::i8 [d], a, b, id, en;\n\t"
      "}\n"
      :: "r"(tmem), "l"(da0), "l"(db0), "r"(p0));
}

// The first chunk of a tile runs p = 1 first (its acc = 0 MMA spans every level's columns); the
// others run p = S .. 1, so the chunk ends on its widest MMAs and the tensor pipe still holds
// ~256 cycles of work while the issuing warp commits, waits for the next stage and sets up.
template <int W>
__device__ __forceinline__ void issue_chunk(uint64_t da0, uint64_t db0, uint32_t tmem, bool first, bool rev, int p0) {
  if (first || !rev)
    issue_chunk_order<W, false>(da0, db0, tmem, first, first ? 0 : p0);
  else
    issue_chunk_order<W, true>(da0, db0, tmem, false, p0);
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}

__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_ozaki(const OzShape* __restrict__ shapes, const OzItem* __restrict__ items, const int* __restrict__ offs,
            double* __restrict__ zpart, int* __restrict__ counters, long long* __restrict__ prof, int dbg) {
  const bool rev = !(dbg & 16);   // FMP_OZ_DBG bit 4 (A/B): forward MMA order in every chunk
  extern __shared__ __align__(1024) uint8_t osm[];
  if (prof && threadIdx.x == 0) prof[blockIdx.x * 8 + 4] = (long long)globaltimer();
  __shared__ __align__(8) uint64_t full_bar[OZ_STAGES], empty_bar[OZ_STAGES], tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_base;
  __shared__ int last_flag;
  __shared__ int eb_sh[OZ_WMAX];   // column exponents (+4) of the epilogue's current item
  __shared__ int stage_p0[OZ_STAGES];   // leading zero slices of the chunk in each stage (producer -> MMA warp)
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
    mbar_init(&tempty_bar, OZ_EPI * 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  pdl_trigger();
  pdl_wait();   // TMEM and barriers are set up under the slicing kernel's tail; its Y slices are read below

  if (warp == OZ_EPI) {
    // ---------------- producer: two bulk copies per stage
    if (lane == 0) {
      int it = 0;
      for (int ti = offs[blockIdx.x]; ti < offs[blockIdx.x + 1]; ++ti) {
        const OzItem tl = items[ti];
        const OzShape sh = shapes[tl.shape];
        const int8_t* a = sh.A + (size_t)tl.mt * sh.kchunks * OZ_S * OZ_ABLK;
        const uint32_t bblk = (uint32_t)sh.R * OZ_KC;
        const int8_t* b = sh.B + (size_t)tl.nt * sh.kchunks * bblk;
        const int base = sh.koff[tl.mt];
        int kc_n = sh.klist[base + tl.k0], p0_n = sh.kp0[base + tl.k0];   // entry j, fetched one ahead
        for (int j = tl.k0; j < tl.k1; ++j, ++it) {
          const int kc = kc_n, p0 = j == tl.k0 ? 0 : p0_n;   // an item's first chunk zeroes every level: all slices
          if (j + 1 < tl.k1) {
            kc_n = sh.klist[base + j + 1];
            p0_n = sh.kp0[base + j + 1];
          }
          const int s = it % OZ_STAGES;
          const uint32_t ph = (it / OZ_STAGES) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          stage_p0[s] = p0;   // published to the MMA warp by the full barrier's arrive
          if (dbg & 1) {   // FMP_OZ_DBG=1 (timing diagnostics only, wrong results): no operand loads
            mbar_arrive(&full_bar[s]);
            continue;
          }
          uint8_t* st = osm + s * OZ_STAGE;
          const uint32_t abytes = (uint32_t)(OZ_S - p0) * OZ_ABLK;   // slices p0 .. S-1 land at their usual offsets
          mbar_expect_tx(&full_bar[s], abytes + bblk);
          bulk_g2s(st + p0 * OZ_ABLK, a + ((size_t)kc * OZ_S + p0) * OZ_ABLK, abytes, &full_bar[s]);
          bulk_g2s(st + OZ_S * OZ_ABLK, b + (size_t)kc * bblk, bblk, &full_bar[s]);
        }
      }
    }
  } else if (warp == OZ_EPI + 1) {
    // ---------------- MMA issuer
    int it = 0, tcount = 0;
    long long t0 = clock64(), w_full = 0, w_empty = 0, w_first = 0, t1;
    for (int ti = offs[blockIdx.x]; ti < offs[blockIdx.x + 1]; ++ti, ++tcount) {
      const OzItem tl = items[ti];
      const OzShape sh = shapes[tl.shape];
      const int w = sh.w;
      const uint32_t lbo_b = (uint32_t)sh.R * 16;
      if (tcount > 0) {   // the epilogue must have drained the accumulators of the previous item
        if (prof) t1 = clock64();
        mbar_wait(&tempty_bar, (tcount - 1) & 1);
        if (prof) w_empty += clock64() - t1;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
      }
      for (int j = tl.k0; j < tl.k1; ++j, ++it) {
        const int s = it % OZ_STAGES;
        const uint32_t ph = (it / OZ_STAGES) & 1;
        if (prof) t1 = clock64();
        mbar_wait(&full_bar[s], ph);
        if (prof) {
          const long long dt = clock64() - t1;
          w_full += dt;
          if (j == tl.k0) w_first += dt;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        {
          const int p0 = *reinterpret_cast<volatile int*>(&stage_p0[s]);
          const uint32_t sa = s_u32(osm + s * OZ_STAGE);
          const uint64_t da0 = umma_desc(sa, OZ_M * 16, 128);
          const uint64_t db0 = umma_desc(sa + OZ_S * OZ_ABLK, lbo_b, 128);
          const bool first = j == tl.k0;
          if (!(dbg & 2)) switch (w) {   // FMP_OZ_DBG=2: no MMAs
            case 8: issue_chunk<8>(da0, db0, tmem, first, rev, p0); break;
            case 16: issue_chunk<16>(da0, db0, tmem, first, rev, p0); break;
            case 24: issue_chunk<24>(da0, db0, tmem, first, rev, p0); break;
            case 32: issue_chunk<32>(da0, db0, tmem, first, rev, p0); break;
            case 40: issue_chunk<40>(da0, db0, tmem, first, rev, p0); break;
            case 48: issue_chunk<48>(da0, db0, tmem, first, rev, p0); break;
            case 56: issue_chunk<56>(da0, db0, tmem, first, rev, p0); break;
            case 64: issue_chunk<64>(da0, db0, tmem, first, rev, p0); break;
            default:
              if (!first && rev && !(dbg & 32))   // FMP_OZ_DBG bit 5 (A/B): the per-MMA form
                issue_chunk72_rev(da0, db0, tmem, p0);
              else
                issue_chunk<72>(da0, db0, tmem, first, rev, p0);
              break;
          }
          umma_commit(&empty_bar[s]);                 // stage free once these MMAs retire
          if (j == tl.k1 - 1) umma_commit(&tfull_bar);   // accumulators complete
        }
        __syncwarp();
      }
    }
    if (prof && lane == 0) {   // FMP_OZ_PROF: MMA-warp cycles waiting for operands / for the epilogue
      prof[blockIdx.x * 8 + 0] = clock64() - t0;
      prof[blockIdx.x * 8 + 1] = w_full;
      prof[blockIdx.x * 8 + 2] = w_empty;
      prof[blockIdx.x * 8 + 3] = tcount;
      prof[blockIdx.x * 8 + 6] = w_first;
    }
  } else {
    // ---------------- epilogue warps 0-7: lane quadrant = warp & 3, one row per thread
    int tcount = 0;
    for (int ti = offs[blockIdx.x]; ti < offs[blockIdx.x + 1]; ++ti, ++tcount) {
      const OzItem tl = items[ti];
      const OzShape sh = shapes[tl.shape];
      const int w = sh.w;
      const int quad = warp & 3, half = warp >> 2;   // TMEM lanes 32 quad .. +31; column groups half, half + 2, ...
      const int rr = quad * 32 + lane, row = tl.mt * OZ_M + rr;
      // operand exponents of this item, fetched while the MMAs still run: the row's into a
      // register, the tile's column exponents into shared memory (one global load per column
      // instead of one dependent L2 round trip per 8 columns inside the drain loop)
      const int ea = row < sh.m ? sh.eA[row] : 0;
      const int zrow = row < sh.m && sh.perm ? sh.perm[row] : row;   // Z row in the reference order
      asm volatile("bar.sync 1, 256;\n" ::: "memory");   // previous item's readers of eb_sh are done
      if (half == 0 && rr < w) {
        const int n = tl.nt * w + rr;
        eb_sh[rr] = n < sh.n ? sh.eB[n] + 4 : 0;
      }
      asm volatile("bar.sync 1, 256;\n" ::: "memory");
      double* part = tl.nseg > 1 ? zpart + (size_t)(tl.slot0 + tl.seg) * OZ_SLOT : nullptr;
      const int nvalid = min(w, sh.n - tl.nt * w);
      mbar_wait(&tfull_bar, tcount & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      for (int c0 = half * 8; c0 < w; c0 += 16) {
        uint32_t v[OZ_S][8];
        const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0;
#pragma unroll
        for (int L = 2; L <= OZ_S + 1; ++L) tmem_ld8(base + (uint32_t)((L - 2) * w), v[L - 2]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        // levels combined in int64 first: hi = D2 2^16 + D3 2^8 + D4 (< 2^48, exact as a double),
        // lo = D5 2^24 + D6 2^16 + D7 2^8 + D8 (< 2^56); sum_L D_L 2^-8L = 2^-32 (hi + 2^-32 lo)
        // with one rounding (fma) -- two int64 conversions instead of seven int32 ones
        static_assert(OZ_S == 7, "level combination written for S = 7");
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const long long hi = ((long long)(int)v[0][j] << 16) + ((long long)(int)v[1][j] << 8) + (long long)(int)v[2][j];
          const long long lo = ((long long)(int)v[3][j] << 24) + ((long long)(int)v[4][j] << 16) +
                               ((long long)(int)v[5][j] << 8) + (long long)(int)v[6][j];
          acc[j] = fma((double)lo, 0x1p-32, (double)hi);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = c0 + j;
          const bool ok = row < sh.m && c < nvalid;
          const int e = ea + eb_sh[c] - 32;
          // 2^e as a double (exact scaling) in the normal range, ldexp outside it
          const double val = !ok ? 0.0
                             : (e >= -1022 && e <= 1023) ? acc[j] * __longlong_as_double((long long)(e + 1023) << 52)
                                                         : ldexp(acc[j], e);
          if (part) {
            part[c * OZ_M + rr] = val;   // [column][row]: coalesced over the warp's rows
          } else if (ok) {
            sh.Z[(size_t)(tl.nt * w + c) * sh.ld + zrow] = val;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      mbar_arrive(&tempty_bar);   // the MMA warp may overwrite the accumulators now
      if (tl.nseg > 1) {
        // split tile: publish this segment, and the last segment to arrive sums all of them in
        // segment order (deterministic, independent of which CTA finishes last)
        __threadfence();
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        if (tid == 0) last_flag = atomicAdd(&counters[tl.slot0], 1) == tl.nseg - 1;
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        if (last_flag) {
          __threadfence();
          if (row < sh.m) {
            const double* src = zpart + (size_t)tl.slot0 * OZ_SLOT + rr;
            constexpr int FC = 24;   // columns per round: FC loads of one segment in flight
            for (int c0 = half * FC; c0 < nvalid; c0 += 2 * FC) {
              double s[FC];
#pragma unroll
              for (int j = 0; j < FC; ++j) s[j] = 0.0;
              for (int sg = 0; sg < tl.nseg; ++sg) {
                double v[FC];
#pragma unroll
                for (int j = 0; j < FC; ++j) v[j] = c0 + j < w ? __ldcg(src + (size_t)sg * OZ_SLOT + (c0 + j) * OZ_M) : 0.0;
#pragma unroll
                for (int j = 0; j < FC; ++j) s[j] += v[j];
              }
#pragma unroll
              for (int j = 0; j < FC; ++j)
                if (c0 + j < nvalid) sh.Z[(size_t)(tl.nt * w + c0 + j) * sh.ld + zrow] = s[j];
            }
          }
          if (tid == 0) counters[tl.slot0] = 0;   // re-armed for the next launch
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (prof && tid == 0) prof[blockIdx.x * 8 + 5] = (long long)globaltimer();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(OZ_TMEM_COLS));
}

// ---------------------------------------------------------------- slicing
// Batched over operands (OzSlice table): one CTA per padded row computes the row exponent e
// (max|x| < 2^e) and writes the row's S digit bytes per 16-byte K group into the tiled UMMA layout.

// S balanced base-256 digits of one 16-byte K group of row r, written into the tiled UMMA layout
// of tile height T.  A operand: [tile][kchunk][S][2 K halves][T/8][8 rows][16 B].  B operand
// (stacked): [tile][kchunk][2 K halves][R rows][16 B] with slice p in rows [p T, (p+1) T) and
// zero rows [S T, R) (T a multiple of 8, so every slice starts on an 8-row core matrix).
template <bool KPERM>
__device__ __forceinline__ void ozaki_write_digits(const OzSlice& o, const double* srow, int r, int gk, int e,
                                                   bool valid) {
  uint32_t w[OZ_S][4];
#pragma unroll
  for (int p = 0; p < OZ_S; ++p) w[p][0] = w[p][1] = w[p][2] = w[p][3] = 0u;
  // the group's 16 values first (read-only loads: all in flight before the digit arithmetic)
  double xs[16];
  if (KPERM && valid && gk * 16 + 15 < o.kvalid) {
    int kp[16];
    const int4* k4 = reinterpret_cast<const int4*>(o.kperm + gk * 16);   // kperm is 64-byte aligned per group
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 t = __ldg(k4 + q);
      kp[4 * q] = t.x; kp[4 * q + 1] = t.y; kp[4 * q + 2] = t.z; kp[4 * q + 3] = t.w;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) xs[j] = __ldg(srow + kp[j]);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k = gk * 16 + j;
      xs[j] = (valid && k < o.kvalid) ? __ldg(srow + (KPERM ? __ldg(o.kperm + k) : k)) : 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double x = xs[j];
    long long V = llrint(ldexp(x, 8 * OZ_S - 2 - e));   // |V| <= 2^(8S-2)
#pragma unroll
    for (int p = OZ_S - 1; p >= 0; --p) {                // balanced base-256 digits, least significant first
      const int d = (int)(((V + 128) & 255) - 128);
      V = (V - d) >> 8;
      w[p][j >> 2] |= (uint32_t)(uint8_t)(int8_t)d << (8 * (j & 3));
    }
  }
  const int rt = r / o.T, rr = r % o.T, kc = gk / 2, kh = gk % 2;
  const size_t blk = o.stacked ? (size_t)o.R * OZ_KC : (size_t)OZ_S * o.T * OZ_KC;
  const size_t slice_stride = o.stacked ? (size_t)o.T * 16 : (size_t)o.T * OZ_KC;
  const size_t half_stride = o.stacked ? (size_t)o.R * 16 : (size_t)o.T * 16;
  uint8_t* base = reinterpret_cast<uint8_t*>(o.dst) + ((size_t)rt * o.kchunks + kc) * blk + kh * half_stride +
                  (rr / 8) * 128 + (rr % 8) * 16;
#pragma unroll
  for (int p = 0; p < OZ_S; ++p)
    *reinterpret_cast<uint4*>(base + p * slice_stride) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// One CTA per (padded) row: the row's exponent (max |x|), then its digits -- one launch, the row
// re-read from L1/L2.  Padding rows of the last tile get zero digits.
constexpr int OZ_SLICE_THREADS = 512;
__global__ void __launch_bounds__(OZ_SLICE_THREADS) k_ozaki_slice_rows(const OzSlice* __restrict__ sl, int count) {
  __shared__ double red[OZ_SLICE_THREADS / 32];
  __shared__ int e_sh;
  pdl_trigger();
  pdl_wait();   // Y is the faces kernel's output
  int si = 0;
  while (si + 1 < count && sl[si + 1].prow0 <= (int64_t)blockIdx.x) ++si;
  const OzSlice o = sl[si];
  const int r = (int)(blockIdx.x - o.prow0);
  const bool valid = r < o.rows;
  double mx = 0.0;
  if (valid) {
    const double* src = o.src + (size_t)(o.rperm ? o.rperm[r] : r) * o.ld;   // the max is order-independent
    // eight independent loads in flight per thread (the row is read once from DRAM here)
    constexpr int U = 8;
    double m8[U];
#pragma unroll
    for (int u = 0; u < U; ++u) m8[u] = 0.0;
    int k = threadIdx.x;
    for (; k + (U - 1) * OZ_SLICE_THREADS < o.kvalid; k += U * OZ_SLICE_THREADS) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = src[k + u * OZ_SLICE_THREADS];
#pragma unroll
      for (int u = 0; u < U; ++u) m8[u] = fmax(m8[u], fabs(v[u]));
    }
    for (; k < o.kvalid; k += OZ_SLICE_THREADS) mx = fmax(mx, fabs(src[k]));
#pragma unroll
    for (int u = 0; u < U; ++u) mx = fmax(mx, m8[u]);
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
  const double* srow = o.src + (size_t)(valid ? (o.rperm ? o.rperm[r] : r) : 0) * o.ld;
  if (o.kperm)
    for (int gk = threadIdx.x; gk < groups; gk += blockDim.x) ozaki_write_digits<true>(o, srow, r, gk, e, valid);
  else
    for (int gk = threadIdx.x; gk < groups; gk += blockDim.x) ozaki_write_digits<false>(o, srow, r, gk, e, valid);
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
  FMP_CHECK_CUDA(launch_pdl(k_ozaki_slice_rows, (unsigned)padded_rows, OZ_SLICE_THREADS, 0, st, d_slices, count));
  FMP_CHECK_LAUNCH();
  return 0;
}

// Column tiles of at most OZ_WMAX columns, as even as possible, width a multiple of 8 (TMEM
// column offsets and 8-row core matrices of the stacked B): 216 -> 3 x 72, 72 -> 72, 8 -> 8.
int ozaki_width(int n) {
  const int nt = (n + OZ_WMAX - 1) / OZ_WMAX;
  const int w = nt > 0 ? (n + nt - 1) / nt : 1;
  return std::min(OZ_WMAX, (w + 7) / 8 * 8);
}
int ozaki_stack_rows(int w) { return oz_pad16(OZ_S * w); }
size_t ozaki_a_bytes(int m, int kchunks) { return (size_t)((m + OZ_M - 1) / OZ_M) * kchunks * OZ_S * OZ_ABLK; }
size_t ozaki_b_bytes(int n, int kchunks) {
  const int w = ozaki_width(n);
  return (size_t)((n + w - 1) / w) * kchunks * ozaki_stack_rows(w) * OZ_KC;
}
int ozaki_kchunks(int m) { return (m + OZ_KC - 1) / OZ_KC; }
int ozaki_tile_m() { return OZ_M; }

int ozaki_setup() {
  FMP_CHECK_CUDA(cudaFuncSetAttribute(k_ozaki, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      OZ_STAGES * OZ_STAGE));
  return 0;
}

static long long* g_oz_prof = nullptr;   // FMP_OZ_PROF=1: per-CTA MMA-warp wait cycles (tools)

int ozaki_launch(const OzPlan& p, cudaStream_t st) {
  if (p.grid <= 0) return 0;
  if (!g_oz_prof && getenv_flag("FMP_OZ_PROF")) FMP_CHECK_CUDA(cudaMalloc(&g_oz_prof, 4096 * 8 * sizeof(long long)));
  static const int dbg = getenv("FMP_OZ_DBG") ? atoi(getenv("FMP_OZ_DBG")) : 0;
  FMP_CHECK_CUDA(launch_pdl(k_ozaki, p.grid, OZ_THREADS, OZ_STAGES * OZ_STAGE, st, p.shapes, p.items, p.offs,
                            p.zpart, p.counters, g_oz_prof, dbg));
  FMP_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------- row order
std::vector<int> ozaki_row_order(int ex, int ey, int ez) {
  struct Pt { uint64_t key; int row; };
  std::vector<Pt> pts;
  auto morton = [](uint64_t i, uint64_t j, uint64_t k) {
    uint64_t c = 0;
    for (int b = 0; b < 10; ++b) c |= (((i >> b) & 1) << (3 * b)) | (((j >> b) & 1) << (3 * b + 1)) | (((k >> b) & 1) << (3 * b + 2));
    return c;
  };
  int row = 0;
  for (int c = 0; c < 3; ++c)   // the reference's row order (ref:subdomain.py:183-194)
    for (int k = 0; k < ez; ++k)
      for (int j = 0; j < ey; ++j)
        for (int i = 0; i < ex; ++i) {
          const bool on = c == 0 ? (j == 0 || k == 0) : c == 1 ? (i == 0 || k == 0) : (i == 0 || j == 0);
          if (on) pts.push_back(Pt{morton(i, j, k) * 4 + c, row++});
        }
  std::stable_sort(pts.begin(), pts.end(), [](const Pt& a, const Pt& b) { return a.key < b.key; });
  std::vector<int> perm(pts.size());
  for (size_t q = 0; q < pts.size(); ++q) perm[q] = pts[q].row;
  return perm;
}

// ---------------------------------------------------------------- zero-slice skipping
// C^-1 decays fast away from the diagonal (the capacitance couples nearby face points; at
// 34^3-class boxes the median 128 x 128 block of the row-scaled C^-1 is ~1e-11 of its rows'
// maxima), so most 128 x 32 B slice blocks of the leading (most significant) slices -- and
// whole chunks -- are all zero digits.  Their products are exactly zero: skipping them changes
// no bit of the result.  One warp per (row tile, K chunk) finds the leading all-zero slice
// count (S when the whole chunk is zero).
__global__ void k_ozaki_p0(const int8_t* __restrict__ A, int nchunks, uint8_t* __restrict__ p0) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= nchunks) return;
  const uint4* blk = reinterpret_cast<const uint4*>(A + (size_t)c * OZ_S * OZ_ABLK);
  int lead = OZ_S;
  for (int p = 0; p < OZ_S; ++p) {
    uint32_t any = 0;
    for (int q = lane; q < OZ_ABLK / 16; q += 32) {
      const uint4 v = __ldg(blk + p * (OZ_ABLK / 16) + q);
      any |= v.x | v.y | v.z | v.w;
    }
    if (__any_sync(0xffffffffu, any != 0)) {
      lead = p;
      break;
    }
  }
  if (lane == 0) p0[c] = (uint8_t)lead;
}

int ozaki_chunk_lists(std::vector<OzShape>& shapes, std::vector<OzLists>* lists, OzPlan* plan) {
  const bool dense = getenv_flag("FMP_OZ_DENSE");
  lists->assign(shapes.size(), OzLists{});
  std::vector<uint16_t> kl;
  std::vector<uint8_t> kp;
  std::vector<int> ko;
  std::vector<size_t> kl0(shapes.size(), 0), ko0(shapes.size(), 0);
  size_t kept = 0, total = 0;
  double mma_kept = 0.0, mma_total = 0.0;   // in units of one slice product of one chunk
  for (size_t s = 0; s < shapes.size(); ++s) {
    const OzShape& sh = shapes[s];
    if (!sh.A) continue;
    const int mtiles = (sh.m + OZ_M - 1) / OZ_M, nch = mtiles * sh.kchunks;
    FMP_REQUIRE(sh.kchunks <= 65535, "Ozaki: %d K chunks exceed the 16-bit chunk list", sh.kchunks);
    std::vector<uint8_t> h(nch, 0);
    if (!dense) {
      uint8_t* d = nullptr;
      FMP_CHECK_CUDA(cudaMalloc(&d, nch));
      k_ozaki_p0<<<(nch + 7) / 8, 256>>>(sh.A, nch, d);
      FMP_CHECK_LAUNCH();
      const cudaError_t e = cudaMemcpy(h.data(), d, nch, cudaMemcpyDeviceToHost);
      cudaFree(d);
      FMP_CHECK_CUDA(e);
    }
    OzLists& L = (*lists)[s];
    L.koff.push_back(0);
    for (int mt = 0; mt < mtiles; ++mt) {
      const size_t before = L.klist.size();
      for (int kc = 0; kc < sh.kchunks; ++kc) {
        const uint8_t lead = h[(size_t)mt * sh.kchunks + kc];
        if (lead < OZ_S) {
          L.klist.push_back((uint16_t)kc);
          L.kp0.push_back(lead);
          kept += OZ_S - lead;
          for (int p = lead + 1; p <= OZ_S; ++p) mma_kept += OZ_S + 1 - p;
        }
      }
      mma_total += (double)sh.kchunks * OZ_S * (OZ_S + 1) / 2;
      if (L.klist.size() == before) {   // an all-zero row tile still runs one chunk (it writes Z = 0)
        L.klist.push_back(0);
        L.kp0.push_back(0);
        kept += OZ_S;
      }
      L.koff.push_back((int)L.klist.size());
      total += (size_t)OZ_S * sh.kchunks;
    }
    kl0[s] = kl.size();
    ko0[s] = ko.size();
    kl.insert(kl.end(), L.klist.begin(), L.klist.end());
    kp.insert(kp.end(), L.kp0.begin(), L.kp0.end());
    ko.insert(ko.end(), L.koff.begin(), L.koff.end());
  }
  plan->kept_slices = total ? (double)kept / (double)total : 1.0;
  plan->kept_mma = mma_total > 0.0 ? mma_kept / mma_total : 1.0;
  if (kl.empty()) return 0;
  FMP_CHECK_CUDA(cudaMalloc(&plan->klist, kl.size() * sizeof(uint16_t)));
  FMP_CHECK_CUDA(cudaMalloc(&plan->kp0, kp.size()));
  FMP_CHECK_CUDA(cudaMalloc(&plan->koff, ko.size() * sizeof(int)));
  FMP_CHECK_CUDA(cudaMemcpy(plan->klist, kl.data(), kl.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
  FMP_CHECK_CUDA(cudaMemcpy(plan->kp0, kp.data(), kp.size(), cudaMemcpyHostToDevice));
  FMP_CHECK_CUDA(cudaMemcpy(plan->koff, ko.data(), ko.size() * sizeof(int), cudaMemcpyHostToDevice));
  for (size_t s = 0; s < shapes.size(); ++s) {
    if (!shapes[s].A) continue;
    shapes[s].klist = plan->klist + kl0[s];
    shapes[s].kp0 = plan->kp0 + kl0[s];
    shapes[s].koff = plan->koff + ko0[s];
  }
  if (getenv_flag("FMP_OZ_VERBOSE")) {
    size_t hist[OZ_S] = {};
    for (uint8_t v : kp) ++hist[v];
    fprintf(stderr, "ozaki chunk lists: %.3f of the C^-1 slice blocks, %.3f of the MMA work kept%s; %zu entries, "
            "leading zero slices 0..6: %zu %zu %zu %zu %zu %zu %zu\n", plan->kept_slices, plan->kept_mma,
            dense ? " (dense)" : "", kp.size(), hist[0], hist[1], hist[2], hist[3], hist[4], hist[5], hist[6]);
  }
  return 0;
}

// Cost model of one K chunk (cycles), fitted to the per-CTA MMA-warp cycles of cfg4 and 64^3
// applies with zero-slice skipping (tools/oz_prof.py with FMP_OZ_DUMP=1) and to the MMA-sequence
// probe (tools/umma_seq.cu): ~560 cycles per chunk (stage wait, commit, issue floor) plus ~0.3
// cycles per issued N column (the N/2 tensor rate, partly overlapped), with the same N splits as
// issue_chunk; every work item adds OZ_ITEM_CYCLES (accumulator drain, pipeline restart).
constexpr double OZ_ITEM_CYCLES = 8000.0;
static double chunk_cycles(int w, int p0 = 0) {
  double n_cols = 0.0;
  for (int p = p0 + 1; p <= OZ_S; ++p) n_cols += oz_pad16((OZ_S + 1 - p) * w);
  return 560.0 + 0.3 * n_cols;
}

// Work plan of one batched GEMM over the persistent CTAs (data-parallel waves + a stream-K
// remainder, after Osama et al.'s hybrid):
//  * a "tile" is (shape, 128-row tile mt, column tile nt); tiles whose K exceeds the int32 level
//    headroom (OZ_PART chunks) are cut into K parts first;
//  * "shared" parts belong to shapes with several column tiles.  They go round-robin in
//    (shape, mt, K part, nt) order, in F = floor(shared / grid) waves, so the CTAs of one wave that
//    hold the column tiles of one row tile stream the same C^-1 slice chunks at the same time (one
//    DRAM read, L2 hits for the siblings);
//  * the remaining shared parts and the "solo" parts (shapes with one column tile, e.g. 72 or 8
//    columns: C^-1 read from DRAM for few columns, HBM-heavy) are laid end to end by K chunk and
//    cut into `grid` ranges of equal modelled cost, one piece per CTA.  Each team of 3 CTAs runs
//    its piece at a different position among its waves (before wave (b/3) mod (F+1)), so the
//    HBM-heavy pieces are spread over the launch instead of all landing at its end;
//  * a tile cut into several segments is completed by the last segment to finish (partials summed
//    in segment order: deterministic).
int ozaki_build(const std::vector<OzShape>& shapes, const std::vector<OzLists>& klists, int sms, OzPlan* out) {
  // a part = list entries [k0, k1) of row tile mt, column tile nt
  struct Part { int shape, mt, nt, k0, k1, tile; };
  std::vector<Part> shared, solo;
  // per shape: modelled cycles of a chunk with p0 leading zero slices, and prefix sums of the
  // entry costs over the shape's concatenated lists
  std::vector<std::vector<double>> cyc(shapes.size()), pref(shapes.size());
  int n_tiles = 0;
  for (size_t s = 0; s < shapes.size(); ++s) {
    const OzShape& sh = shapes[s];
    if (sh.n <= 0 || !sh.A) continue;
    const OzLists& L = klists[s];
    for (int q = 0; q <= OZ_S; ++q) cyc[s].push_back(chunk_cycles(sh.w, std::min(q, OZ_S)));
    pref[s].assign(L.klist.size() + 1, 0.0);
    for (size_t e = 0; e < L.klist.size(); ++e) pref[s][e + 1] = pref[s][e] + cyc[s][L.kp0[e]];
    const int nts = (sh.n + sh.w - 1) / sh.w;
    for (int mt = 0; mt * OZ_M < sh.m; ++mt) {
      const int ne = L.koff[mt + 1] - L.koff[mt];
      const int kparts = (ne + OZ_PART - 1) / OZ_PART;   // <= 16384 K terms per accumulation
      for (int kp = 0; kp < kparts; ++kp) {
        const int k0 = (int)((int64_t)ne * kp / kparts), k1 = (int)((int64_t)ne * (kp + 1) / kparts);
        for (int nt = 0; nt < nts; ++nt)
          (nts > 1 ? shared : solo).push_back(Part{(int)s, mt, nt, k0, k1, n_tiles + nt});
      }
      n_tiles += nts;
    }
  }
  if (shared.empty() && solo.empty()) return 0;
  // modelled cycles of entries [k0, k1) of part r run as one item (its first chunk runs every slice)
  auto cost = [&](const Part& r, int k0, int k1) -> double {
    if (k1 <= k0) return 0.0;
    const std::vector<double>& P = pref[r.shape];
    const int base = klists[r.shape].koff[r.mt];
    return P[base + k1] - P[base + k0] + cyc[r.shape][0] - cyc[r.shape][klists[r.shape].kp0[base + k0]];
  };
  const int grid = std::min<int>(sms, (int)(shared.size() + solo.size()));
  // sibling teams: when every shared shape has the same number k of column tiles, the waves use
  // gw = grid - grid % k CTAs, so CTAs k t .. k t + k - 1 hold the k column tiles of one row tile
  // in EVERY wave and share one remainder position (they stream the same C^-1 chunks together;
  // siblings have the same chunk list, so the same cost); the grid % k CTAs left out of the waves
  // take a larger remainder piece instead
  int team = 0;
  for (const Part& r : shared) {
    const int nts = (shapes[r.shape].n + shapes[r.shape].w - 1) / shapes[r.shape].w;
    team = team == 0 ? nts : (team == nts ? team : -1);
  }
  const int gw = team > 1 && grid >= team ? grid - grid % team : grid;
  const int tsz = team > 1 ? team : 3;
  const char* fv = getenv("FMP_OZ_WAVES");   // diagnostics: cap the number of data-parallel waves
  int waves = (int)(shared.size() / gw);
  if (fv) waves = std::min(waves, atoi(fv));
  std::vector<Part> rest(shared.begin() + (size_t)waves * gw, shared.end());
  rest.insert(rest.end(), solo.begin(), solo.end());
  double total = 0.0;
  for (const Part& r : rest) total += cost(r, r.k0, r.k1) + OZ_ITEM_CYCLES;
  std::vector<double> wave_cost(grid, 0.0);
  for (int j = 0; j < waves; ++j)
    for (int b = 0; b < gw; ++b) {
      const Part& q = shared[(size_t)j * gw + b];
      wave_cost[b] += cost(q, q.k0, q.k1) + OZ_ITEM_CYCLES;
    }
  for (int b = 0; b < grid; ++b) total += wave_cost[b];
  // Cut the remainder into `grid` contiguous pieces (list-entry granularity) so that every CTA's
  // modelled load -- its wave items plus its piece, each item charged OZ_ITEM_CYCLES -- comes out
  // at the same level T: greedy fill for a given T, T found by bisection so that the remainder
  // is exactly used up.
  auto cut = [&](double T, std::vector<std::vector<Part>>* outp) -> double {   // the last CTA's load
    if (outp) outp->assign(grid, {});
    int b = 0;
    double load = wave_cost[0];
    for (const Part& r : rest) {
      int k = r.k0;
      while (k < r.k1) {
        int e = k;
        if (b == grid - 1) {
          e = r.k1;
        } else {
          while (e < r.k1) {
            const double cn = cost(r, k, e + 1), cp = cost(r, k, e);
            if (load + OZ_ITEM_CYCLES + cn > T) {
              if (T - (load + OZ_ITEM_CYCLES + cp) >= 0.5 * (cn - cp)) ++e;   // more than half of it fits
              break;
            }
            ++e;
          }
        }
        if (e > k) {
          if (outp) {
            Part seg = r;
            seg.k0 = k;
            seg.k1 = e;
            (*outp)[b].push_back(seg);
          }
          load += cost(r, k, e) + OZ_ITEM_CYCLES;
          k = e;
        }
        if (k < r.k1 && b < grid - 1) load = wave_cost[++b];
      }
    }
    return b == grid - 1 ? load : 0.0;
  };
  double lo = 0.0, hi = total / grid * 2.0 + OZ_ITEM_CYCLES * 8;
  for (int itn = 0; itn < 60; ++itn) {
    const double mid = 0.5 * (lo + hi);
    if (cut(mid, nullptr) > mid) lo = mid; else hi = mid;
  }
  std::vector<std::vector<Part>> piece;
  cut(hi, &piece);
  std::vector<std::vector<Part>> lists(grid);
  if (getenv_flag("FMP_OZ_NOSPLIT")) {   // tests: whole tiles round-robin, no K segments (schedule-independent sums)
    std::vector<Part> all(shared);
    all.insert(all.end(), solo.begin(), solo.end());
    for (auto& pc : piece) pc.clear();
    for (size_t i = 0; i < all.size(); ++i) piece[i % grid].push_back(all[i]);
    waves = 0;
  }
  for (int b = 0; b < grid; ++b) {
    const int pos = (b / tsz) % (waves + 1);
    for (int j = 0; j <= waves; ++j) {
      if (j == pos) lists[b].insert(lists[b].end(), piece[b].begin(), piece[b].end());
      if (j < waves && b < gw) lists[b].push_back(shared[(size_t)j * gw + b]);
    }
  }
  if (getenv_flag("FMP_OZ_DUMP")) {   // per CTA: items, modelled cost, list entries by kind (tools/oz_prof.py)
    for (int b = 0; b < grid; ++b) {
      double c = 0.0;
      long sh_ch = 0, solo_wide = 0, solo_narrow = 0, segs = 0;
      for (const Part& q : lists[b]) {
        const int nts = (shapes[q.shape].n + shapes[q.shape].w - 1) / shapes[q.shape].w;
        c += cost(q, q.k0, q.k1);
        const int ne = klists[q.shape].koff[q.mt + 1] - klists[q.shape].koff[q.mt];
        segs += (q.k1 - q.k0) < ne;
        if (nts > 1) sh_ch += q.k1 - q.k0;
        else if (shapes[q.shape].w >= 32) solo_wide += q.k1 - q.k0;
        else solo_narrow += q.k1 - q.k0;
      }
      double mma = 0.0;   // modelled tensor cycles without the per-chunk constant
      long nch = 0;
      for (const Part& q : lists[b]) {
        nch += q.k1 - q.k0;
        mma += cost(q, q.k0, q.k1) - 60.0 * (q.k1 - q.k0);
      }
      fprintf(stderr, "ozdump %d %zu %.0f %ld %ld %ld %ld %ld %.0f\n", b, lists[b].size(), c, sh_ch, solo_wide, solo_narrow,
              segs, nch, mma);
    }
  }
  // segments per tile (in K order), partial slots for the split tiles
  std::vector<std::vector<std::pair<int, int>>> segs(n_tiles);   // (k0, owner index) per tile
  std::vector<OzItem> items;
  std::vector<int> offs(1, 0);
  for (auto& l : lists) {
    for (const Part& q : l) {
      items.push_back(OzItem{q.shape, q.mt, q.nt, q.k0, q.k1, 0, 1, 0});
      segs[q.tile].emplace_back(q.k0, (int)items.size() - 1);
    }
    offs.push_back((int)items.size());
  }
  int slots = 0;
  for (auto& sg : segs) {
    if (sg.size() <= 1) continue;
    std::sort(sg.begin(), sg.end());
    for (size_t j = 0; j < sg.size(); ++j) {
      OzItem& it = items[sg[j].second];
      it.seg = (int)j;
      it.nseg = (int)sg.size();
      it.slot0 = slots;
    }
    slots += (int)sg.size();
  }
  out->n_slots = slots;
  out->grid = grid;
  out->n_items = (int)items.size();
  if (getenv_flag("FMP_OZ_VERBOSE"))
    fprintf(stderr, "ozaki schedule: %d items on %d CTAs (%d waves of %d CTAs over %zu shared parts, teams of %d; %zu solo parts; %zu remainder parts), %d split slots\n",
            out->n_items, grid, waves, gw, shared.size(), tsz, solo.size(), rest.size(), out->n_slots);
  FMP_CHECK_CUDA(cudaMalloc(&out->shapes, sizeof(OzShape) * shapes.size()));
  FMP_CHECK_CUDA(cudaMemcpy(out->shapes, shapes.data(), sizeof(OzShape) * shapes.size(), cudaMemcpyHostToDevice));
  FMP_CHECK_CUDA(cudaMalloc(&out->items, sizeof(OzItem) * items.size()));
  FMP_CHECK_CUDA(cudaMemcpy(out->items, items.data(), sizeof(OzItem) * items.size(), cudaMemcpyHostToDevice));
  FMP_CHECK_CUDA(cudaMalloc(&out->offs, sizeof(int) * offs.size()));
  FMP_CHECK_CUDA(cudaMemcpy(out->offs, offs.data(), sizeof(int) * offs.size(), cudaMemcpyHostToDevice));
  if (out->n_slots > 0) {
    FMP_CHECK_CUDA(cudaMalloc(&out->zpart, sizeof(double) * OZ_SLOT * (size_t)out->n_slots));
    FMP_CHECK_CUDA(cudaMalloc(&out->counters, sizeof(int) * out->n_slots));
    FMP_CHECK_CUDA(cudaMemset(out->counters, 0, sizeof(int) * out->n_slots));
  }
  return 0;
}

void ozaki_free(OzPlan* p) {
  cudaFree(p->klist);
  cudaFree(p->kp0);
  cudaFree(p->koff);
  cudaFree(p->shapes);
  cudaFree(p->items);
  cudaFree(p->offs);
  cudaFree(p->zpart);
  cudaFree(p->counters);
  *p = OzPlan{};
}

}  // namespace fmp

// Diagnostics (tools/oz_prof.py): the last Ozaki launch's per-CTA MMA-warp cycles
// [total, waiting for operand stages, waiting for the epilogue, tiles, CTA start ns, CTA end ns,
// -, -] (8 per CTA), FMP_OZ_PROF=1 only.
extern "C" int fmp_debug_ozaki_prof(long long* out, int n) {
  if (!fmp::g_oz_prof) return -1;
  FMP_CHECK_CUDA(cudaMemcpy(out, fmp::g_oz_prof, (size_t)n * 8 * sizeof(long long), cudaMemcpyDeviceToHost));
  return 0;
}
