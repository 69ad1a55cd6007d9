// FlashMP subdomain solves batched over every subdomain of a GPU block (K1-K6).
//
// Reference algorithm (ref:subdomain.py:265-287, ref:schwarz.py:320-339):
//     e0 = G^-1 B^-1 G r,  z = C^-1 e0[rows],  e = e0 - G^-1 B^-1 G Q z,  out = e[owned]
// with G the per-component separable SVD transform (ref:transform.py:120-160) and B^-1
// the per-point 3x3 inverse (ref:subdomain.py:137-153).  The build computes the same
// operator with the correction folded into the transformed domain:
//     y^ = B^-1 G r                        (K1 plane pass x,y; K2 column pass z + B^-1)
//     Y  = Q^T G^-1 y^                     (K5 faces: only the 2 boundary faces per comp)
//     Z  = C^-1 Y                          (one DGEMM per extended shape, all subdomains)
//     e  = G^-1 (y^ - B^-1 G Q Z)          (K6 builds the rank-structured G Q Z planes;
//                                           K3 column pass applies it + inverse z;
//                                           K4 plane pass inverse x,y, owned tile only)
// G Q Z is supported on two face planes per component, so it is two outer products in
// the transformed domain and costs O(n^3); the full transforms drop from four to two.
//
// Axis contractions run on FP64 tensor cores (DMMA m8n8k4, mma.sync) from shared
// memory.  Layout of every per-subdomain workspace slot: [c][k][j][i] for the three
// components of the extended box (x fastest), i.e. the reference's own order.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>
#include <cublas_v2.h>
#include "common.cuh"
#include "ozaki.cuh"
#include "tma.cuh"

namespace fmp {

// gemm.cu
struct GemmShape {
  const double* A;
  const double* B;
  double* C;
  int m, n, ld;
};
struct GemmTile {
  int shape, i0, n0, pad;
};
int gemm_setup();
int gemm_config_of(int n);
int gemm_tile_m(int cfg);
int gemm_tile_n(int cfg);
int gemm_launch(int cfg, const GemmShape* shapes, const GemmTile* tiles, int n_tiles, int sms, cudaStream_t st);

__host__ __device__ constexpr int pad8(int n) { return (n + 7) & ~7; }
__host__ __device__ constexpr int pad4(int n) { return (n + 3) & ~3; }
// Row stride (doubles) for an operand with pad8(n) columns: == 4 (mod 8) so the
// DMMA fragment loads (8 rows x 4 cols per warp) hit 16 distinct 8-byte banks.
__host__ __device__ constexpr int sstride(int n) { return pad8(n) + 4; }

// Workspace slots store each component as ez planes of stride ps = ex*ey rounded up to 4
// doubles (32 B), so every plane and every 8-column tile starts 32-byte aligned.
struct SubD {
  int ex, ey, ez, lx, ly, lz, ox, oy, oz, wx, wy, wz, shape, column, ps;
  int64_t ws_off, in_off;
  __device__ __forceinline__ int64_t cstride() const { return (int64_t)ps * ez; }
};

__device__ __forceinline__ SubD load_sub(const fmp_subdomain* s) {
  const int64_t* w = reinterpret_cast<const int64_t*>(s);
  SubD d;
  d.ex = (int)w[0]; d.ey = (int)w[1]; d.ez = (int)w[2];
  d.lx = (int)w[3]; d.ly = (int)w[4]; d.lz = (int)w[5];
  d.ox = (int)w[6]; d.oy = (int)w[7]; d.oz = (int)w[8];
  d.wx = (int)w[9]; d.wy = (int)w[10]; d.wz = (int)w[11];
  d.shape = (int)w[12]; d.column = (int)w[13];
  d.ws_off = w[14]; d.in_off = w[15];
  d.ps = (d.ex * d.ey + 3) & ~3;
  return d;
}

// Forward factor of component c along axis a: U^T on the component's own axis, V^T on
// the other two (ref:transform.py:120-132).  Row-major n x n; inverse = transpose.
__device__ __forceinline__ const double* fwd_factor(const double* factors, const fmp_shape& sh, int c, int a) {
  return factors + (a == c ? sh.ut_off[a] : sh.vt_off[a]);
}

// ---------------------------------------------------------------- restriction (index maps)
// Extended vectors of every subdomain, [c][k][j][i] at ws_off: the reference Exchanger's
// output (ref:schwarz.py:217-257), read with the same addressing (point_ptr) as K1.
__global__ void k_restrict(const fmp_subdomain* subs, Geo g, const double* __restrict__ src,
                           double* __restrict__ out) {
  const SubD d = load_sub(subs + blockIdx.z);
  const int c = blockIdx.y, k = blockIdx.x;
  if (k >= d.ez) return;
  const int64_t P = (int64_t)d.ex * d.ey;
  double* o = out + d.ws_off + (c * d.ez + k) * P;
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int r = q / d.ex, col = q - r * d.ex;
    const double* sp = point_ptr(g, src, c, d.lz + k, d.ly + r, d.lx + col);
    o[q] = sp ? __ldg(sp) : 0.0;
  }
}

// ---------------------------------------------------------------- K1 / K4: plane passes
// Work item = (subdomain, component, slab of nk consecutive z-planes).  nk planes are stacked
// so that both GEMMs of the 2-D transform have one combined dimension (nk*ey rows, then
// nk*ex columns) of up to MAXR = 72 = 9 DMMA tiles, which keeps the 8-padding waste on one
// side only.  One warp owns one 8-wide strip per GEMM and keeps NT independent accumulator
// tiles (ILP).  CTAs are persistent over a contiguous item range; the next slab streams in
// with cp.async (LDGSTS) while the current one is multiplied.
constexpr int MAXR = 72;
constexpr int PW = 9;                 // warps per plane CTA
constexpr int TS = 76;                // stride of the step-1 result (>= MAXR, == 4 mod 8)
__host__ __device__ constexpr int kstride(int n) { return (pad4(n) & 7) == 4 ? pad4(n) : pad4(n) + 4; }
__host__ __device__ inline int slab_planes(int ex, int ey) {
  const int a = MAXR / ex, b = MAXR / ey;
  const int m = a < b ? a : b;
  return m < 1 ? 1 : m;
}

struct PlaneArgs {
  const fmp_subdomain* subs;
  const fmp_shape* shapes;
  const double* factors;
  const int4* items;   // (sub, comp, k0, nk)
  int n_items;
  Geo g;
  const double* src;
  double* dst;
  int mode;            // FMP_SOLVE_*
};

// Load an n x n factor (row-major) into smem rows of stride s, zero padded to pad8(n) x s.
__device__ __forceinline__ void load_factor(double* dst, int s, const double* __restrict__ f, int n, int tid,
                                            int nt) {
  const int P = pad8(n);
  for (int r = 0; r < P; ++r)
    for (int c = tid; c < s; c += nt) dst[r * s + c] = (r < n && c < n) ? __ldg(f + r * n + c) : 0.0;
}

// INV = false (K1): slab of r restricted to the extended box -> Fy X Fx^T per plane -> work
// INV = true  (K4): slab of work planes -> Fy^T X Fx -> owned tile of the block field z
// NT = 8-wide tiles covering the largest x/y extent of the plan (5 for 33/34, 9 for <= 72):
// all strides are compile-time, and tiles past the current extent compute on zero padding
// instead of branching (mma.sync under a predicate costs a WARPSYNC per instruction).
template <int NT>
struct PlaneSmem {
  static constexpr int FS = NT * 8 + 4;            // factor row stride (== 4 mod 8)
  static constexpr int XS = NT * 8 + 4;            // slab row stride
  static constexpr int F = NT * 8 * FS;            // one factor
  static constexpr int X = MAXR * XS;              // one slab buffer
  static constexpr int T = NT * 8 * TS;            // step-1 result
  static constexpr size_t bytes = (size_t)(2 * F + 2 * X + T) * sizeof(double) + 2 * MAXR * sizeof(int);
};

template <bool INV, int NT>
__global__ void __launch_bounds__(PW * 32, 2) k_plane(PlaneArgs A) {
  using L = PlaneSmem<NT>;
  constexpr int FS = L::FS, XS = L::XS;
  extern __shared__ __align__(16) double smem[];
  double* sFx = smem;
  double* sFy = sFx + L::F;
  double* sXb = sFy + L::F;       // 2 x [MAXR][XS]
  double* sT = sXb + 2 * L::X;    // [NT*8][TS]
  int* sMap1 = reinterpret_cast<int*>(sT + L::T);
  int* sMap2 = sMap1 + MAXR;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int per = (A.n_items + gridDim.x - 1) / gridDim.x;
  const int beg = blockIdx.x * per, end = min(beg + per, A.n_items);
  if (beg >= end) return;
  // zero the factor and result buffers once: padding rows/cols must read as 0 (K padding)
  for (int q = tid; q < 2 * L::F; q += nth) smem[q] = 0.0;
  for (int q = tid; q < L::T; q += nth) sT[q] = 0.0;
  __syncthreads();

  auto issue = [&](int it, int buf) {
    const int4 w = A.items[it];
    const SubD d = load_sub(A.subs + w.x);
    const int c = w.y, ex = d.ex, ey = d.ey, cols = pad4(ex), rows = w.w * ey;
    const int64_t P = (int64_t)ex * ey, V = P * d.ez;
    double* X = sXb + buf * L::X;
    const bool inside = d.lx >= 0 && d.ly >= 0 && d.lz >= 0 && d.lx + ex <= A.g.bx && d.ly + ey <= A.g.by &&
                        d.lz + d.ez <= A.g.bz;
    const int rpp = nth / cols;  // rows per pass
    const int col = tid % cols, r0 = tid / cols;
    if (r0 < rpp) {
      for (int r = r0; r < rows; r += rpp) {
        const int kk = r / ey, j = r - kk * ey;
        const double* src = nullptr;
        if (col < ex) {
          if (INV) {
            src = A.src + d.ws_off + (int64_t)(c * d.ez + d.oz + w.z + kk) * d.ps + j * ex + col;
          } else if (A.mode == FMP_SOLVE_FACES) {
            src = A.src + d.in_off + c * V + (w.z + kk) * P + j * ex + col;
          } else if (inside) {
            src = A.src + fidx(A.g, c, d.lz + w.z + kk, d.ly + j, d.lx + col);
          } else {
            src = point_ptr(A.g, A.src, c, d.lz + w.z + kk, d.ly + j, d.lx + col);
          }
        }
        cp_async8(X + r * XS + col, src, A.factors);
      }
    }
  };

  int buf = 0, cur_shape = -1, cur_c = -1, cur_ey = NT * 8;
  issue(beg, 0);
  cp_async_commit();
  for (int it = beg; it < end; ++it) {
    if (it + 1 < end) issue(it + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    const int4 w = A.items[it];
    const SubD d = load_sub(A.subs + w.x);
    const int c = w.y, ex = d.ex, ey = d.ey, nk = w.w;
    const int M1 = nk * ey, N2 = nk * ex;
    __syncthreads();  // (a) slab `buf` landed for everyone; previous item fully consumed
    if (d.shape != cur_shape || c != cur_c) {
      const fmp_shape& sh = A.shapes[d.shape];
      const double* fx = fwd_factor(A.factors, sh, c, 0);
      const double* fy = fwd_factor(A.factors, sh, c, 1);
      for (int q = tid; q < ex * ex; q += nth) sFx[(q / ex) * FS + q % ex] = __ldg(fx + q);
      for (int q = tid; q < ey * ey; q += nth) sFy[(q / ey) * FS + q % ey] = __ldg(fy + q);
      if (ey < cur_ey)  // rows ey.. of T are the K padding of step 2: clear what a larger shape left
        for (int q = tid; q < (cur_ey - ey) * TS; q += nth) sT[ey * TS + q] = 0.0;
      cur_shape = d.shape;
      cur_c = c;
      cur_ey = ey;
    }
    for (int q = tid; q < MAXR; q += nth) {
      sMap1[q] = q < M1 ? ((q / ey) << 16) | (q % ey) : 0;
      sMap2[q] = q < N2 ? ((q / ex) << 16) | (q % ex) : 0;
    }
    __syncthreads();  // (b)
    const double* X = sXb + buf * L::X;
    // ---- step 1: T[j][k*ex + a] = sum_i X[(k,j)][i] Fx[a][i]   (INV: sum_a X[(k,b)][a] Fx[a][i])
    if (warp * 8 < M1) {
      double acc[NT][2];
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
      const int k4 = pad4(ex) / 4;
      const double* xa = X + (warp * 8 + g) * XS + t;
      const double* fb = INV ? sFx + t * FS + g : sFx + g * FS + t;
      for (int kk = 0; kk < k4; ++kk) {
        const double av = xa[kk * 4];
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const double bv = INV ? fb[kk * 4 * FS + n * 8] : fb[n * 8 * FS + kk * 4];
          dmma884(acc[n][0], acc[n][1], av, bv);
        }
      }
      const int r = warp * 8 + g;
      if (r < M1) {
        const int mp = sMap1[r], kk = mp >> 16, j = mp & 0xffff;
        double* trow = sT + j * TS + kk * ex;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int a = n * 8 + 2 * t;
          if (a < ex) trow[a] = acc[n][0];
          if (a + 1 < ex) trow[a + 1] = acc[n][1];
        }
      }
    }
    __syncthreads();  // (c)
    // ---- step 2: O[b][(k,a)] = sum_j Fy[b][j] T[j][(k,a)]   (INV: sum_b Fy[b][j] T[b][(k,i)])
    if (warp * 8 < N2) {
      double acc[NT][2];
#pragma unroll
      for (int m = 0; m < NT; ++m) acc[m][0] = acc[m][1] = 0.0;
      const int k4 = pad4(ey) / 4;
      const double* tb = sT + t * TS + warp * 8 + g;
      const double* fa = INV ? sFy + t * FS + g : sFy + g * FS + t;
      for (int kk = 0; kk < k4; ++kk) {
        const double bv = tb[kk * 4 * TS];
#pragma unroll
        for (int m = 0; m < NT; ++m) {
          const double av = INV ? fa[kk * 4 * FS + m * 8] : fa[m * 8 * FS + kk * 4];
          dmma884(acc[m][0], acc[m][1], av, bv);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = warp * 8 + 2 * t + h;
        if (n >= N2) continue;
        const int mp = sMap2[n], kk = mp >> 16, a = mp & 0xffff;
#pragma unroll
        for (int m = 0; m < NT; ++m) {
          const int row = m * 8 + g;
          if (row >= ey) continue;
          if (!INV) {
            A.dst[d.ws_off + (int64_t)(c * d.ez + w.z + kk) * d.ps + row * ex + a] = acc[m][h];
          } else {
            const int jo = row - d.oy, io = a - d.ox;
            if ((unsigned)jo < (unsigned)d.wy && (unsigned)io < (unsigned)d.wx)
              A.dst[fidx(A.g, c, d.lz + d.oz + w.z + kk, d.ly + row, d.lx + a)] = acc[m][h];
          }
        }
      }
    }
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------- K2 / K3: column passes
// Work item = (subdomain, 32 consecutive columns p = j*ex + i of the plane), all three
// components and all z.  The z contraction is the DMMA GEMM Fz (ez x ez) x X (ez x 32);
// each warp owns 8 columns and keeps 3 components x MT row tiles of accumulators, so the
// per-point 3x3 block solve happens in registers right after the GEMM (K2), and the
// folded Woodbury correction is applied to the tile in shared memory before the inverse
// GEMM (K3).  Persistent CTAs, cp.async double buffering as in the plane pass.
constexpr int TP = 32;
constexpr int CW = TP / 8;
constexpr int SC = TP + 4;   // tile row stride (== 4 mod 8)

struct ColArgs {
  const fmp_subdomain* subs;
  const fmp_shape* shapes;
  const double* factors;
  const int2* items;   // (sub, p0)
  int n_items;
  const double* src;
  double* dst;
  const double* corr;  // K3 only, may be null (no correction)
  int pmax;
};

template <int MT>
struct ColSmem {
  static constexpr int FS = MT * 8 + 4;      // factor row stride
  static constexpr int XR = MT * 8;          // tile rows per component
  static constexpr int F = MT * 8 * FS;
  static constexpr int X = 3 * XR * SC;      // one tile buffer (3 components)
  static constexpr size_t bytes = (size_t)(2 * F + 2 * X) * sizeof(double);
};

template <int MT, bool INV>
__global__ void __launch_bounds__(CW * 32, 2) k_column(ColArgs A) {
  using L = ColSmem<MT>;
  constexpr int FS = L::FS, XR = L::XR;
  extern __shared__ __align__(16) double smem[];
  double* sF = smem;               // [2][MT*8][FS]: V^T_z (comps x,y), U^T_z (comp z)
  double* sXb = sF + 2 * L::F;     // 2 x [3][XR][SC]
  const int tid = threadIdx.x, nth = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int per = (A.n_items + gridDim.x - 1) / gridDim.x;
  const int beg = blockIdx.x * per, end = min(beg + per, A.n_items);
  if (beg >= end) return;
  for (int q = tid; q < 2 * L::F; q += nth) sF[q] = 0.0;

  auto issue = [&](int it, int buf) {
    const int2 w = A.items[it];
    const SubD d = load_sub(A.subs + w.x);
    const int P = d.ex * d.ey, rows = pad4(d.ez);
    const int64_t V = d.cstride();
    const double* src = A.src + d.ws_off;
    double* X = sXb + buf * L::X;
    const int col = tid % TP;
    const bool cval = w.y + col < P;
    for (int r = tid / TP; r < 3 * rows; r += nth / TP) {
      const int cc = r / rows, k = r - cc * rows;
      cp_async8(X + (cc * XR + k) * SC + col,
                (cval && k < d.ez) ? src + cc * V + (int64_t)k * d.ps + w.y + col : nullptr, A.factors);
    }
  };

  int buf = 0, cur_shape = -1;
  issue(beg, 0);
  cp_async_commit();
  for (int it = beg; it < end; ++it) {
    if (it + 1 < end) issue(it + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    const int2 w = A.items[it];
    const SubD d = load_sub(A.subs + w.x);
    const fmp_shape& sh = A.shapes[d.shape];
    const int ex = d.ex, ey = d.ey, ez = d.ez, P = ex * ey, p0 = w.y;
    const int64_t V = d.cstride();
    double* X = sXb + buf * L::X;
    __syncthreads();  // (a)
    if (d.shape != cur_shape) {
      const double* fv = A.factors + sh.vt_off[2];
      const double* fu = A.factors + sh.ut_off[2];
      for (int q = tid; q < ez * ez; q += nth) {
        const int r = q / ez, cc = q - r * ez;
        sF[r * FS + cc] = __ldg(fv + q);
        sF[L::F + r * FS + cc] = __ldg(fu + q);
      }
      cur_shape = d.shape;
      __syncthreads();
    }
    const double* Sx = A.factors + sh.s_off[0];
    const double* Sy = A.factors + sh.s_off[1];
    const double* Sz = A.factors + sh.s_off[2];
    const double* QW = A.factors + sh.qw_off;
    if (INV && A.corr) {
      // y^ -= B^-1 (G Q Z): two rank-structured face terms per component (see K6)
      const double* cb = A.corr + (int64_t)w.x * 6 * A.pmax * A.pmax;
      const int pm = A.pmax, pm2 = pm * pm;
      const double* Vx = A.factors + sh.vt_off[0];
      const double* Vy = A.factors + sh.vt_off[1];
      const int col = tid % TP, p = p0 + col;
      if (p < P) {
        const int b = p / ex, a = p - b * ex;
        const double vy0 = __ldg(Vy + b * ey), vx0 = __ldg(Vx + a * ex), sx = __ldg(Sx + a), sy = __ldg(Sy + b);
        for (int cz = tid / TP; cz < ez; cz += nth / TP) {
          const double vz0 = sF[cz * FS];  // V^T_z[cz][0]
          const double dx = vz0 * cb[0 * pm2 + b * pm + a] + vy0 * cb[1 * pm2 + cz * pm + a];
          const double dy = vz0 * cb[2 * pm2 + b * pm + a] + vx0 * cb[3 * pm2 + cz * pm + b];
          const double dz = vy0 * cb[4 * pm2 + cz * pm + a] + vx0 * cb[5 * pm2 + cz * pm + b];
          const double sz = __ldg(Sz + cz);
          const double q = __ldg(QW + 2 * ((int64_t)cz * P + p)), wq = __ldg(QW + 2 * ((int64_t)cz * P + p) + 1);
          const double pr = wq * (sx * dx + sy * dy + sz * dz);
          X[(0 * XR + cz) * SC + col] -= q * dx + pr * sx;
          X[(1 * XR + cz) * SC + col] -= q * dy + pr * sy;
          X[(2 * XR + cz) * SC + col] -= q * dz + pr * sz;
        }
      }
      __syncthreads();
    }
    const int k4 = pad4(ez) / 4;
    double acc[3][MT][2];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
      for (int m = 0; m < MT; ++m) acc[cc][m][0] = acc[cc][m][1] = 0.0;
    const double* xb = X + t * SC + warp * 8 + g;
    const double* fa = INV ? sF + t * FS + g : sF + g * FS + t;
    for (int kk = 0; kk < k4; ++kk) {
      const double b0 = xb[(0 * XR + kk * 4) * SC];
      const double b1 = xb[(1 * XR + kk * 4) * SC];
      const double b2 = xb[(2 * XR + kk * 4) * SC];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const double av = INV ? fa[kk * 4 * FS + m * 8] : fa[m * 8 * FS + kk * 4];
        const double au = INV ? fa[L::F + kk * 4 * FS + m * 8] : fa[L::F + m * 8 * FS + kk * 4];
        dmma884(acc[0][m][0], acc[0][m][1], av, b0);
        dmma884(acc[1][m][0], acc[1][m][1], av, b1);
        dmma884(acc[2][m][0], acc[2][m][1], au, b2);
      }
    }
    // epilogue per row tile over the lane's column pair (16-byte stores when both are in the plane)
    double* dst = A.dst + d.ws_off;
    const int pA = p0 + warp * 8 + 2 * t;
    const bool v0 = pA < P, v1 = pA + 1 < P;
    double sx[2] = {0.0, 0.0}, sy[2] = {0.0, 0.0};
    if (!INV) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (pA + h >= P) continue;
        const int b = (pA + h) / ex, a = pA + h - b * ex;
        sx[h] = __ldg(Sx + a);
        sy[h] = __ldg(Sy + b);
      }
    }
    if (v0) {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int r = m * 8 + g;
        if (r >= ez) continue;
        double y[3][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double y0 = acc[0][m][h], y1 = acc[1][m][h], y2 = acc[2][m][h];
          if (!INV && (h == 0 || v1)) {  // B^-1 y = q y + w s (s . y)   (ref:subdomain.py:145-153, table form)
            const double sz = __ldg(Sz + r);
            const double2 qw = __ldg(reinterpret_cast<const double2*>(QW) + ((int64_t)r * P + pA + h));
            const double pr = qw.y * (sx[h] * y0 + sy[h] * y1 + sz * y2);
            y0 = qw.x * y0 + pr * sx[h];
            y1 = qw.x * y1 + pr * sy[h];
            y2 = qw.x * y2 + pr * sz;
          }
          y[0][h] = y0;
          y[1][h] = y1;
          y[2][h] = y2;
        }
        const int64_t o = (int64_t)r * d.ps + pA;
        if (v1) {
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            *reinterpret_cast<double2*>(dst + cc * V + o) = make_double2(y[cc][0], y[cc][1]);
        } else {
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) dst[cc * V + o] = y[cc][0];
        }
      }
    }
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// ================================================================ fast path (extents <= 40)
// Warp-independent variants of K1-K4.  Each warp owns whole work items (one z-plane of one
// component, or 8 columns of one subdomain), double-buffers its own inputs with cp.async and
// never waits on other warps: DMMA of one warp overlaps loads/epilogues of the others, which
// is what keeps the per-SMSP DMMA pipe (1 issue / 16 cycles, 26-cycle latency, measured by
// tools/dmma_latency.cu) busy.  The SVD factors of every distinct extent of the plan (at most
// FX_MAXE) stay resident in shared memory for the whole launch.
constexpr int FN = 40;               // padded extent (5 DMMA tiles)
constexpr int FSM = 44;              // factor / T row stride (== 4 mod 8)
constexpr int FMAT = FN * FSM;       // one padded factor matrix (doubles)
constexpr int FX_MAXE = 2;           // distinct extents with resident factors
constexpr int PXS = 36;              // plane buffer row stride (== 4 mod 8)
constexpr int PX_ROWS = 36;          // plane buffer rows (DMMA row tile 4 reads rows 36..39 of the
                                     // next buffer: finite data, discarded outputs)
constexpr int PX_BUF = PX_ROWS * PXS;
constexpr int PX_SLACK = 5 * PXS;    // after the last buffer (row tile 4 + the K-pad column overrun)
constexpr int PW_WARPS = 16;         // warps per plane CTA, each independent (4 per SMSP)
constexpr int CXS = 8;               // column tile row stride (8 columns; fragment loads are contiguous)
constexpr int CXR = 36;              // column tile rows per component (pad4 of the max extent)
constexpr int CX_BUF = 3 * CXR * CXS;  // one column tile (3 components)
constexpr int CW_WARPS = 12;         // single-buffered inverse pass
constexpr int CW_WARPS_FWD = 12;     // double-buffered forward column pass (3 warps per SM sub-partition)
constexpr int CW_WARPS_INV = 12;     // double-buffered inverse column pass (3 warps per SM sub-partition)
constexpr int FAST_MAX_EXT = CXR;    // the fast path serves plans whose extents are all <= 36

struct ExtTable {
  int n;
  int ext[FX_MAXE];
  int64_t ut[FX_MAXE], vt[FX_MAXE], sg[FX_MAXE];   // offsets in the factor buffer
};

// Resident factors: slot e holds [U^T_e, V^T_e] as zero-padded FN x FSM matrices + sigma_e.
__device__ __forceinline__ void load_resident(double* sm, const ExtTable& et, const double* factors, int tid,
                                              int nth) {
  for (int e = 0; e < et.n; ++e) {
    const int n = et.ext[e];
    for (int h = 0; h < 2; ++h) {
      const double* f = factors + (h == 0 ? et.ut[e] : et.vt[e]);
      double* m = sm + (2 * e + h) * FMAT;
      for (int q = tid; q < FMAT; q += nth) {
        const int r = q / FSM, c = q - r * FSM;
        m[q] = (r < n && c < n) ? __ldg(f + r * n + c) : 0.0;
      }
    }
    double* sg = sm + 2 * FX_MAXE * FMAT + e * FN;
    for (int q = tid; q < FN; q += nth) sg[q] = q < n ? __ldg(factors + et.sg[e] + q) : 0.0;
  }
}
__device__ __forceinline__ int ext_slot(const ExtTable& et, int n) { return (et.n > 1 && et.ext[1] == n) ? 1 : 0; }
// forward factor of component c on axis a for extent n: U^T on the own axis, V^T otherwise
__device__ __forceinline__ const double* res_factor(const double* sm, const ExtTable& et, int c, int a, int n) {
  return sm + (2 * ext_slot(et, n) + (a == c ? 0 : 1)) * FMAT;
}
__device__ __forceinline__ const double* res_sigma(const double* sm, const ExtTable& et, int n) {
  return sm + 2 * FX_MAXE * FMAT + ext_slot(et, n) * FN;
}
constexpr int RES_WORDS = 2 * FX_MAXE * FMAT + FX_MAXE * FN;

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

struct FastPlaneArgs {
  const fmp_subdomain* subs;
  const int4* items;   // (sub, comp, plane, -)
  int n_items;
  Geo g;
  const double* src;
  double* dst;
  const double* factors;
  int mode;
  ExtTable et;
  int tma_rows;        // > 0: forward planes inside the block arrive as one TMA box of PXS x tma_rows
  int interleave;      // 1: warp gw takes items gw, gw + nw, ... (round-robin plane order)
  // fused BiCGSTAB vector update (forward pass only; single block, no ghosts): the transformed
  // input is formed per point from the landed plane X of src as
  //   lc_kind 1 (fmp_precond_apply_lincomb): s = X + beta v                 (src = r)
  //   lc_kind 2 (fmp_precond_apply_bicg_p):  p = r + beta (X + gamma v)      (src = p_old)
  // and each owned point's value is written to lc_out, rounded exactly as the vector kernels
  int lc_kind;         // 0: plain apply of src
  int lc_prefetch;     // 1: L2 prefetch of the next item's operand rows (FMP_LC_PREFETCH=1, A/B)
  const double* lc_r;
  const double* lc_v;
  double lc_beta, lc_gamma;
  double* lc_out;
};

// The fused vector update over one landed forward plane (X = the plane in shared memory, src
// values), in place; owned points also go to A.lc_out.  Points outside the block stay zero (every
// operand is zero there).  U points' loads in flight per lane; (j, i) walked without division.
// Planes of subdomains inside the block take the unchecked path: one base pointer per operand,
// a point at base + j bx + i.
template <int KIND, bool INSIDE>
__device__ __forceinline__ void plane_lincomb(double* X, const FastPlaneArgs& A, const SubD& d, int c, int z,
                                              int lane) {
  const int ex = d.ex, n = ex * d.ey, kz = d.lz + z, bx = A.g.bx;
  if (!INSIDE && (unsigned)kz >= (unsigned)A.g.bz) return;
  const bool zown = z >= d.oz && z < d.oz + d.wz;
  const double beta = A.lc_beta, gamma = A.lc_gamma;
  const int64_t o0 = fidx(A.g, c, kz, d.ly, d.lx);   // may point outside the block (!INSIDE): offsets only
  const double* v0 = A.lc_v + o0;
  const double* r0 = A.lc_r + o0;
  double* s0 = A.lc_out + o0;
  int j = 0, i = lane;
  while (i >= ex) { i -= ex; ++j; }
  constexpr int U = 8;
  for (int q0 = 0; q0 < n; q0 += 32 * U) {
    double v[U], r[U];
    int jj[U], ii[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      jj[u] = j;
      ii[u] = i;
      bool ok = q0 + u * 32 + lane < n;
      if (!INSIDE) ok = ok && (unsigned)(d.ly + j) < (unsigned)A.g.by && (unsigned)(d.lx + i) < (unsigned)bx;
      const int64_t o = (int64_t)j * bx + i;
      v[u] = ok ? v0[o] : 0.0;
      if (KIND == 2) r[u] = ok ? r0[o] : 0.0;
      i += 32;
      while (i >= ex) { i -= ex; ++j; }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bool ok = q0 + u * 32 + lane < n;
      if (!INSIDE) ok = ok && (unsigned)(d.ly + jj[u]) < (unsigned)A.g.by && (unsigned)(d.lx + ii[u]) < (unsigned)bx;
      if (ok) {
        double* xp = X + jj[u] * PXS + ii[u];
        double sv;
        if (KIND == 1)   // ref:krylov.py:199, 126: s = 1.0 r + (-alpha) v
          sv = __dadd_rn(*xp, __dmul_rn(beta, v[u]));
        else             // ref:krylov.py:181-182 (k_bicg_p): p = 1.0 r + beta (1.0 p + (-omega) v)
          sv = __dadd_rn(r[u], __dmul_rn(beta, __dadd_rn(*xp, __dmul_rn(gamma, v[u]))));
        *xp = sv;
        if (zown && (unsigned)(jj[u] - d.oy) < (unsigned)d.wy && (unsigned)(ii[u] - d.ox) < (unsigned)d.wx)
          s0[(int64_t)jj[u] * bx + ii[u]] = sv;
      }
    }
  }
}

// L2 prefetch of one forward plane's rows of field f (clipped to the block): one bulk prefetch
// per row and lane
__device__ __forceinline__ void prefetch_plane_l2(const double* f, const FastPlaneArgs& A, const SubD& d, int c,
                                                  int z, int lane) {
  const int kz = d.lz + z, x0 = max(d.lx, 0), x1 = min(d.lx + d.ex, A.g.bx);
  if ((unsigned)kz >= (unsigned)A.g.bz || x1 <= x0) return;
  for (int jj = lane; jj < d.ey; jj += 32) {
    const int gy = d.ly + jj;
    if ((unsigned)gy >= (unsigned)A.g.by) continue;
    const uintptr_t s = (uintptr_t)(f + fidx(A.g, c, kz, gy, x0)) & ~(uintptr_t)15;
    const uintptr_t e = ((uintptr_t)(f + fidx(A.g, c, kz, gy, x1)) + 15) & ~(uintptr_t)15;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(s), "r"((unsigned)(e - s)) : "memory");
  }
}

template <bool INV, int NM, int nt = 5>
__device__ __forceinline__ void plane_step1(const double* X, double* T, const double* Fx, int m0, int k4, int g,
                                            int t, int coff = 0) {
  // INV: only the nt column tiles of the owned range [coff, coff + 8 nt) are produced
  // (nt is a template constant: a runtime tile count breaks the DMMA issue schedule)
  double acc[NM][5][2];
#pragma unroll
  for (int q = 0; q < NM; ++q)
#pragma unroll
    for (int n = 0; n < 5; ++n) acc[q][n][0] = acc[q][n][1] = 0.0;
  const double* fb = INV ? Fx + t * FSM + g + coff : Fx + g * FSM + t;
  const double* xa = X + (m0 * 8 + g) * PXS + t;
  for (int kk = 0; kk < k4; ++kk) {
    double av[NM];
#pragma unroll
    for (int q = 0; q < NM; ++q) av[q] = xa[q * 8 * PXS + kk * 4];
#pragma unroll
    for (int n = 0; n < 5; ++n) {
      if (n >= nt) break;
      const double bv = INV ? fb[kk * 4 * FSM + n * 8] : fb[n * 8 * FSM + kk * 4];
#pragma unroll
      for (int q = 0; q < NM; ++q) dmma884(acc[q][n][0], acc[q][n][1], av[q], bv);
    }
  }
  __syncwarp();   // every lane has read these rows of X before they are overwritten
#pragma unroll
  for (int q = 0; q < NM; ++q) {
    const int r = (m0 + q) * 8 + g;
    if (r < PX_ROWS) {
      double* tr = T + r * PXS + 2 * t;
#pragma unroll
      for (int n = 0; n < 5; ++n) {
        if (n < nt && n * 8 + 2 * t < PXS) {
          tr[n * 8] = acc[q][n][0];
          tr[n * 8 + 1] = acc[q][n][1];
        }
      }
    }
  }
}

// step 2 for NN consecutive 8-column tiles starting at n0: O[b][cols] = sum_j Fy[b][j] T[j][cols]
// (INV: only the mt row tiles of the owned rows [d.oy, d.oy + 8 mt); columns are relative to d.ox)
template <bool INV, int NN, int mt = 5>
__device__ __forceinline__ void plane_step2(const double* T, const double* Fy, const FastPlaneArgs& A, const SubD& d,
                                            int c, int kplane, int n0, int k4, int g, int t) {
  double acc[NN][5][2];
#pragma unroll
  for (int q = 0; q < NN; ++q)
#pragma unroll
    for (int m = 0; m < 5; ++m) acc[q][m][0] = acc[q][m][1] = 0.0;
  const double* fa = INV ? Fy + t * FSM + g + d.oy : Fy + g * FSM + t;
  const double* tb = T + t * PXS + n0 * 8 + g;
  for (int kk = 0; kk < k4; ++kk) {
    double bv[NN];
#pragma unroll
    for (int q = 0; q < NN; ++q) bv[q] = tb[kk * 4 * PXS + q * 8];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      if (m >= mt) break;
      const double av = INV ? fa[kk * 4 * FSM + m * 8] : fa[m * 8 * FSM + kk * 4];
#pragma unroll
      for (int q = 0; q < NN; ++q) dmma884(acc[q][m][0], acc[q][m][1], av, bv[q]);
    }
  }
  const int ex = d.ex, ey = d.ey;
  const int64_t obase = INV ? 0 : d.ws_off + (int64_t)(c * d.ez + kplane) * d.ps;
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    if (m >= mt) break;
    const int row = m * 8 + g;
    if (!INV && row >= ey) continue;
    if (INV && row >= d.wy) continue;
#pragma unroll
    for (int q = 0; q < NN; ++q) {
      // the lane's adjacent column pair: one 16-byte store when both columns are in range and the
      // pair is 16-byte aligned (even plane rows forward; the owned tile starts at an even x)
      const int col = (n0 + q) * 8 + 2 * t;
      if (!INV) {
        double* o = A.dst + obase + row * ex + col;
        if ((ex & 1) == 0 && col + 1 < ex) {
          *reinterpret_cast<double2*>(o) = make_double2(acc[q][m][0], acc[q][m][1]);
        } else {
          if (col < ex) o[0] = acc[q][m][0];
          if (col + 1 < ex) o[1] = acc[q][m][1];
        }
      } else if (col < d.wx) {
        double* o = A.dst + fidx(A.g, c, d.lz + d.oz + kplane, d.ly + d.oy + row, d.lx + d.ox + col);
        if (col + 1 < d.wx && (((uintptr_t)o) & 15) == 0) {
          *reinterpret_cast<double2*>(o) = make_double2(acc[q][m][0], acc[q][m][1]);
        } else {
          o[0] = acc[q][m][0];
          if (col + 1 < d.wx) o[1] = acc[q][m][1];
        }
      }
    }
  }
}

// LC: the fused Krylov update compiled in (0: plain apply; 1, 2: FastPlaneArgs::lc_kind), so the
// plain and fused forward passes are separate instances with their own register allocation
template <bool INV, int NT = 5, int LC = 0>   // NT: 8-row DMMA tiles per padded extent (3: extents <= 24, 5: <= 40)
__global__ void __launch_bounds__(PW_WARPS * 32, 1) k_plane_fast(const __grid_constant__ CUtensorMap tm,
                                                                  FastPlaneArgs A) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t pbar[PW_WARPS];   // per-warp TMA completion (forward planes)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  load_resident(smem, A.et, A.factors, tid, blockDim.x);
  double* T = smem + RES_WORDS + warp * PX_BUF;   // this warp's plane buffer (also the step-1 result)
  for (int q = tid; q < PW_WARPS * PX_BUF + PX_SLACK; q += blockDim.x) smem[RES_WORDS + q] = 0.0;
  if ((INV || A.tma_rows > 0) && lane == 0) {   // forward TMA boxes / inverse bulk rows
    mbar_init(&pbar[warp], 1);
    fence_mbar_init();
  }
  uint32_t tphase = 0;
  // TMA destinations must be 128-byte aligned (RES_WORDS and PX_BUF keep the warp buffers so)
  const bool tma_ok = !INV && A.tma_rows > 0 && (s_u32(T) & 127) == 0;
  pdl_trigger();
  pdl_wait();   // factors are resident; the source field is the previous kernel's output
  __syncthreads();
  const int gw = blockIdx.x * PW_WARPS + warp, nw = gridDim.x * PW_WARPS;
  const int per = (A.n_items + nw - 1) / nw;
  const int stp = A.interleave ? nw : 1;
  const int beg = A.interleave ? gw : gw * per, end = A.interleave ? A.n_items : min(beg + per, A.n_items);

  // returns the column shift of the plane data inside the buffer (16-byte superset loads);
  // no integer division in the copy loops (the XU pipe would become the bottleneck)
  auto issue = [&](const int4 w, const SubD& d) -> int {
    const int c = w.y, ex = d.ex, ey = d.ey;
    double* X = T;
    if (INV || A.mode == FMP_SOLVE_FACES) {
      const int64_t P = (int64_t)ex * ey;
      const double* base = INV ? A.src + d.ws_off + (int64_t)(c * d.ez + d.oz + w.z) * d.ps
                               : A.src + d.in_off + c * P * d.ez + w.z * P;
      if (INV && (ex & 1) == 0 && ((uintptr_t)base & 15) == 0) {
        // one bulk copy per row (rows of an even extent are 16-byte aligned), completion on the
        // warp's mbarrier; the generic reads of the previous plane precede the async writes
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_expect_tx(&pbar[warp], (uint32_t)(ex * ey * 8));
        __syncwarp();
        for (int j = lane; j < ey; j += 32) bulk_g2s(X + j * PXS, base + j * ex, (uint32_t)(ex * 8), &pbar[warp]);
        return -16;
      }
      if ((ex & 1) == 0 && ((uintptr_t)base & 15) == 0) {   // 16-byte chunks of whole rows
        const int nch = ex >> 1, ch0 = lane & 15, j0 = lane >> 4;
        for (int j = j0; j < ey; j += 2)
          for (int ch = ch0; ch < nch; ch += 16) cp_async16(X + j * PXS + 2 * ch, base + j * ex + 2 * ch);
        return 0;
      }
      int j = 0, i = lane;   // the plane is contiguous: walk it flat, tracking (j, i)
      while (i >= ex) { i -= ex; ++j; }
      for (int q = lane; q < ey * ex; q += 32) {
        cp_async8(X + j * PXS + i, base + q, A.factors);
        i += 32;
        while (i >= ex) { i -= ex; ++j; }
      }
      return 0;
    }
    const bool inside = d.lx >= 0 && d.ly >= 0 && d.lz >= 0 && d.lx + ex <= A.g.bx && d.ly + ey <= A.g.by &&
                        d.lz + d.ez <= A.g.bz;
    // the caller issues one TMA box (below); the box starts at an even x (16-byte aligned
    // inner coordinate, tools/tma_test.cu), so odd-x planes land shifted by one column
    if (!INV && inside && tma_ok) return -1 - (d.lx & 1);
    if (inside && (A.g.bx & 1) == 0) {
      const double* row0 = A.src + fidx(A.g, c, d.lz + w.z, d.ly, d.lx);
      const int shift = (int)(((uintptr_t)row0 >> 3) & 1);
      const int span = ex + shift, nch = (span + 1) >> 1;   // 16-byte chunks per row (last may be half)
      const double* a0 = row0 - shift;
      // lanes 0..15 -> even rows, 16..31 -> odd rows; chunk = lane & 15 (+16)
      const int ch0 = lane & 15, j0 = lane >> 4;
      for (int j = j0; j < ey; j += 2) {
        for (int ch = ch0; ch < nch; ch += 16) {
          const double* sp = a0 + (int64_t)j * A.g.bx + 2 * ch;
          if (2 * ch + 1 < span)
            cp_async16(X + j * PXS + 2 * ch, sp);
          else
            cp_async8(X + j * PXS + 2 * ch, sp, A.factors);   // never read past the row
        }
      }
      return shift;
    }
    for (int j = 0; j < ey; ++j)
      for (int i = lane; i < ex; i += 32)
        cp_async8(X + j * PXS + i, point_ptr(A.g, A.src, c, d.lz + w.z, d.ly + j, d.lx + i), A.factors);
    return 0;
  };

  // item metadata is software-pipelined: items[it+1] (and its subdomain record, when it
  // changes) is fetched while item it computes, so no dependent global round trip sits in
  // front of the next plane's copies
  if (beg >= end) return;
  int4 w_cur = A.items[beg];
  SubD d_cur = load_sub(A.subs + w_cur.x);
  for (int it = beg; it < end; it += stp) {
    int shift = issue(w_cur, d_cur);
    if (shift < 0 && shift != -16) {   // one TMA box: rows of PXS doubles land at stride PXS (issued here, in the
                       // kernel body: the tensor map must stay a __grid_constant__ parameter)
      fence_proxy_async();   // earlier generic accesses of the buffer before the async write
      __syncwarp();
      if (lane == 0) {
        mbar_expect_tx(&pbar[warp], (uint32_t)(PXS * A.tma_rows * 8));
        tma_load_4d(T, &tm, d_cur.lx & ~1, d_cur.ly, d_cur.lz + w_cur.z, w_cur.y, &pbar[warp]);
      }
    }
    cp_async_commit();
    const int4 w_nxt = it + stp < end ? A.items[it + stp] : w_cur;
    if (shift < 0) {   // TMA box or bulk rows
      mbar_wait(&pbar[warp], tphase);
      tphase ^= 1u;
      shift = shift == -16 ? 0 : -1 - shift;
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int4 w = w_cur;
    const SubD& d = d_cur;
    const int c = w.y;
    if (!INV && LC != 0) {
      if (A.lc_prefetch && it + stp < end) {   // the next item's operands into L2 (its record is an L1/L2 hit)
        const SubD dn = w_nxt.x != w_cur.x ? load_sub(A.subs + w_nxt.x) : d_cur;
        prefetch_plane_l2(A.lc_v, A, dn, w_nxt.y, w_nxt.z, lane);
        if (LC == 2) prefetch_plane_l2(A.lc_r, A, dn, w_nxt.y, w_nxt.z, lane);
      }
      const bool inside = d.lx >= 0 && d.ly >= 0 && d.lz >= 0 && d.lx + d.ex <= A.g.bx && d.ly + d.ey <= A.g.by &&
                          d.lz + d.ez <= A.g.bz;
      if (LC == 1) {
        if (inside)
          plane_lincomb<1, true>(T + shift, A, d, c, w.z, lane);
        else
          plane_lincomb<1, false>(T + shift, A, d, c, w.z, lane);
      } else {
        if (inside)
          plane_lincomb<2, true>(T + shift, A, d, c, w.z, lane);
        else
          plane_lincomb<2, false>(T + shift, A, d, c, w.z, lane);
      }
      __syncwarp();
    }
    const double* Fx = res_factor(smem, A.et, c, 0, d.ex);
    const double* Fy = res_factor(smem, A.et, c, 1, d.ey);
    const double* X = T + shift;
    const int k41 = pad4(d.ex) / 4, k42 = pad4(d.ey) / 4;
    // ---- step 1: T[j][a] = sum_i X[j][i] Fx[a][i]   (INV: T[b][i] = sum_a X[b][a] Fx[a][i])
    // INV (prolongation): only the owned columns / rows of the plane are formed (4 tiles
    // when the owned tile is <= 32 wide, the common case)
    if (NT == 3) {   // extents <= 24 (16^3-class subdomains): 3 tiles, 2 for an owned tile <= 16
      if (INV && d.wx <= 16 && d.wy <= 16) {
        plane_step1<INV, 2, 2>(X, T, Fx, 0, k41, g, t, d.ox);
        plane_step1<INV, 1, 2>(X, T, Fx, 2, k41, g, t, d.ox);
        __syncwarp();
        plane_step2<INV, 2, 2>(T, Fy, A, d, c, w.z, 0, k42, g, t);
      } else {
        plane_step1<INV, 2, 3>(X, T, Fx, 0, k41, g, t, INV ? d.ox : 0);
        plane_step1<INV, 1, 3>(X, T, Fx, 2, k41, g, t, INV ? d.ox : 0);
        __syncwarp();
        plane_step2<INV, 2, 3>(T, Fy, A, d, c, w.z, 0, k42, g, t);
        plane_step2<INV, 1, 3>(T, Fy, A, d, c, w.z, 2, k42, g, t);
      }
    } else if (INV && d.wx <= 32 && d.wy <= 32) {
      plane_step1<INV, 2, 4>(X, T, Fx, 0, k41, g, t, d.ox);
      plane_step1<INV, 2, 4>(X, T, Fx, 2, k41, g, t, d.ox);
      plane_step1<INV, 1, 4>(X, T, Fx, 4, k41, g, t, d.ox);
      __syncwarp();
      plane_step2<INV, 2, 4>(T, Fy, A, d, c, w.z, 0, k42, g, t);
      plane_step2<INV, 2, 4>(T, Fy, A, d, c, w.z, 2, k42, g, t);
    } else {
      plane_step1<INV, 2>(X, T, Fx, 0, k41, g, t, INV ? d.ox : 0);
      plane_step1<INV, 2>(X, T, Fx, 2, k41, g, t, INV ? d.ox : 0);
      plane_step1<INV, 1>(X, T, Fx, 4, k41, g, t, INV ? d.ox : 0);
      __syncwarp();
      // ---- step 2: O[b][a] = sum_j Fy[b][j] T[j][a]   (INV: O[j][i] = sum_b Fy[b][j] T[b][i])
      plane_step2<INV, 2>(T, Fy, A, d, c, w.z, 0, k42, g, t);
      plane_step2<INV, 2>(T, Fy, A, d, c, w.z, 2, k42, g, t);
      plane_step2<INV, 1>(T, Fy, A, d, c, w.z, 4, k42, g, t);
    }
    __syncwarp();
    if (w_nxt.x != w_cur.x) d_cur = load_sub(A.subs + w_nxt.x);
    w_cur = w_nxt;
  }
}


// 1 / x for x in [1, 1 + 12 alpha] (the block-solve denominators): hardware seed + two Newton
// steps, branch-free (__drcp_rn's special-case branch serialised the column epilogues); within
// one ulp of the correctly rounded reciprocal.
__device__ __forceinline__ double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

struct FastColArgs {
  const fmp_subdomain* subs;
  const int2* items;   // (sub, p0), 8 columns each
  int n_items;
  const double* src;
  double* dst;
  const double* factors;
  const double* corr;  // K3 only (Woodbury), may be null
  int pmax;
  double alpha;
  ExtTable et;
  int interleave;      // 1: warp gw takes items gw, gw + nw, ...; 2: CTA-contiguous ranges, warps interleaved inside
  const CUtensorMap* maps;   // k_column_fast_db: per-subdomain [3][ez][ps] maps of src (box 8 x CXR x 3), or null
  int no_rem;                // 1: the fifth row tile on DMMA too (FMP_COL_NO_REM, A/B)
  int unroll;                // 1: compile-time k loop over CXR (TMA tiles only: rows past ez are zero)
};

// K2 (INV=false): y^ = B^-1 (Fz X) over 8 columns x all z, 3 components;  K3 (INV=true): Fz^T (y^ - corr)
template <bool INV>
__global__ void __launch_bounds__(CW_WARPS * 32, 1) k_column_fast(FastColArgs A) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  load_resident(smem, A.et, A.factors, tid, blockDim.x);
  double* wbase = smem + RES_WORDS + warp * CX_BUF;   // single-buffered: 3 warps per SMSP hide the loads
  for (int q = lane; q < CX_BUF; q += 32) wbase[q] = 0.0;
  __syncthreads();
  const int gw = blockIdx.x * CW_WARPS + warp, nw = gridDim.x * CW_WARPS;
  const int per = (A.n_items + nw - 1) / nw;
  const int beg = A.interleave ? gw : gw * per, end = A.interleave ? A.n_items : min(beg + per, A.n_items);
  const int step = A.interleave ? nw : 1;
  if (beg >= end) return;

  auto issue = [&](int it) {
    const int2 w = A.items[it];
    const SubD d = load_sub(A.subs + w.x);
    const int P = d.ex * d.ey, ez = d.ez;
    const int64_t V = d.cstride();
    const double* src = A.src + d.ws_off + w.y;
    double* X = wbase;
    if (w.y + 8 <= d.ps) {   // 4 aligned 16-byte chunks per row (ps, ws_off, p0 all multiples of 4/8)
      const int ch = lane & 3;
      for (int cc = 0; cc < 3; ++cc)
        for (int k = lane >> 2; k < ez; k += 8)
          cp_async16(X + (cc * CXR + k) * CXS + 2 * ch, src + cc * V + (int64_t)k * d.ps + 2 * ch);
    } else {
      const int col = lane & 7;
      for (int cc = 0; cc < 3; ++cc)
        for (int k = lane >> 3; k < ez; k += 4)
          cp_async8(X + (cc * CXR + k) * CXS + col, w.y + col < P ? src + cc * V + (int64_t)k * d.ps + col : nullptr,
                    A.factors);
    }
  };

  for (int it = beg; it < end; it += step) {
    issue(it);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    const int2 w = A.items[it];
    const SubD d = load_sub(A.subs + w.x);
    const int ex = d.ex, ey = d.ey, ez = d.ez, P = ex * ey, p0 = w.y;
    const int64_t V = d.cstride();
    double* X = wbase;
    const double* Fv = res_factor(smem, A.et, 0, 2, ez);   // V^T_z (components x, y)
    const double* Fu = res_factor(smem, A.et, 2, 2, ez);   // U^T_z (component z)
    const double* Sx = res_sigma(smem, A.et, ex);
    const double* Sy = res_sigma(smem, A.et, ey);
    const double* Sz = res_sigma(smem, A.et, ez);
    if (INV && A.corr) {
      // y^ -= B^-1 (G Q Z): two rank-structured face terms per component (K6)
      const double* cb = A.corr + (int64_t)w.x * 6 * A.pmax * A.pmax;
      const int pm = A.pmax, pm2 = pm * pm;
      const double* Vx = res_factor(smem, A.et, 1, 0, ex);   // V^T_x
      const double* Vy = res_factor(smem, A.et, 0, 1, ey);   // V^T_y
      const int col = lane & 7, p = p0 + col;
      if (p < P) {
        const int b0 = p0 / ex;
        int b = b0, a = p - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        const double vy0 = Vy[b * FSM], vx0 = Vx[a * FSM], sx = Sx[a], sy = Sy[b];
        const double gx = cb[0 * pm2 + b * pm + a], gy = cb[2 * pm2 + b * pm + a];
        for (int cz = lane >> 3; cz < ez; cz += 4) {
          const double vz0 = Fv[cz * FSM];
          const double dx = vz0 * gx + vy0 * cb[1 * pm2 + cz * pm + a];
          const double dy = vz0 * gy + vx0 * cb[3 * pm2 + cz * pm + b];
          const double dz = vy0 * cb[4 * pm2 + cz * pm + a] + vx0 * cb[5 * pm2 + cz * pm + b];
          const double sz = Sz[cz];
          const double q = __drcp_rn(1.0 + A.alpha * (sx * sx + sy * sy + sz * sz));
          const double pr = A.alpha * (sx * dx + sy * dy + sz * dz);
          X[(0 * CXR + cz) * CXS + col] -= q * (dx + pr * sx);
          X[(1 * CXR + cz) * CXS + col] -= q * (dy + pr * sy);
          X[(2 * CXR + cz) * CXS + col] -= q * (dz + pr * sz);
        }
      }
      __syncwarp();
    }
    const int k4 = pad4(ez) / 4;
    double acc[3][5][2];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
      for (int m = 0; m < 5; ++m) acc[cc][m][0] = acc[cc][m][1] = 0.0;
    const double* xb = X + t * CXS + g;
    const double* fv = INV ? Fv + t * FSM + g : Fv + g * FSM + t;
    const double* fu = INV ? Fu + t * FSM + g : Fu + g * FSM + t;
    for (int kk = 0; kk < k4; ++kk) {
      const double b0 = xb[(0 * CXR + kk * 4) * CXS];
      const double b1 = xb[(1 * CXR + kk * 4) * CXS];
      const double b2 = xb[(2 * CXR + kk * 4) * CXS];
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        const double av = INV ? fv[kk * 4 * FSM + m * 8] : fv[m * 8 * FSM + kk * 4];
        const double au = INV ? fu[kk * 4 * FSM + m * 8] : fu[m * 8 * FSM + kk * 4];
        dmma884(acc[0][m][0], acc[0][m][1], av, b0);
        dmma884(acc[1][m][0], acc[1][m][1], av, b1);
        dmma884(acc[2][m][0], acc[2][m][1], au, b2);
      }
    }
    double* dst = A.dst + d.ws_off;
    const int b0 = p0 / ex;   // one division per item; the 8 columns advance b a few times at most
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int p = p0 + 2 * t + h;
      if (p >= P) continue;
      double sx = 0.0, sy = 0.0;
      if (!INV) {
        int b = b0, a = p - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        sx = Sx[a];
        sy = Sy[b];
      }
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        const int r = m * 8 + g;
        if (r >= ez) continue;
        double y0 = acc[0][m][h], y1 = acc[1][m][h], y2 = acc[2][m][h];
        if (!INV) {  // B^-1 y = q (y + alpha s (s . y)), q = 1/(1 + alpha |s|^2)  (ref:subdomain.py:145-153)
          const double sz = Sz[r];
          const double q = __drcp_rn(1.0 + A.alpha * (sx * sx + sy * sy + sz * sz));
          const double pr = A.alpha * (sx * y0 + sy * y1 + sz * y2);
          y0 = q * (y0 + pr * sx);
          y1 = q * (y1 + pr * sy);
          y2 = q * (y2 + pr * sz);
        }
        const int64_t o = (int64_t)r * d.ps + p;
        dst[o] = y0;
        dst[V + o] = y1;
        dst[2 * V + o] = y2;
      }
    }
    __syncwarp();
  }
}

// z mode product of one 8-column item: acc[c][m] += F(rows m) * X(column tile), MT row tiles.
// K4 > 0: a compile-time k-step count (the loop unrolls, so the next step's fragment loads
// issue under this step's DMMAs); rows past the extent are zero in both the tile and the factor.
template <bool INV, int MT, int K4 = 0>
__device__ __forceinline__ void col_mma(double (&acc)[3][5][2], const double* xb, const double* fv, const double* fu,
                                        int k4) {
#pragma unroll
  for (int kk = 0; kk < (K4 > 0 ? K4 : k4); ++kk) {
    const double b0 = xb[(0 * CXR + kk * 4) * CXS];
    const double b1 = xb[(1 * CXR + kk * 4) * CXS];
    const double b2 = xb[(2 * CXR + kk * 4) * CXS];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const double av = INV ? fv[kk * 4 * FSM + m * 8] : fv[m * 8 * FSM + kk * 4];
      const double au = INV ? fu[kk * 4 * FSM + m * 8] : fu[m * 8 * FSM + kk * 4];
      dmma884(acc[0][m][0], acc[0][m][1], av, b0);
      dmma884(acc[1][m][0], acc[1][m][1], av, b1);
      dmma884(acc[2][m][0], acc[2][m][1], au, b2);
    }
  }
}

// Double-buffered column pass for both directions (K2 forward + B^-1, K3 correction + inverse):
// 8 independent warps per SM, each over a contiguous item range.  The item metadata is
// software-pipelined (items[it+2] is fetched while item it computes; consecutive items of a
// warp share their subdomain record, reloaded only when it changes), so the cp.async of the
// next tile is issued with no dependent global round trip in front of it; the correction
// planes of K3 are read with all loads of a lane hoisted ahead of the arithmetic.
// NB = 1 (TMA only): one tile buffer per warp; the next tile is requested as soon as the DMMA
// loop has consumed the current one, so its latency hides behind the epilogue.
template <bool INV, int NW = INV ? CW_WARPS_INV : CW_WARPS_FWD, int NT = 5, int NB = 2>   // NT: z tiles (3 or 5)
__global__ void __launch_bounds__(NW * 32, 1) k_column_fast_db(FastColArgs A) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  load_resident(smem, A.et, A.factors, tid, blockDim.x);
  double* wbase = smem + RES_WORDS + warp * NB * CX_BUF;
  for (int q = lane; q < NB * CX_BUF; q += 32) wbase[q] = 0.0;
  pdl_trigger();
  pdl_wait();   // factors are resident; the source tiles are the previous kernel's output
  __syncthreads();
  const int gw = blockIdx.x * NW + warp, nw = gridDim.x * NW;
  const int per = (A.n_items + nw - 1) / nw;
  // interleaved (1): warp gw takes items gw, gw + nw, ... so the warps in flight read and write
  // neighbouring 8-column tiles (whole DRAM pages) instead of nw scattered 64-byte rows
  int stp = A.interleave ? nw : 1;
  int beg = A.interleave ? gw : gw * per, end = A.interleave ? A.n_items : min(beg + per, A.n_items);
  if (A.interleave == 2) {   // CTA-contiguous ranges, warps interleaved inside the CTA
    const int pc = (A.n_items + gridDim.x - 1) / gridDim.x;
    beg = blockIdx.x * pc + warp;
    end = min(A.n_items, (blockIdx.x + 1) * pc);
    stp = NW;
  }
  if (beg >= end) return;

  __shared__ __align__(8) uint64_t cbar[NW][2];   // TMA tile arrival, per warp and buffer
  const bool tma = A.maps != nullptr;
  if (lane == 0) {
    mbar_init(&cbar[warp][0], 1);
    mbar_init(&cbar[warp][1], 1);
    fence_mbar_init();
  }
  uint32_t phase = 0;   // bit b: parity of buffer b's next completion
  auto issue = [&](const int2 w, const SubD& d, int buf) {
    if (tma) {   // one box: 8 columns x CXR z rows x 3 components, zero-filled past ez / the plane
      if (lane == 0) {
        fence_proxy_async();   // this buffer's generic reads/writes precede the async-proxy fill
        mbar_expect_tx(&cbar[warp][buf], CX_BUF * (int)sizeof(double));
        tma_load_3d(wbase + buf * CX_BUF, A.maps + w.x, w.y, 0, 0, &cbar[warp][buf]);
      }
      return;
    }
    const int P = d.ex * d.ey, ez = d.ez;
    const int64_t V = d.cstride();
    const double* src = A.src + d.ws_off + w.y;
    double* X = wbase + buf * CX_BUF;
    if (w.y + 8 <= d.ps) {   // 4 aligned 16-byte chunks per row (ps, ws_off, p0 all multiples of 4/8)
      const int ch = lane & 3;
      for (int cc = 0; cc < 3; ++cc)
        for (int k = lane >> 2; k < ez; k += 8)
          cp_async16(X + (cc * CXR + k) * CXS + 2 * ch, src + cc * V + (int64_t)k * d.ps + 2 * ch);
    } else {
      const int col = lane & 7;
      for (int cc = 0; cc < 3; ++cc)
        for (int k = lane >> 3; k < ez; k += 4)
          cp_async8(X + (cc * CXR + k) * CXS + col, w.y + col < P ? src + cc * V + (int64_t)k * d.ps + col : nullptr,
                    A.factors);
    }
  };

  int buf = 0;
  int2 w_cur = A.items[beg];
  SubD d_cur = load_sub(A.subs + w_cur.x);
  int2 w_nxt = beg + stp < end ? A.items[beg + stp] : w_cur;
  __syncwarp();
  issue(w_cur, d_cur, 0);
  if (!tma) cp_async_commit();
  for (int it = beg; it < end; it += stp) {
    SubD d_nxt = d_cur;
    if (it + stp < end) {
      if (w_nxt.x != w_cur.x) d_nxt = load_sub(A.subs + w_nxt.x);
      if (NB == 2) issue(w_nxt, d_nxt, buf ^ 1);
    }
    const int2 w_nn = it + 2 * stp < end ? A.items[it + 2 * stp] : w_nxt;   // consumed next iteration
    if (tma) {
      mbar_wait(&cbar[warp][buf], (phase >> buf) & 1);
      phase ^= 1u << buf;
    } else {
      cp_async_commit();
      if (NB == 2)
        cp_async_wait<1>();
      else
        cp_async_wait<0>();
    }
    __syncwarp();
    const int2 w = w_cur;
    const SubD& d = d_cur;
    const int ex = d.ex, ey = d.ey, ez = d.ez, P = ex * ey, p0 = w.y;
    const int64_t V = d.cstride();
    double* X = wbase + buf * CX_BUF;
    const double* Fv = res_factor(smem, A.et, 0, 2, ez);   // V^T_z (components x, y)
    const double* Fu = res_factor(smem, A.et, 2, 2, ez);   // U^T_z (component z)
    const double* Sx = res_sigma(smem, A.et, ex);
    const double* Sy = res_sigma(smem, A.et, ey);
    const double* Sz = res_sigma(smem, A.et, ez);
    if (INV && A.corr) {
      // y^ -= B^-1 (G Q Z): two rank-structured face terms per component (K6)
      const double* cb = A.corr + (int64_t)w.x * 6 * A.pmax * A.pmax;
      const int pm = A.pmax, pm2 = pm * pm;
      const double* Vx = res_factor(smem, A.et, 1, 0, ex);   // V^T_x
      const double* Vy = res_factor(smem, A.et, 0, 1, ey);   // V^T_y
      const int col = lane & 7, p = p0 + col;
      if (p < P) {
        const int b0 = p0 / ex;
        int b = b0, a = p - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        const double vy0 = Vy[b * FSM], vx0 = Vx[a * FSM], sx = Sx[a], sy = Sy[b];
        const double gx = cb[0 * pm2 + b * pm + a], gy = cb[2 * pm2 + b * pm + a];
        constexpr int NZ = (CXR + 3) / 4;   // z rows per lane
        double c1[NZ], c3[NZ], c4[NZ], c5[NZ];
#pragma unroll
        for (int u = 0; u < NZ; ++u) {   // every load of this lane in flight at once
          const int cz = (lane >> 3) + 4 * u;
          const bool ok = cz < ez;
          c1[u] = ok ? cb[1 * pm2 + cz * pm + a] : 0.0;
          c3[u] = ok ? cb[3 * pm2 + cz * pm + b] : 0.0;
          c4[u] = ok ? cb[4 * pm2 + cz * pm + a] : 0.0;
          c5[u] = ok ? cb[5 * pm2 + cz * pm + b] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NZ; ++u) {
          const int cz = (lane >> 3) + 4 * u;
          if (cz >= ez) break;
          const double vz0 = Fv[cz * FSM];
          const double dx = vz0 * gx + vy0 * c1[u];
          const double dy = vz0 * gy + vx0 * c3[u];
          const double dz = vy0 * c4[u] + vx0 * c5[u];
          const double sz = Sz[cz];
          const double q = rcp_pos(1.0 + A.alpha * (sx * sx + sy * sy + sz * sz));
          const double pr = A.alpha * (sx * dx + sy * dy + sz * dz);
          X[(0 * CXR + cz) * CXS + col] -= q * (dx + pr * sx);
          X[(1 * CXR + cz) * CXS + col] -= q * (dy + pr * sy);
          X[(2 * CXR + cz) * CXS + col] -= q * (dz + pr * sz);
        }
      }
      __syncwarp();
    }
    const int k4 = pad4(ez) / 4;
    double acc[3][5][2];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
      for (int m = 0; m < 5; ++m) acc[cc][m][0] = acc[cc][m][1] = 0.0;
    // INV (prolongation): only the owned z rows [oz, oz + wz) are formed (4 row tiles when
    // wz <= 32; the tile count is a template constant of col_mma)
    // forward, 33/34-point columns: rows 32.. of the fifth 8-row tile would be 75-88% padding,
    // so the DMMA covers rows 0-31 and the one or two remainder rows are DFMA dot products below
    const bool rem = !INV && NT == 5 && ez > 32 && ez <= 34 && !A.no_rem;
    const int mt = NT == 3 ? (INV && d.wz <= 16 ? 2 : 3) : ((INV && d.wz <= 32) || rem ? 4 : 5);
    const double* xb = X + t * CXS + g;
    const double* fv = INV ? Fv + t * FSM + g + d.oz : Fv + g * FSM + t;
    const double* fu = INV ? Fu + t * FSM + g + d.oz : Fu + g * FSM + t;
    if (NT == 3) {
      if (mt == 2)
        col_mma<INV, 2>(acc, xb, fv, fu, k4);
      else
        col_mma<INV, 3>(acc, xb, fv, fu, k4);
    } else if (mt == 4 && A.unroll)
      col_mma<INV, 4, CXR / 4>(acc, xb, fv, fu, k4);
    else if (mt == 4)
      col_mma<INV, 4>(acc, xb, fv, fu, k4);
    else if (A.unroll)
      col_mma<INV, 5, CXR / 4>(acc, xb, fv, fu, k4);
    else
      col_mma<INV, 5>(acc, xb, fv, fu, k4);
    if (NB == 1 && it + stp < end) {   // the tile is consumed: fetch the next one under the epilogue
      __syncwarp();
      issue(w_nxt, d_nxt, 0);
    }
    double* dst = A.dst + d.ws_off;
    if (!INV && rem) {
      // remainder rows r = 32 + (lane >> 4): lanes split K in halves ((lane >> 3) & 1) and add by
      // shuffle; column lane & 7; then the 3x3 block solve of the point and its three stores
      const int rr = 32 + (lane >> 4), half = (lane >> 3) & 1, col = lane & 7;
      const int kb = half * 17, ke = min(ez, kb + 17);
      double o3[3] = {0.0, 0.0, 0.0};
      const double* fvr = Fv + min(rr, ez - 1) * FSM;
      const double* fur = Fu + min(rr, ez - 1) * FSM;
      for (int k = kb; k < ke; ++k) {
        const double fv0 = fvr[k], fu0 = fur[k];
        o3[0] = fma(fv0, X[(0 * CXR + k) * CXS + col], o3[0]);
        o3[1] = fma(fv0, X[(1 * CXR + k) * CXS + col], o3[1]);
        o3[2] = fma(fu0, X[(2 * CXR + k) * CXS + col], o3[2]);
      }
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) o3[cc] += __shfl_xor_sync(0xffffffffu, o3[cc], 8);
      const int p = p0 + col;
      if (half == 0 && rr < ez && p < P) {
        const int b0 = p0 / ex;
        int b = b0, a = p - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        const double sxv = Sx[a], syv = Sy[b], sz = Sz[rr];
        const double q = rcp_pos(1.0 + A.alpha * (sxv * sxv + syv * syv + sz * sz));
        const double pr = A.alpha * (sxv * o3[0] + syv * o3[1] + sz * o3[2]);
        const int64_t o = (int64_t)rr * d.ps + p;
        dst[o] = q * (o3[0] + pr * sxv);
        dst[V + o] = q * (o3[1] + pr * syv);
        dst[2 * V + o] = q * (o3[2] + pr * sz);
      }
    }
    // epilogue: this lane's column pair p = p0 + 2t, p + 1 (adjacent doubles, one 16-byte store
    // per row and component when both lie in the plane)
    const int pA = p0 + 2 * t;
    const bool v0 = pA < P, v1 = pA + 1 < P;
    double sx[2] = {0.0, 0.0}, sy[2] = {0.0, 0.0};
    if (!INV) {
      const int b0 = p0 / ex;   // one division per item; the 8 columns advance b a few times at most
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (pA + h >= P) continue;
        int b = b0, a = pA + h - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        sx[h] = Sx[a];
        sy[h] = Sy[b];
      }
    }
    if (v0) {
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        if (m >= mt) break;
        if (INV && m * 8 + g >= d.wz) continue;
        const int r = INV ? d.oz + m * 8 + g : m * 8 + g;
        if (r >= ez) continue;
        double y[3][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double y0 = acc[0][m][h], y1 = acc[1][m][h], y2 = acc[2][m][h];
          if (!INV) {  // B^-1 y = q (y + alpha s (s . y)), q = 1/(1 + alpha |s|^2)  (ref:subdomain.py:145-153)
            const double sz = Sz[r];
            const double q = rcp_pos(1.0 + A.alpha * (sx[h] * sx[h] + sy[h] * sy[h] + sz * sz));
            const double pr = A.alpha * (sx[h] * y0 + sy[h] * y1 + sz * y2);
            y0 = q * (y0 + pr * sx[h]);
            y1 = q * (y1 + pr * sy[h]);
            y2 = q * (y2 + pr * sz);
          }
          y[0][h] = y0;
          y[1][h] = y1;
          y[2][h] = y2;
        }
        const int64_t o = (int64_t)r * d.ps + pA;
        if (v1) {
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            *reinterpret_cast<double2*>(dst + cc * V + o) = make_double2(y[cc][0], y[cc][1]);
        } else {
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) dst[cc * V + o] = y[cc][0];
        }
      }
    }
    __syncwarp();
    buf ^= NB - 1;
    w_cur = w_nxt;
    d_cur = d_nxt;
    w_nxt = w_nn;
  }
  cp_async_wait<0>();
}

// ================================================================ large path (extents 41..72)
// Warp-independent column and plane passes for 64^3-class subdomains (extents up to 72 = 9 DMMA
// tiles), replacing the CTA-synchronous general kernels there.  Factors of every extent do not
// fit in shared memory next to 64^3-class tiles, so the host groups the work: a column-pass
// launch serves one z extent (its V^T_z / U^T_z resident), a plane-pass CTA one
// (component, ex, ey) combination (its F_x / F_y resident).
constexpr int LN = 72;                     // padded extent (9 DMMA tiles)
constexpr int LSM = 76;                    // factor / plane row stride (== 4 mod 8)
constexpr int LMAT = LN * LSM;             // one padded factor matrix (doubles)
constexpr int LCXR = 72;                   // column tile rows per component
constexpr int LCX_BUF = 3 * LCXR * CXS;    // one column tile: 3 components x 72 z x 8 columns
constexpr int LCW = 8;                     // warps per large column CTA (single-buffered tiles)
constexpr int kColLargeSmem = (2 * LMAT + LCW * LCX_BUF) * (int)sizeof(double);

struct LargeColArgs {
  const fmp_subdomain* subs;
  const fmp_shape* shapes;
  const int2* items;   // (sub, p0): 8 columns of a subdomain whose z extent is `ez`
  int n_items;
  const double* src;
  double* dst;
  const double* factors;
  int64_t ut, vt;      // U^T_z / V^T_z of extent ez (offsets into factors)
  int ez;
  const double* corr;  // K3 only (Woodbury), may be null
  int pmax;
  double alpha;
  const CUtensorMap* maps;   // per-subdomain (p, z, component) maps with box 8 x 72 x 3, or null
};

// z mode product of one 8-column item with the resident factors (stride LSM): MT row tiles
template <bool INV, int MT>
__device__ __forceinline__ void col_mma_large(double (&acc)[3][MT][2], const double* xb, const double* fv,
                                              const double* fu, int k4) {
  for (int kk = 0; kk < k4; ++kk) {
    const double b0 = xb[(0 * LCXR + kk * 4) * CXS];
    const double b1 = xb[(1 * LCXR + kk * 4) * CXS];
    const double b2 = xb[(2 * LCXR + kk * 4) * CXS];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const double av = INV ? fv[kk * 4 * LSM + m * 8] : fv[m * 8 * LSM + kk * 4];
      const double au = INV ? fu[kk * 4 * LSM + m * 8] : fu[m * 8 * LSM + kk * 4];
      dmma884(acc[0][m][0], acc[0][m][1], av, b0);
      dmma884(acc[1][m][0], acc[1][m][1], av, b1);
      dmma884(acc[2][m][0], acc[2][m][1], au, b2);
    }
  }
}

// K2 (INV=false): y^ = B^-1 (Fz X), rows 0..8MT-1 on DMMA and the remainder rows 8MT..ez-1 (at
// most 4) as DFMA dot products;  K3 (INV=true): Fz^T (y^ - corr) over the owned rows (MT tiles).
// One warp per 8-column item; the next item's tile is requested as soon as the current one is
// consumed, so its TMA latency hides behind this warp's epilogue and the other warps' DMMA.
template <bool INV, int MT>
__global__ void __launch_bounds__(LCW * 32, 1) k_column_large(LargeColArgs A) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t cbar[LCW];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  double* Fv = smem;              // V^T_z (components x, y), zero padded to LN x LSM
  double* Fu = smem + LMAT;       // U^T_z (component z)
  double* X = smem + 2 * LMAT + warp * LCX_BUF;
  const int ez = A.ez;
  for (int q = tid; q < LMAT; q += blockDim.x) {
    const int r = q / LSM, c = q - r * LSM;
    const bool ok = r < ez && c < ez;
    Fv[q] = ok ? __ldg(A.factors + A.vt + r * ez + c) : 0.0;
    Fu[q] = ok ? __ldg(A.factors + A.ut + r * ez + c) : 0.0;
  }
  for (int q = lane; q < LCX_BUF; q += 32) X[q] = 0.0;
  if (lane == 0) {
    mbar_init(&cbar[warp], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int gw = blockIdx.x * LCW + warp, nw = gridDim.x * LCW;
  if (gw >= A.n_items) return;
  const bool tma = A.maps != nullptr;
  uint32_t phase = 0;
  auto issue = [&](const int2 w, const SubD& d) {
    if (tma) {   // one box: 8 columns x 72 z rows x 3 components, zero-filled past ez / the plane
      if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(&cbar[warp], LCX_BUF * (int)sizeof(double));
        tma_load_3d(X, A.maps + w.x, w.y, 0, 0, &cbar[warp]);
      }
      return;
    }
    const int P = d.ex * d.ey;
    const int64_t V = d.cstride();
    const double* src = A.src + d.ws_off + w.y;
    const int col = lane & 7;
    for (int cc = 0; cc < 3; ++cc)
      for (int k = lane >> 3; k < LCXR; k += 4)
        cp_async8(X + (cc * LCXR + k) * CXS + col,
                  (k < d.ez && w.y + col < P) ? src + cc * V + (int64_t)k * d.ps + col : nullptr, A.factors);
    cp_async_commit();
  };
  int2 w = A.items[gw];
  SubD d = load_sub(A.subs + w.x);
  issue(w, d);
  const int k4 = pad4(ez) / 4;
  for (int it = gw; it < A.n_items; it += nw) {
    const bool more = it + nw < A.n_items;
    const int2 wn = more ? A.items[it + nw] : w;
    const SubD dn = (more && wn.x != w.x) ? load_sub(A.subs + wn.x) : d;
    const fmp_shape& sh = A.shapes[d.shape];
    const double* Sx = A.factors + sh.s_off[0];
    const double* Sy = A.factors + sh.s_off[1];
    const double* Sz = A.factors + sh.s_off[2];
    const int ex = d.ex, ey = d.ey, P = ex * ey, p0 = w.y;
    const int64_t V = d.cstride();
    if (tma) {
      mbar_wait(&cbar[warp], phase);
      phase ^= 1u;
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    if (INV && A.corr) {
      // y^ -= B^-1 (G Q Z): two rank-structured face terms per component (K6), in two halves of
      // the lane's z rows with every load of a half in flight at once
      const double* cb = A.corr + (int64_t)w.x * 6 * A.pmax * A.pmax;
      const int pm = A.pmax, pm2 = pm * pm;
      const int col = lane & 7, p = p0 + col;
      if (p < P) {
        const int b0 = p0 / ex;
        int b = b0, a = p - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        const double vy0 = __ldg(A.factors + sh.vt_off[1] + b * ey), vx0 = __ldg(A.factors + sh.vt_off[0] + a * ex);
        const double sx = __ldg(Sx + a), sy = __ldg(Sy + b);
        const double gx = cb[0 * pm2 + b * pm + a], gy = cb[2 * pm2 + b * pm + a];
        constexpr int NZ = LCXR / 8;   // z rows per lane and half
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          double c1[NZ], c3[NZ], c4[NZ], c5[NZ];
#pragma unroll
          for (int u = 0; u < NZ; ++u) {
            const int cz = (lane >> 3) + 4 * (hf * NZ + u);
            const bool ok = cz < ez;
            c1[u] = ok ? cb[1 * pm2 + cz * pm + a] : 0.0;
            c3[u] = ok ? cb[3 * pm2 + cz * pm + b] : 0.0;
            c4[u] = ok ? cb[4 * pm2 + cz * pm + a] : 0.0;
            c5[u] = ok ? cb[5 * pm2 + cz * pm + b] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < NZ; ++u) {
            const int cz = (lane >> 3) + 4 * (hf * NZ + u);
            if (cz >= ez) break;
            const double vz0 = Fv[cz * LSM];
            const double dx = vz0 * gx + vy0 * c1[u];
            const double dy = vz0 * gy + vx0 * c3[u];
            const double dz = vy0 * c4[u] + vx0 * c5[u];
            const double sz = __ldg(Sz + cz);
            const double q = rcp_pos(1.0 + A.alpha * (sx * sx + sy * sy + sz * sz));
            const double pr = A.alpha * (sx * dx + sy * dy + sz * dz);
            X[(0 * LCXR + cz) * CXS + col] -= q * (dx + pr * sx);
            X[(1 * LCXR + cz) * CXS + col] -= q * (dy + pr * sy);
            X[(2 * LCXR + cz) * CXS + col] -= q * (dz + pr * sz);
          }
        }
      }
      __syncwarp();
    }
    double acc[3][MT][2];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
      for (int m = 0; m < MT; ++m) acc[cc][m][0] = acc[cc][m][1] = 0.0;
    const double* xb = X + t * CXS + g;
    const double* fv = INV ? Fv + t * LSM + g + d.oz : Fv + g * LSM + t;
    const double* fu = INV ? Fu + t * LSM + g + d.oz : Fu + g * LSM + t;
    col_mma_large<INV, MT>(acc, xb, fv, fu, k4);
    // forward remainder rows 8MT..ez-1 (at most 4): lane -> (column lane & 7, row / K part lane >> 3)
    const int rem = INV ? 0 : ez - 8 * MT;
    double o3[3] = {0.0, 0.0, 0.0};
    int rr = 0;
    if (rem > 0) {
      const int ks = rem == 1 ? 4 : (rem == 2 ? 2 : 1);   // K parts per row
      const int sub = lane >> 3, col = lane & 7, part = sub % ks;
      rr = 8 * MT + sub / ks;
      const int kb = ez * part / ks, ke = ez * (part + 1) / ks;
      const double* fvr = Fv + min(rr, ez - 1) * LSM;
      const double* fur = Fu + min(rr, ez - 1) * LSM;
      for (int k = kb; k < ke; ++k) {
        const double fv0 = fvr[k], fu0 = fur[k];
        o3[0] = fma(fv0, X[(0 * LCXR + k) * CXS + col], o3[0]);
        o3[1] = fma(fv0, X[(1 * LCXR + k) * CXS + col], o3[1]);
        o3[2] = fma(fu0, X[(2 * LCXR + k) * CXS + col], o3[2]);
      }
      if (ks >= 2)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) o3[cc] += __shfl_xor_sync(0xffffffffu, o3[cc], 8);
      if (ks == 4)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) o3[cc] += __shfl_xor_sync(0xffffffffu, o3[cc], 16);
    }
    __syncwarp();   // the tile is consumed: fetch the next one under the epilogue
    if (more) issue(wn, dn);
    double* dst = A.dst + d.ws_off;
    if (rem > 0) {
      const int ks = rem == 1 ? 4 : (rem == 2 ? 2 : 1);
      const int sub = lane >> 3, col = lane & 7, p = p0 + col;
      if (sub % ks == 0 && rr < ez && p < P) {
        const int b0 = p0 / ex;
        int b = b0, a = p - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        const double sxv = __ldg(Sx + a), syv = __ldg(Sy + b), sz = __ldg(Sz + rr);
        const double q = rcp_pos(1.0 + A.alpha * (sxv * sxv + syv * syv + sz * sz));
        const double pr = A.alpha * (sxv * o3[0] + syv * o3[1] + sz * o3[2]);
        const int64_t o = (int64_t)rr * d.ps + p;
        dst[o] = q * (o3[0] + pr * sxv);
        dst[V + o] = q * (o3[1] + pr * syv);
        dst[2 * V + o] = q * (o3[2] + pr * sz);
      }
    }
    // epilogue: this lane's column pair p = p0 + 2t, p + 1 (one 16-byte store per row and component)
    const int pA = p0 + 2 * t;
    const bool v0 = pA < P, v1 = pA + 1 < P;
    double sx[2] = {0.0, 0.0}, sy[2] = {0.0, 0.0};
    if (!INV) {
      const int b0 = p0 / ex;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (pA + h >= P) continue;
        int b = b0, a = pA + h - b0 * ex;
        while (a >= ex) { a -= ex; ++b; }
        sx[h] = __ldg(Sx + a);
        sy[h] = __ldg(Sy + b);
      }
    }
    if (v0) {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (INV && m * 8 + g >= d.wz) continue;
        const int r = INV ? d.oz + m * 8 + g : m * 8 + g;
        if (r >= ez) continue;
        double y[3][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double y0 = acc[0][m][h], y1 = acc[1][m][h], y2 = acc[2][m][h];
          if (!INV) {  // B^-1 y = q (y + alpha s (s . y)), q = 1/(1 + alpha |s|^2)  (ref:subdomain.py:145-153)
            const double sz = __ldg(Sz + r);
            const double q = rcp_pos(1.0 + A.alpha * (sx[h] * sx[h] + sy[h] * sy[h] + sz * sz));
            const double pr = A.alpha * (sx[h] * y0 + sy[h] * y1 + sz * y2);
            y0 = q * (y0 + pr * sx[h]);
            y1 = q * (y1 + pr * sy[h]);
            y2 = q * (y2 + pr * sz);
          }
          y[0][h] = y0;
          y[1][h] = y1;
          y[2][h] = y2;
        }
        const int64_t o = (int64_t)r * d.ps + pA;
        if (v1) {
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            *reinterpret_cast<double2*>(dst + cc * V + o) = make_double2(y[cc][0], y[cc][1]);
        } else {
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) dst[cc * V + o] = y[cc][0];
        }
      }
    }
    w = wn;
    d = dn;
  }
  cp_async_wait<0>();
}

// Plane passes for extents up to 72: a CTA holds the F_x / F_y of one (component, ex, ey)
// combination and LPG groups of 4 warps; each group transforms one plane at a time in its own
// buffer (the step-1 result overwrites the plane in place, rows split over the group's warps),
// with named barriers inside the group only, so the groups overlap each other's loads.
constexpr int LPG = 3;                     // warp groups per CTA
constexpr int kPlaneLargeSmem = (2 * LMAT + LPG * LMAT) * (int)sizeof(double);

struct LargePlaneCta {   // one CTA's work: items [beg, end) of one (component, ex, ey) combination
  int beg, end, c, ex, ey, pad;
  int64_t fx, fy;        // forward factors along x and y (offsets into the factor buffer)
};

struct LargePlaneArgs {
  const fmp_subdomain* subs;
  const LargePlaneCta* ctas;
  const int2* items;     // (sub, plane): forward planes k < ez, inverse planes k < wz (owned)
  Geo g;
  const double* src;
  double* dst;
  const double* factors;
  int mode;
  int tma_rows;          // > 0: forward planes inside the block arrive as one TMA box of LSM x tma_rows
};

__device__ __forceinline__ void group_sync(int gi) {
  asm volatile("bar.sync %0, 128;\n" ::"r"(gi + 1) : "memory");
}

// acc[r][n] += X(row tile rows[r]) * B(col tile n), NR row tiles x NN column tiles of 8, K = 4 k4
//   A(m, k) = Xa[(8 rows[r] + g) * sa + 4 kk + t]          (row-major operand, lda = sa)
//   B(k, n) = INV-style or forward-style addressing through (bk, bn) strides
template <int NR, int NN>
__device__ __forceinline__ void lmma(double (&acc)[NR][NN][2], const double* a0, int sa, const double* b0, int bsk,
                                     int bsn, int k4, const int (&rows)[NR]) {
  for (int kk = 0; kk < k4; ++kk) {
    double av[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) av[r] = a0[rows[r] * 8 * sa + kk * 4];
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      const double bv = b0[kk * 4 * bsk + n * 8 * bsn];
#pragma unroll
      for (int r = 0; r < NR; ++r) dmma884(acc[r][n][0], acc[r][n][1], av[r], bv);
    }
  }
}

// Steps 1 and 2 of one plane of k_plane_large (group barrier between them).  FULL: 9 output
// tiles per axis (forward, and inverse when the owned tile is wider than 64); else 8.
template <bool INV, bool FULL>
__device__ __forceinline__ void plane_large_steps(double* X, const double* Fx, const double* Fy, const SubD& d,
                                                  const LargePlaneArgs& A, int2 w, int c, int ex, int ey, int k41,
                                                  int k42, int shift, int role, int gi, int g, int t) {
    // ---- step 1: T[r][a] = sum_i X[r][i] Fx[a][i]  (INV: T[b][i'] = sum_a X[b][a] Fx[a][ox + i'])
    // row tiles of this warp: role, role + 4 (+ 8 for role 0); 9 column tiles (INV: 8, owned)
    {
      const double* xa = X + g * LSM + t + shift;
      const double* fb = INV ? Fx + t * LSM + g + d.ox : Fx + g * LSM + t;
      const int bsk = INV ? LSM : 1, bsn = INV ? 1 : LSM;
      constexpr int NN = FULL ? 9 : 8;   // INV: only the owned columns (8 tiles when wx <= 64)
      if (role == 0) {
        double acc[3][NN][2] = {};
        const int rows[3] = {0, 4, 8};
        lmma<3, NN>(acc, xa, LSM, fb, bsk, bsn, k41, rows);
        __syncwarp();   // this warp's X rows are consumed: overwrite them with T
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          double* tr = X + (rows[r] * 8 + g) * LSM + 2 * t;
#pragma unroll
          for (int n = 0; n < NN; ++n) *reinterpret_cast<double2*>(tr + n * 8) = make_double2(acc[r][n][0], acc[r][n][1]);
        }
      } else {
        double acc[2][NN][2] = {};
        const int rows[2] = {role, role + 4};
        lmma<2, NN>(acc, xa, LSM, fb, bsk, bsn, k41, rows);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          double* tr = X + (rows[r] * 8 + g) * LSM + 2 * t;
#pragma unroll
          for (int n = 0; n < NN; ++n) *reinterpret_cast<double2*>(tr + n * 8) = make_double2(acc[r][n][0], acc[r][n][1]);
        }
      }
    }
    // the shifted forward plane: T starts at column 0 (written above); rows keep their index
    group_sync(gi);
    // ---- step 2: O[b][a] = sum_j Fy[b][j] T[j][a]  (INV: O[j'][i'] = sum_b Fy[b][oy + j'] T[b][i'])
    // column tiles of this warp: role, role + 4 (+ 8 for role 0); 9 row tiles (INV: 8, owned)
    {
      const double* fa = INV ? Fy + t * LSM + g + d.oy : Fy + g * LSM + t;   // A(m, k) = Fy-based
      const int ask = INV ? LSM : 1, asm_ = INV ? 1 : LSM;
      const int64_t obase = INV ? 0 : d.ws_off + (int64_t)(c * d.ez + w.y) * d.ps;
      auto run = [&](auto ncols) {
        constexpr int NC = decltype(ncols)::value;
        int cols[NC];
        cols[0] = role;
        cols[1] = role + 4;
        if (NC == 3) cols[NC - 1] = 8;
        double acc[9][NC][2] = {};
        const double* tb = X + t * LSM + g;
        for (int kk = 0; kk < k42; ++kk) {
          double bv[NC];
#pragma unroll
          for (int q = 0; q < NC; ++q) bv[q] = tb[kk * 4 * LSM + cols[q] * 8];
#pragma unroll
          for (int m = 0; m < 9; ++m) {
            if (!FULL && m == 8) break;
            const double av = fa[kk * 4 * ask + m * 8 * asm_];
#pragma unroll
            for (int q = 0; q < NC; ++q) dmma884(acc[m][q][0], acc[m][q][1], av, bv[q]);
          }
        }
#pragma unroll
        for (int m = 0; m < 9; ++m) {
          if (!FULL && m == 8) break;
          const int row = m * 8 + g;
          if (!INV && row >= ey) continue;
          if (INV && row >= d.wy) continue;
#pragma unroll
          for (int q = 0; q < NC; ++q) {
            const int col = cols[q] * 8 + 2 * t;
            if (!INV) {
              double* o = A.dst + obase + row * ex + col;
              if ((ex & 1) == 0 && col + 1 < ex) {
                *reinterpret_cast<double2*>(o) = make_double2(acc[m][q][0], acc[m][q][1]);
              } else {
                if (col < ex) o[0] = acc[m][q][0];
                if (col + 1 < ex) o[1] = acc[m][q][1];
              }
            } else if (col < d.wx) {
              double* o = A.dst + fidx(A.g, c, d.lz + d.oz + w.y, d.ly + d.oy + row, d.lx + d.ox + col);
              if (col + 1 < d.wx && (((uintptr_t)o) & 15) == 0) {
                *reinterpret_cast<double2*>(o) = make_double2(acc[m][q][0], acc[m][q][1]);
              } else {
                o[0] = acc[m][q][0];
                if (col + 1 < d.wx) o[1] = acc[m][q][1];
              }
            }
          }
        }
      };
      if (role == 0 && FULL)
        run(std::integral_constant<int, 3>{});
      else
        run(std::integral_constant<int, 2>{});
    }
}

template <bool INV>
__global__ void __launch_bounds__(LPG * 128, 1) k_plane_large(const __grid_constant__ CUtensorMap tm, LargePlaneArgs A) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t pbar[LPG];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int gi = warp >> 2, wq = warp & 3;
  // rotated row-tile role inside the group: the heavy role (3 tiles) lands on a different SM
  // sub-partition in each group
  const int role = (wq + gi) & 3;
  const LargePlaneCta cw = A.ctas[blockIdx.x];
  double* Fx = smem;
  double* Fy = smem + LMAT;
  double* X = smem + (2 + gi) * LMAT;
  const int ex = cw.ex, ey = cw.ey;
  for (int q = tid; q < LMAT; q += blockDim.x) {
    const int r = q / LSM, c = q - r * LSM;
    Fx[q] = (r < ex && c < ex) ? __ldg(A.factors + cw.fx + r * ex + c) : 0.0;
    Fy[q] = (r < ey && c < ey) ? __ldg(A.factors + cw.fy + r * ey + c) : 0.0;
  }
  for (int q = tid; q < LPG * LMAT; q += blockDim.x) smem[2 * LMAT + q] = 0.0;
  if (tid == 0) {
    for (int q = 0; q < LPG; ++q) mbar_init(&pbar[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int c = cw.c;
  uint32_t tphase = 0;
  const int k41 = pad4(ex) / 4, k42 = pad4(ey) / 4;
  for (int it = cw.beg + gi; it < cw.end; it += LPG) {
    const int2 w = A.items[it];
    const SubD d = load_sub(A.subs + w.x);
    // ---- load the plane (rows at stride LSM): TMA box (forward, inside the block) or cp.async
    int shift = 0;
    const bool inside = d.lx >= 0 && d.ly >= 0 && d.lz >= 0 && d.lx + ex <= A.g.bx && d.ly + ey <= A.g.by &&
                        d.lz + d.ez <= A.g.bz;
    if (!INV && A.mode != FMP_SOLVE_FACES && inside && A.tma_rows > 0) {
      shift = d.lx & 1;   // the box starts at an even x (16-byte aligned inner coordinate)
      if (wq == 0 && lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(&pbar[gi], (uint32_t)(LSM * A.tma_rows * 8));
        tma_load_4d(X, &tm, d.lx & ~1, d.ly, d.lz + w.y, c, &pbar[gi]);
      }
      mbar_wait(&pbar[gi], tphase);
      tphase ^= 1u;
    } else {
      const int64_t P = (int64_t)ex * ey;
      for (int j = wq; j < ey; j += 4) {
        for (int i = lane; i < ex; i += 32) {
          const double* sp;
          if (INV)
            sp = A.src + d.ws_off + (int64_t)(c * d.ez + d.oz + w.y) * d.ps + j * ex + i;
          else if (A.mode == FMP_SOLVE_FACES)
            sp = A.src + d.in_off + c * P * d.ez + w.y * P + j * ex + i;
          else
            sp = point_ptr(A.g, A.src, c, d.lz + w.y, d.ly + j, d.lx + i);
          cp_async8(X + j * LSM + i, sp, A.factors);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
    }
    group_sync(gi);
    if (!INV || d.wx > 64 || d.wy > 64)
      plane_large_steps<INV, true>(X, Fx, Fy, d, A, w, c, ex, ey, k41, k42, shift, role, gi, g, t);
    else
      plane_large_steps<INV, false>(X, Fx, Fy, d, A, w, c, ex, ey, k41, k42, shift, role, gi, g, t);
    group_sync(gi);   // the buffer is free for the group's next plane
  }
}

// ---------------------------------------------------------------- K5 / K6: boundary faces
// Component c has two boundary faces with nonzero delta (ref:operators.py:151-164):
//   c = x: z-normal (k = 0, all j,i) and y-normal (j = 0, k >= 1)
//   c = y: z-normal (k = 0, all j,i) and x-normal (i = 0, k >= 1)
//   c = z: y-normal (j = 0, all k,i) and x-normal (i = 0, j >= 1)
// Rows of the correction (ref:subdomain.py:183-194) are component-major and ascending in
// the linear index; the helpers below map face-plane coordinates to that row.
struct FaceGeo {
  int n1, n2;          // normal axes of the primary / secondary face
  int u1, v1, u2, v2;  // in-plane axes (slow, fast) for each face
};
__device__ __forceinline__ FaceGeo face_geo(int c) {
  FaceGeo f;
  if (c == 0) { f.n1 = 2; f.u1 = 1; f.v1 = 0; f.n2 = 1; f.u2 = 2; f.v2 = 0; }
  else if (c == 1) { f.n1 = 2; f.u1 = 1; f.v1 = 0; f.n2 = 0; f.u2 = 2; f.v2 = 1; }
  else { f.n1 = 1; f.u1 = 2; f.v1 = 0; f.n2 = 0; f.u2 = 2; f.v2 = 1; }
  return f;
}
// row (within the component) of the physical face point (u, v) of face f (0 primary, 1 secondary);
// returns -1 for the excluded edge line of the secondary face.
__device__ __forceinline__ int face_row(int c, int f, int u, int v, int ex, int ey) {
  if (c == 0) return f == 0 ? u * ex + v : (u == 0 ? -1 : ex * ey + (u - 1) * ex + v);
  if (c == 1) return f == 0 ? u * ex + v : (u == 0 ? -1 : ex * ey + (u - 1) * ey + v);
  return f == 0 ? u * (ex + ey - 1) + v : (v == 0 ? -1 : u * (ex + ey - 1) + ex + v - 1);
}

struct FaceArgs {
  const fmp_subdomain* subs;
  const fmp_shape* shapes;
  const double* factors;
  const double* yhat;          // K5 input
  double* corr;                // K6 output
  double* const* ymat;         // device array of per-shape Y pointers (K5 out)
  const double* const* zmat;   // device array of per-shape Z pointers (K6 in)
  int pmax;
  int max_ps;                  // largest padded plane stride of the plan
  const int* rowmap;           // shape row -> group row maps (fmp_shape::rowmap_off), may be null
  const double* facepad;       // per distinct extent n: [U^T_n, V^T_n] zero-padded to FaceMat<NT> (N x S)
  unsigned char pad_slot[80];  // extent n -> its slot in facepad
  int bulk_factors;            // 1: k_faces loads the transform factors with bulk copies
};

__device__ __forceinline__ int ext_of(const SubD& d, int a) { return a == 0 ? d.ex : (a == 1 ? d.ey : d.ez); }

// Small dense products of the face kernels on the FP64 tensor cores: C = op(A) op(B) for
// zero-padded NT*8 x NT*8 matrices in shared memory (row stride NT*8+4, == 4 mod 8: the
// fragment loads are bank-conflict free in either orientation); warps take 8x8 output tiles.
template <int NT>
struct FaceMat {
  static constexpr int N = NT * 8, S = N + 4, WORDS = N * S;
};
template <int NT, bool TA, bool TB>
__device__ __forceinline__ void face_mm(const double* A, const double* B, double* C, int warp, int nwarps,
                                        int lane) {
  constexpr int S = FaceMat<NT>::S;
  const int g = lane >> 2, t = lane & 3;
  for (int tile = warp; tile < NT * NT; tile += nwarps) {
    const int m0 = (tile / NT) * 8, n0 = (tile % NT) * 8;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int k = 0; k < NT * 8; k += 4) {
      const double a = TA ? A[(k + t) * S + m0 + g] : A[(m0 + g) * S + k + t];
      const double b = TB ? B[(n0 + g) * S + k + t] : B[(k + t) * S + n0 + g];
      dmma884(d0, d1, a, b);
    }
    C[(m0 + g) * S + n0 + 2 * t] = d0;
    C[(m0 + g) * S + n0 + 2 * t + 1] = d1;
  }
}
// the zero-padded N x S copy of the forward factor of component c on axis a (extent n): one
// 16-byte vectorised copy of the plan's pre-padded matrix (no per-element index arithmetic)
template <int NT>
__device__ __forceinline__ void face_load_factor(double* M, const FaceArgs& A, int c, int a, int n, int tid, int nth) {
  constexpr int W2 = FaceMat<NT>::WORDS / 2;
  const double2* f = reinterpret_cast<const double2*>(A.facepad + (size_t)(2 * A.pad_slot[n] + (a == c ? 0 : 1)) * FaceMat<NT>::WORDS);
  double2* m2 = reinterpret_cast<double2*>(M);
  for (int q = tid; q < W2; q += nth) m2[q] = __ldg(f + q);
}

// K5: Y[:, col] = e0 on the two faces per component, e0 = G^-1 y^ evaluated only there.
// Projection along the face normal with weights F_n[t][0] (inverse factor row 0), then
// a 2-D inverse transform over the in-plane axes (two DMMA products).  One CTA per
// (component, subdomain).  A producer warp streams the component's y^ planes (contiguous,
// 32-byte padded) into a shared-memory ring with one cp.async.bulk each (full/empty
// mbarriers); consumer warp w owns the rows b = w, w+8, ... of every plane and lane l the
// columns a = l, l+32, l+64, so no projection needs a CTA barrier per plane:
//   z-normal [b][a] = sum_z w_z[z] y^[z][b][a]   accumulated in place in shared memory
//                                                (every element owned by one thread);
//   x-normal [z][b] = sum_a w_x[a] y^[z][b][a]   a warp-shuffle reduction per row;
//   y-normal [z][a] = sum_b w_y[b] y^[z][b][a]   per-warp partials over the warp's rows,
//                                                summed over warps in a fixed order once per
//                                                chunk of FZ planes (consumer-only barrier).
constexpr int FACE_WARPS = 8;                       // consumer warps
constexpr int FACE_THREADS = (FACE_WARPS + 1) * 32; // + producer warp
constexpr int FZ = 4;                               // planes per y-normal partial chunk
template <int NT>
struct FaceRing {
  static constexpr int NS = NT <= 5 ? 3 : 2;   // ring slots (3: three CTAs per SM at 34^3 planes)
};
// ring slot (doubles): the plan's largest padded plane, rounded to 128 bytes
__host__ __device__ inline int face_slot(int max_ps) { return (max_ps + 15) / 16 * 16; }
// work region: max(Fu, Fv, temp) during the transforms vs ring + weights + partials
template <int NT>
inline size_t face_smem_bytes(int slot) {
  const size_t stream = (size_t)FaceRing<NT>::NS * slot + 3 * FaceMat<NT>::N + FACE_WARPS * FZ * FaceMat<NT>::N;
  const size_t work = std::max<size_t>(stream, 3 * (size_t)FaceMat<NT>::WORDS);
  return (2 * (size_t)FaceMat<NT>::WORDS + work) * sizeof(double);
}

// One staged y^ plane of the face projections (consumer warp `warp` of FACE_WARPS): all row
// loads first, then the z-normal update, the y-normal partial and the x-normal row sums with
// the FR shuffle reductions interleaved (independent chains, no early exit).
template <int FR, int FA, int S>
__device__ __forceinline__ void face_plane(const double* pl, int z, int rowstep, bool zn, bool xn,
                                           double wz, const double* Wy, const double (&wx)[FA],
                                           double (&za)[FR][FA], double* sB, double (&yp)[FA], int ey, int warp,
                                           int lane) {
  // pl points at this thread's first point (row warp, column lane).  Points outside the plane
  // (b >= ey or a >= ex) are loaded unpredicated: they read other rows, the zeroed slot tail, the
  // next slot or the zeroed weights / partials -- always finite -- and meet zero weights (x, y
  // normals) or are never written out (z normal), so no per-point predicate is needed
  double val[FR][FA];
#pragma unroll
  for (int r = 0; r < FR; ++r)
#pragma unroll
    for (int h = 0; h < FA; ++h) val[r][h] = pl[r * rowstep + 32 * h];
  if (zn) {   // z-normal: this thread's (b, a) accumulators live in registers
#pragma unroll
    for (int r = 0; r < FR; ++r)
#pragma unroll
      for (int h = 0; h < FA; ++h) za[r][h] += wz * val[r][h];
  }
#pragma unroll
  for (int h = 0; h < FA; ++h) yp[h] = 0.0;
#pragma unroll
  for (int r = 0; r < FR; ++r) {
    const double wy = Wy[warp + FACE_WARPS * r];   // zero-padded past ey
#pragma unroll
    for (int h = 0; h < FA; ++h) yp[h] += wy * val[r][h];
  }
  if (xn) {
    double xs[FR];
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      xs[r] = 0.0;
#pragma unroll
      for (int h = 0; h < FA; ++h) xs[r] += wx[h] * val[r][h];
    }
    if (FR <= 8) {
      // transpose-reduce of up to 8 row sums over the 32 lanes: each exchange halves the values a
      // lane carries (4 + 2 + 1 + 1 + 1 shuffles instead of 5 per row)
      double v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = r < FR ? xs[r] : 0.0;
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double send = b4 ? v[i] : v[i + 4], keep = b4 ? v[i + 4] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double send = b3 ? v[i] : v[i + 2], keep = b3 ? v[i + 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
      {
        const double send = b2 ? v[0] : v[1], keep = b2 ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
      const int r = (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0), b = warp + FACE_WARPS * r;
      if ((lane & 3) == 0 && r < FR && b < ey) sB[z * S + b] = v[0];
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < FR; ++r) xs[r] += __shfl_xor_sync(0xffffffffu, xs[r], o);
#pragma unroll
      for (int r = 0; r < FR; ++r) {
        const int b = warp + FACE_WARPS * r;
        if (lane == r && b < ey) sB[z * S + b] = xs[r];
      }
    }
  }
}

// FR rows per warp, FA columns per lane, NT 8-wide tiles per padded extent (register and
// shared-memory footprints sized for the plan's extents)
template <int FR, int FA, int NT>
__global__ void __launch_bounds__(FACE_THREADS, NT <= 3 ? 4 : (NT <= 5 ? 3 : 1)) k_faces(FaceArgs A) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[FaceRing<NT>::NS], empty[FaceRing<NT>::NS], fbar;
  constexpr int S = FaceMat<NT>::S, W = FaceMat<NT>::WORDS, N = FaceMat<NT>::N;
  constexpr int NS = FaceRing<NT>::NS;
  const int SLOT = face_slot(A.max_ps);
  const SubD d = load_sub(A.subs + blockIdx.y);
  const fmp_shape& sh = A.shapes[d.shape];
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ex = d.ex, ey = d.ey, ez = d.ez;
  const int ext[3] = {ex, ey, ez};
  double* sA = smem;                 // primary projection   [u1][v1]
  double* sB = sA + W;               // secondary projection [u2][v2]
  double* sX = sB + W;               // streaming: ring, weights, partials; transforms: Fu, Fv, temp
  double* ring = sX;
  double* sWt = ring + NS * SLOT;    // weights F_n[t][0] of axis n at sWt[n * N + t]
  double* sP = sWt + 3 * N;          // y-normal partials [warp][FZ][N]
  const double* src = A.yhat + d.ws_off + (int64_t)c * d.cstride();
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], FACE_WARPS);
    }
    mbar_init(&fbar, 1);
    fence_mbar_init();
  }
  // ring, weights and partials zeroed before the first bulk copy: the consumers' unpredicated
  // loads of points outside a plane may reach past its slot (face_plane)
  for (int q = tid; q < NS * SLOT + 3 * N + FACE_WARPS * FZ * N; q += FACE_THREADS) ring[q] = 0.0;
  fence_proxy_async();   // these generic writes precede the async-proxy fills of the ring
  pdl_trigger();
  pdl_wait();   // y^ is the forward column pass's output
  const FaceGeo fg = face_geo(c);
  const bool zn = fg.n1 == 2, yn = fg.n1 == 1 || fg.n2 == 1, xn = fg.n2 == 0;
  double* sY = fg.n1 == 1 ? sA : sB;   // y-normal destination [z][a]
  __syncthreads();   // barriers initialised: the producer streams while the consumers set up
  if (warp != FACE_WARPS) {
    constexpr int CT = FACE_WARPS * 32;
    for (int q = tid; q < 3 * N; q += CT) {
      const int n = q / N, t = q - n * N;
      sWt[q] = t < ext[n] ? __ldg(fwd_factor(A.factors, sh, c, n) + t * ext[n]) : 0.0;
    }
    for (int q = tid; q < 2 * W; q += CT) sA[q] = 0.0;   // sA, sB: zero padding
    asm volatile("bar.sync 1, %0;\n" ::"n"(CT) : "memory");
  }
  if (warp == FACE_WARPS) {
    // ---------------- producer: one bulk copy per z-plane
    if (lane == 0)
      for (int z = 0; z < ez; ++z) {
        const int slot = z % NS;
        if (z >= NS) mbar_wait(&empty[slot], (uint32_t)(((z / NS) - 1) & 1));
        mbar_expect_tx(&full[slot], (uint32_t)d.ps * 8);
        bulk_g2s(ring + slot * SLOT, src + (int64_t)z * d.ps, (uint32_t)d.ps * 8, &full[slot]);
      }
  } else {
    // ---------------- consumers
    const double* Wz = sWt + 2 * N;
    const double* Wy = sWt + N;
    // plane-invariant per-thread state, computed once: which of this thread's points lie in the
    // plane (bit mask, for the z-normal write-out), its first point's offset and the row step
    double wx[FA], za[FR][FA];
    uint32_t vmask = 0;
#pragma unroll
    for (int h = 0; h < FA; ++h) wx[h] = lane + 32 * h < N ? sWt[lane + 32 * h] : 0.0;
#pragma unroll
    for (int r = 0; r < FR; ++r)
#pragma unroll
      for (int h = 0; h < FA; ++h) {
        const int b = warp + FACE_WARPS * r, a = lane + 32 * h;
        if (b < ey && a < ex) vmask |= 1u << (r * FA + h);
        za[r][h] = 0.0;
      }
    const int first = warp * ex + lane, rowstep = FACE_WARPS * ex;
    int slot = 0;
    uint32_t ph = 0;
    for (int z0 = 0; z0 < ez; z0 += FZ) {
      const int nzc = min(FZ, ez - z0);
      for (int zz = 0; zz < nzc; ++zz) {
        const int z = z0 + zz;
        mbar_wait(&full[slot], ph);
        const double* pl = ring + slot * SLOT + first;
        double yp[FA];
        face_plane<FR, FA, S>(pl, z, rowstep, zn, xn, Wz[z], Wy, wx, za, sB, yp, ey, warp, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == NS) {
          slot = 0;
          ph ^= 1u;
        }
        if (yn) {
#pragma unroll
          for (int h = 0; h < FA; ++h)
            if (lane + 32 * h < ex) sP[(warp * FZ + zz) * N + lane + 32 * h] = yp[h];
        }
      }
      if (yn) {
        asm volatile("bar.sync 1, %0;\n" ::"n"(FACE_WARPS * 32) : "memory");
        for (int q = tid; q < nzc * ex; q += FACE_WARPS * 32) {
          const int zz = q / ex, a = q - zz * ex;
          double acc = 0.0;
          for (int w = 0; w < FACE_WARPS; ++w) acc += sP[(w * FZ + zz) * N + a];
          sY[(z0 + zz) * S + a] = acc;
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(FACE_WARPS * 32) : "memory");
      }
    }
    if (zn) {   // z-normal projection [b][a] from the register accumulators
#pragma unroll
      for (int r = 0; r < FR; ++r)
#pragma unroll
        for (int h = 0; h < FA; ++h) {
          const int b = warp + FACE_WARPS * r, a = lane + 32 * h;
          if (b < ey && a < ex) sA[b * S + a] = za[r][h];
        }
    }
  }
  __syncthreads();
  // 2-D inverse transforms: E[u][v] = sum_tu Fu[tu][u] sum_tv Fv[tv][v] Proj[tu][tv]
  double* Y = A.ymat[d.shape] + (int64_t)d.column * sh.ld;
  const int* rm = sh.rowmap_off >= 0 ? A.rowmap + sh.rowmap_off : nullptr;
  int base = 0;
  for (int q = 0; q < c; ++q) base += (int)sh.m_comp[q];
  for (int f = 0; f < 2; ++f) {
    const int ua = f == 0 ? fg.u1 : fg.u2, va = f == 0 ? fg.v1 : fg.v2;
    const int nu = ext[ua], nv_ = ext[va];
    double *sFu = sX, *sFv = sX + W, *sT = sX + 2 * W;
    // the two padded factor matrices as two bulk copies (one round trip); face 1's are issued as
    // soon as face 0's products are done, under its write-out
    auto issue_factors = [&](int ff) {
      const int fu = ff == 0 ? fg.u1 : fg.u2, fv = ff == 0 ? fg.v1 : fg.v2;
      fence_proxy_async();   // the generic accesses of this region precede the async fill
      mbar_expect_tx(&fbar, 2u * W * (uint32_t)sizeof(double));
      bulk_g2s(sFu, A.facepad + (size_t)(2 * A.pad_slot[ext[fu]] + (fu == c ? 0 : 1)) * W, W * sizeof(double), &fbar);
      bulk_g2s(sFv, A.facepad + (size_t)(2 * A.pad_slot[ext[fv]] + (fv == c ? 0 : 1)) * W, W * sizeof(double), &fbar);
    };
    if (A.bulk_factors) {
      if (f == 0 && tid == 0) issue_factors(0);
      mbar_wait(&fbar, (uint32_t)f);
    } else {
      face_load_factor<NT>(sFu, A, c, ua, nu, tid, FACE_THREADS);
      face_load_factor<NT>(sFv, A, c, va, nv_, tid, FACE_THREADS);
    }
    __syncthreads();
    face_mm<NT, false, false>(f == 0 ? sA : sB, sFv, sT, warp, FACE_THREADS / 32, lane);   // T = Proj Fv
    __syncthreads();
    double* E = f == 0 ? sA : sB;                                                  // E = Fu^T T
    face_mm<NT, true, false>(sFu, sT, E, warp, FACE_THREADS / 32, lane);
    __syncthreads();
    if (A.bulk_factors && f == 0 && tid == 0) issue_factors(1);
    if (rm) {   // every row-map read of this thread first, then the stores (one round trip)
      constexpr int GQ = (N * N + FACE_THREADS - 1) / FACE_THREADS;
      int yi[GQ];
#pragma unroll
      for (int i = 0; i < GQ; ++i) {
        const int q = tid + i * FACE_THREADS, u = q / nv_, vv = q - u * nv_;
        const int row = q < nu * nv_ ? face_row(c, f, u, vv, ex, ey) : -1;
        yi[i] = row < 0 ? -1 : rm[base + row];
      }
#pragma unroll
      for (int i = 0; i < GQ; ++i) {
        const int q = tid + i * FACE_THREADS, u = q / nv_, vv = q - u * nv_;
        if (yi[i] >= 0) Y[yi[i]] = E[u * S + vv];
      }
    } else {
      for (int q = tid; q < nu * nv_; q += FACE_THREADS) {
        const int u = q / nv_, vv = q - u * nv_;
        const int row = face_row(c, f, u, vv, ex, ey);
        if (row >= 0) Y[base + row] = E[u * S + vv];
      }
    }
    __syncthreads();
  }
}

// K6: from Z (C^-1 Y) build, per component and face, the forward-transformed face plane
// Proj[tu][tv] = sum_{u,v} Fu[tu][u] Fv[tv][v] Zface[u][v]  -> corr planes (see K3);
// the two products on DMMA.
template <int NT>
__global__ void __launch_bounds__(FACE_THREADS) k_corr(FaceArgs A) {
  extern __shared__ __align__(16) double smem[];
  constexpr int S = FaceMat<NT>::S, W = FaceMat<NT>::WORDS;
  const SubD d = load_sub(A.subs + blockIdx.y);
  const fmp_shape& sh = A.shapes[d.shape];
  // one CTA per (component, face, subdomain): blockIdx.x = 2 c + f
  const int c = blockIdx.x >> 1, f = blockIdx.x & 1, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ex = d.ex, ey = d.ey, ez = d.ez;
  const int ext[3] = {ex, ey, ez};
  const int pm = A.pmax;
  double* sFu = smem;     // padded factors of the face's in-plane axes
  double* sFv = sFu + W;
  double* sZ = sFv + W;   // face values of Z, then the result
  double* sT = sZ + W;
  double* sO = sZ;
  const FaceGeo fg = face_geo(c);
  const double* Z = A.zmat[d.shape] + (int64_t)d.column * sh.ld;
  const int* rm = sh.rowmap_off >= 0 ? A.rowmap + sh.rowmap_off : nullptr;
  pdl_trigger();
  int base = 0;
  for (int q = 0; q < c; ++q) base += (int)sh.m_comp[q];
  {
    const int ua = f == 0 ? fg.u1 : fg.u2, va = f == 0 ? fg.v1 : fg.v2;
    const int nu = ext[ua], nv = ext[va];
    if (A.bulk_factors) {   // both factors by bulk copy, in flight during the Z gather below
      __shared__ __align__(8) uint64_t fbar;
      if (tid == 0) {
        mbar_init(&fbar, 1);
        fence_mbar_init();
        mbar_expect_tx(&fbar, 2u * W * (uint32_t)sizeof(double));
        bulk_g2s(sFu, A.facepad + (size_t)(2 * A.pad_slot[nu] + (ua == c ? 0 : 1)) * W, W * sizeof(double), &fbar);
        bulk_g2s(sFv, A.facepad + (size_t)(2 * A.pad_slot[nv] + (va == c ? 0 : 1)) * W, W * sizeof(double), &fbar);
      }
      // the face's Z values: every row-map read of this thread first, then every Z read (two
      // round trips in all instead of two per element)
      constexpr int GQ = (W + FACE_THREADS - 1) / FACE_THREADS;
      int zi[GQ];
#pragma unroll
      for (int i = 0; i < GQ; ++i) {
        const int q = tid + i * FACE_THREADS, u = q / S, v = q - u * S;
        const int row = (q < W && u < nu && v < nv) ? face_row(c, f, u, v, ex, ey) : -1;
        zi[i] = row < 0 ? -1 : (rm ? rm[base + row] : base + row);
      }
      pdl_wait();   // factors and row map are constant; Z is the GEMM's output
      double zv[GQ];
#pragma unroll
      for (int i = 0; i < GQ; ++i) zv[i] = zi[i] < 0 ? 0.0 : Z[zi[i]];
#pragma unroll
      for (int i = 0; i < GQ; ++i)
        if (tid + i * FACE_THREADS < W) sZ[tid + i * FACE_THREADS] = zv[i];
      __syncthreads();   // fbar's initialisation is visible before anyone waits on it
      mbar_wait(&fbar, 0);
    } else {
      pdl_wait();
      face_load_factor<NT>(sFu, A, c, ua, nu, tid, FACE_THREADS);
      face_load_factor<NT>(sFv, A, c, va, nv, tid, FACE_THREADS);
      for (int q = tid; q < W; q += FACE_THREADS) {
        const int u = q / S, v = q - u * S;
        const int row = (u < nu && v < nv) ? face_row(c, f, u, v, ex, ey) : -1;
        sZ[q] = row < 0 ? 0.0 : Z[rm ? rm[base + row] : base + row];
      }
    }
    __syncthreads();
    face_mm<NT, false, true>(sZ, sFv, sT, warp, FACE_THREADS / 32, lane);    // T[u][tv] = sum_v Z[u][v] Fv[tv][v]
    __syncthreads();
    face_mm<NT, false, false>(sFu, sT, sO, warp, FACE_THREADS / 32, lane);   // Proj = Fu T
    __syncthreads();
    double* out = A.corr + ((int64_t)blockIdx.y * 6 + c * 2 + f) * pm * pm;
    for (int q = tid; q < nu * nv; q += FACE_THREADS) {
      const int tu = q / nv, tv = q - tu * nv;
      out[tu * pm + tv] = sO[tu * S + tv];
    }
  }
}

// Padded forward factors for the face kernels: slot e holds [U^T_n, V^T_n] of extent n as
// zero-padded N x S matrices (N = 8 NT, S = N + 4), built once per plan.
__global__ void k_pad_factors(const double* __restrict__ factors, const int64_t* __restrict__ src_off,
                              const int* __restrict__ ext, int nmat, int N, int S, double* __restrict__ out) {
  const int mat = blockIdx.y, n = ext[mat];
  if (mat >= nmat) return;
  const double* f = factors + src_off[mat];
  double* o = out + (size_t)mat * N * S;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < N * S; q += gridDim.x * blockDim.x) {
    const int r = q / S, cc = q - r * S;
    o[q] = (r < n && cc < n) ? f[r * n + cc] : 0.0;
  }
}

}  // namespace fmp

using namespace fmp;

struct fmp_precond {
  fmp_precond_desc d;
  std::vector<fmp_subdomain> subs;
  std::vector<fmp_shape> shapes;
  std::vector<int64_t> first;
  std::vector<const double*> cinv;
  std::vector<double*> ymat, zmat;
  double** d_ymat = nullptr;  // device copies of the pointer tables
  double** d_zmat = nullptr;
  int4* d_fwd_items = nullptr;   // K1 work items
  int4* d_inv_items = nullptr;   // K4 work items
  int2* d_col_items = nullptr;   // K2/K3 work items
  int n_fwd = 0, n_inv = 0, n_col = 0;
  // fast path (all extents <= FAST_MAX_EXT, at most FX_MAXE distinct): warp-independent kernels
  bool fast = false;
  ExtTable et{};
  int4* d_ffwd = nullptr;
  int4* d_finv = nullptr;
  int2* d_fcol = nullptr;
  int n_ffwd = 0, n_finv = 0, n_fcol = 0;
  int n_ffwd_int = 0;                     // forward plane items of subdomains that read no ghost (listed first)
  CUtensorMap* d_colmaps = nullptr;       // column tiles by TMA: [work_a maps | work_b maps], one per subdomain
  // large path (extents 41..72): column items grouped by z extent (one launch per group, its z
  // factors resident), column tile maps with 72-row boxes
  struct LColGroup { int ez, off, n, mt_fwd, mt_inv; int64_t ut, vt; };
  bool large = false;
  std::vector<LColGroup> lcol;
  int2* d_lcol = nullptr;
  CUtensorMap* d_lcolmaps = nullptr;
  // large plane passes: per-CTA (combination, item range) tables, forward and inverse
  LargePlaneCta* d_lpc[2] = {nullptr, nullptr};
  int2* d_lpi[2] = {nullptr, nullptr};
  int n_lpc[2] = {0, 0};
  // Woodbury GEMM (set at plan creation from FMP_GEMM): Ozaki INT8 tensor-core GEMM (default,
  // "ozaki": int8 slices of C^-1 built once, Y sliced per apply), the own DMMA kernel ("own") or
  // cuBLAS DGEMM ("cublas")
  bool use_cublas = false;
  bool use_ozaki = true;
  std::vector<int8_t*> oz_a, oz_b;
  std::vector<int*> oz_ea, oz_eb, oz_perm;
  double* facepad = nullptr;            // padded forward factors of the face kernels (k_pad_factors)
  unsigned char pad_slot[80] = {};
  OzPlan oz;                              // work items, schedule and split-K workspace
  OzSlice* d_ozslices = nullptr;          // per-apply slicing of Y, all shapes in two launches
  int n_ozslices = 0;
  int64_t oz_rows = 0, oz_threads = 0;
  static constexpr int kAux = 4;          // concurrent GEMM streams (small shapes are HBM-bound)
  cudaStream_t aux[kAux] = {};
  cublasHandle_t aux_blas[kAux] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kAux] = {};
  std::vector<int> gemm_order;            // canonical shapes by decreasing GEMM size
  std::vector<int> gcols;                 // Y/Z columns of each rotation group (0 for members)
  GemmShape* d_gshapes = nullptr;
  GemmTile* d_gtiles[3] = {nullptr, nullptr, nullptr};
  int n_gtiles[3] = {0, 0, 0};
  cublasHandle_t blas = nullptr;
  int max_ex = 1, max_ey = 1, max_ez = 1, max_p = 1;
  int sms = kNumSM;
  bool profile = false;                   // stage events (fmp_precond_profile)
  cudaEvent_t stage_ev[FMP_PRECOND_STAGES + 1] = {};
};

template <class T>
static int upload(const std::vector<T>& v, T** out) {
  *out = nullptr;
  if (v.empty()) return 0;
  FMP_CHECK_CUDA(cudaMalloc(out, sizeof(T) * v.size()));
  FMP_CHECK_CUDA(cudaMemcpy(*out, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return 0;
}

static void free_plan(fmp_precond* p) {
  for (auto& e : p->stage_ev)
    if (e) cudaEventDestroy(e);
  if (!p) return;
  if (p->blas) cublasDestroy(p->blas);
  cudaFree(p->d_ymat);
  cudaFree(p->d_zmat);
  cudaFree(p->d_fwd_items);
  cudaFree(p->d_inv_items);
  cudaFree(p->d_col_items);
  cudaFree(p->d_ffwd);
  cudaFree(p->d_finv);
  cudaFree(p->d_fcol);
  cudaFree(p->d_colmaps);
  cudaFree(p->d_lcol);
  cudaFree(p->d_lcolmaps);
  for (int q = 0; q < 2; ++q) {
    cudaFree(p->d_lpc[q]);
    cudaFree(p->d_lpi[q]);
  }
  cudaFree(p->d_gshapes);
  for (int q = 0; q < fmp_precond::kAux; ++q) {
    if (p->aux_blas[q]) cublasDestroy(p->aux_blas[q]);
    if (p->aux[q]) cudaStreamDestroy(p->aux[q]);
    if (p->ev_join[q]) cudaEventDestroy(p->ev_join[q]);
  }
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  for (auto* q : p->oz_a) cudaFree(q);
  for (auto* q : p->oz_b) cudaFree(q);
  for (auto* q : p->oz_ea) cudaFree(q);
  for (auto* q : p->oz_perm) cudaFree(q);
  cudaFree(p->facepad);
  for (auto* q : p->oz_eb) cudaFree(q);
  ozaki_free(&p->oz);
  cudaFree(p->d_ozslices);
  for (int c = 0; c < 3; ++c) cudaFree(p->d_gtiles[c]);
  delete p;
}

constexpr int kPlaneFastSmem = (RES_WORDS + PW_WARPS * PX_BUF + PX_SLACK) * (int)sizeof(double);
constexpr int kColFastSmem = (RES_WORDS + CW_WARPS * CX_BUF) * (int)sizeof(double);
constexpr int col_db_smem(int nw, int nb = 2) { return (RES_WORDS + nw * nb * CX_BUF) * (int)sizeof(double); }

static int plane_nt(const fmp_precond* p) { return std::max(p->max_ex, p->max_ey) <= 40 ? 5 : 9; }
static int column_mt(const fmp_precond* p) { return pad8(p->max_ez) / 8; }

template <bool INV, int NT>
static void plane_attr() {
  cudaFuncSetAttribute(k_plane<INV, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PlaneSmem<NT>::bytes);
}
template <int MT>
static void column_attr() {
  cudaFuncSetAttribute(k_column<MT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColSmem<MT>::bytes);
  cudaFuncSetAttribute(k_column<MT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColSmem<MT>::bytes);
}

extern "C" int fmp_precond_create(const fmp_precond_desc* desc, fmp_precond** out) {
  FMP_REQUIRE(desc && out, "null argument");
  FMP_REQUIRE(desc->n_sub >= 1 && desc->n_shape >= 1, "empty plan");
  auto* p = new fmp_precond();
  p->d = *desc;
  p->subs.assign(desc->subs_host, desc->subs_host + desc->n_sub);
  p->shapes.assign(desc->shapes_host, desc->shapes_host + desc->n_shape);
  p->first.assign(desc->shape_first, desc->shape_first + desc->n_shape + 1);
  p->cinv.assign(desc->cinv, desc->cinv + desc->n_shape);
  p->ymat.assign(desc->ymat, desc->ymat + desc->n_shape);
  p->zmat.assign(desc->zmat, desc->zmat + desc->n_shape);
  std::vector<int4> fwd, inv;
  std::vector<int2> col;
  for (int64_t q = 0; q < desc->n_sub; ++q) {
    const auto& s = p->subs[q];
    const int ex = (int)s.ext[0], ey = (int)s.ext[1], ez = (int)s.ext[2], wz = (int)s.own[2];
    p->max_ex = std::max(p->max_ex, ex);
    p->max_ey = std::max(p->max_ey, ey);
    p->max_ez = std::max(p->max_ez, ez);
    p->max_p = std::max(p->max_p, ex * ey);
    const int ns = slab_planes(ex, ey);
    for (int c = 0; c < 3; ++c) {
      for (int k0 = 0; k0 < ez; k0 += ns) fwd.push_back(make_int4((int)q, c, k0, std::min(ns, ez - k0)));
      for (int k0 = 0; k0 < wz; k0 += ns) inv.push_back(make_int4((int)q, c, k0, std::min(ns, wz - k0)));
    }
    for (int p0 = 0; p0 < ex * ey; p0 += TP) col.push_back(make_int2((int)q, p0));
  }
  const int mx = std::max(p->max_ex, std::max(p->max_ey, p->max_ez));
  if (mx > MAXR || mx > desc->pmax) {
    free_plan(p);
    FMP_REQUIRE(false, "extended extent %d exceeds the supported maximum %d (or pmax %lld)", mx, MAXR,
                (long long)desc->pmax);
  }
  // fast-path eligibility and its per-plane / per-8-column work items
  {
    std::vector<int> exts;
    for (const auto& sh : p->shapes)
      for (int a = 0; a < 3; ++a)
        if (std::find(exts.begin(), exts.end(), (int)sh.ext[a]) == exts.end()) exts.push_back((int)sh.ext[a]);
    const char* force = getenv("FMP_FORCE_GENERAL");
    p->fast = (int)exts.size() <= FX_MAXE && mx <= FAST_MAX_EXT && !(force && force[0] == '1');
    if (p->fast) {
      p->et.n = (int)exts.size();
      for (int e = 0; e < p->et.n; ++e) {
        p->et.ext[e] = exts[e];
        for (const auto& sh : p->shapes)
          for (int a = 0; a < 3; ++a)
            if ((int)sh.ext[a] == exts[e]) {
              p->et.ut[e] = sh.ut_off[a];
              p->et.vt[e] = sh.vt_off[a];
              p->et.sg[e] = sh.s_off[a];
            }
      }
      std::vector<int4> ff, ffb, fi;
      std::vector<int2> fc;
      // block extents = the union of the owned tiles; a subdomain whose extended box leaves the
      // block reads neighbour ghosts (its forward plane items go last, fmp_precond_apply_part)
      int64_t blk_ext[3] = {0, 0, 0};
      for (int64_t q = 0; q < desc->n_sub; ++q)
        for (int a = 0; a < 3; ++a)
          blk_ext[a] = std::max(blk_ext[a], p->subs[q].ext_lo[a] + p->subs[q].own_off[a] + p->subs[q].own[a]);
      for (int64_t q = 0; q < desc->n_sub; ++q) {
        const auto& sd = p->subs[q];
        const int ez = (int)sd.ext[2], wz = (int)sd.own[2], P = (int)(sd.ext[0] * sd.ext[1]);
        bool ghost = false;
        for (int a = 0; a < 3; ++a) ghost = ghost || sd.ext_lo[a] < 0 || sd.ext_lo[a] + sd.ext[a] > blk_ext[a];
        for (int c = 0; c < 3; ++c) {
          for (int k = 0; k < ez; ++k) (ghost ? ffb : ff).push_back(make_int4((int)q, c, k, 1));
          for (int k = 0; k < wz; ++k) fi.push_back(make_int4((int)q, c, k, 1));
        }
        for (int p0 = 0; p0 < P; p0 += 8) fc.push_back(make_int2((int)q, p0));
      }
      p->n_ffwd_int = (int)ff.size();
      ff.insert(ff.end(), ffb.begin(), ffb.end());
      p->n_ffwd = (int)ff.size();
      p->n_finv = (int)fi.size();
      p->n_fcol = (int)fc.size();
      if (upload(ff, &p->d_ffwd) || upload(fi, &p->d_finv) || upload(fc, &p->d_fcol)) {
        free_plan(p);
        return -1;
      }
      // one 3-D tensor map per subdomain slot and workspace: (column p, z, component), so a
      // column tile (8 columns x CXR z x 3 components) is a single TMA box; z rows past ez and
      // columns past the plane come back zero-filled
      bool col_tma = !getenv_flag("FMP_COL_NO_TMA") && ((uintptr_t)desc->work_a & 15) == 0 &&
                     ((uintptr_t)desc->work_b & 15) == 0;
      for (int64_t q = 0; q < desc->n_sub; ++q) col_tma = col_tma && (p->subs[q].ws_off & 1) == 0;
      if (col_tma) {
        std::vector<CUtensorMap> maps(2 * desc->n_sub);
        for (int w = 0; w < 2; ++w) {
          const double* base = w == 0 ? desc->work_a : desc->work_b;
          for (int64_t q = 0; q < desc->n_sub; ++q) {
            const auto& sd = p->subs[q];
            const uint64_t ps = (uint64_t)((sd.ext[0] * sd.ext[1] + 3) & ~3LL), ez = (uint64_t)sd.ext[2];
            const uint64_t dims[3] = {ps, ez, 3};
            const uint64_t strides[2] = {ps * 8, ps * ez * 8};
            const uint32_t box[3] = {8, CXR, 3};
            if (encode_tensor_map_f64(&maps[w * desc->n_sub + q], base + sd.ws_off, 3, dims, strides, box)) {
              free_plan(p);
              return -1;
            }
          }
        }
        if (upload(maps, &p->d_colmaps)) {
          free_plan(p);
          return -1;
        }
      }
    }
  }
  // large-path eligibility (not fast, every extent <= LN): column items per z extent
  {
    const char* force = getenv("FMP_FORCE_GENERAL");
    p->large = !p->fast && mx <= LN && !(force && force[0] == '1') && !getenv_flag("FMP_NO_LARGE");
    if (p->large) {
      std::vector<int> ezs;
      for (const auto& sd : p->subs)
        if (std::find(ezs.begin(), ezs.end(), (int)sd.ext[2]) == ezs.end()) ezs.push_back((int)sd.ext[2]);
      std::sort(ezs.begin(), ezs.end());
      std::vector<int2> items;
      for (int ez : ezs) {
        fmp_precond::LColGroup gr{ez, (int)items.size(), 0, 0, 0, -1, -1};
        int wzmax = 1;
        for (int64_t q = 0; q < desc->n_sub; ++q) {
          const auto& sd = p->subs[q];
          if ((int)sd.ext[2] != ez) continue;
          wzmax = std::max(wzmax, (int)sd.own[2]);
          for (int p0 = 0; p0 < (int)(sd.ext[0] * sd.ext[1]); p0 += 8) items.push_back(make_int2((int)q, p0));
        }
        for (const auto& sh : p->shapes)
          if ((int)sh.ext[2] == ez) {
            gr.ut = sh.ut_off[2];
            gr.vt = sh.vt_off[2];
          }
        gr.n = (int)items.size() - gr.off;
        gr.mt_fwd = ez % 8 <= 4 ? ez / 8 : ez / 8 + 1;   // remainder rows (<= 4) on DFMA
        gr.mt_inv = pad8(wzmax) / 8;
        if (gr.mt_fwd < 5 || gr.mt_fwd > 9 || gr.mt_inv < 5 || gr.mt_inv > 9) p->large = false;
        p->lcol.push_back(gr);
      }
      if (p->large && upload(items, &p->d_lcol)) {
        free_plan(p);
        return -1;
      }
      // plane items grouped by (component, ex, ey); CTAs assigned to combinations in proportion
      // to their planes, each CTA a contiguous range of one combination's items
      int sms_now = kNumSM;
      {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms_now, cudaDevAttrMultiProcessorCount, dev);
      }
      for (int dir = 0; dir < 2 && p->large; ++dir) {
        struct Combo { int c, ex, ey; int64_t fx, fy; std::vector<int2> items; };
        std::vector<Combo> combos;
        for (int64_t q = 0; q < desc->n_sub; ++q) {
          const auto& sd = p->subs[q];
          const auto& sh = p->shapes[sd.shape];
          const int ex = (int)sd.ext[0], ey = (int)sd.ext[1], np = dir == 0 ? (int)sd.ext[2] : (int)sd.own[2];
          for (int c = 0; c < 3; ++c) {
            size_t k = 0;
            while (k < combos.size() && !(combos[k].c == c && combos[k].ex == ex && combos[k].ey == ey)) ++k;
            if (k == combos.size())
              combos.push_back(Combo{c, ex, ey, c == 0 ? sh.ut_off[0] : sh.vt_off[0], c == 1 ? sh.ut_off[1] : sh.vt_off[1], {}});
            for (int z = 0; z < np; ++z) combos[k].items.push_back(make_int2((int)q, z));
          }
        }
        int64_t total = 0;
        for (const auto& cb : combos) total += (int64_t)cb.items.size();
        const int budget = std::max<int>(sms_now, (int)combos.size());
        std::vector<LargePlaneCta> ctas;
        std::vector<int2> items;
        for (const auto& cb : combos) {
          const int n = (int)cb.items.size();
          const int nc = std::max(1, std::min(n, (int)((int64_t)budget * n / std::max<int64_t>(total, 1))));
          const int base = (int)items.size();
          items.insert(items.end(), cb.items.begin(), cb.items.end());
          for (int b = 0; b < nc; ++b)
            ctas.push_back(LargePlaneCta{base + (int)((int64_t)n * b / nc), base + (int)((int64_t)n * (b + 1) / nc), cb.c,
                                         cb.ex, cb.ey, 0, cb.fx, cb.fy});
        }
        p->n_lpc[dir] = (int)ctas.size();
        if (upload(ctas, &p->d_lpc[dir]) || upload(items, &p->d_lpi[dir])) {
          free_plan(p);
          return -1;
        }
      }
      bool col_tma = p->large && !getenv_flag("FMP_COL_NO_TMA") && ((uintptr_t)desc->work_a & 15) == 0 &&
                     ((uintptr_t)desc->work_b & 15) == 0;
      for (int64_t q = 0; q < desc->n_sub; ++q) col_tma = col_tma && (p->subs[q].ws_off & 1) == 0;
      if (col_tma) {
        std::vector<CUtensorMap> maps(2 * desc->n_sub);
        for (int w = 0; w < 2; ++w) {
          const double* base = w == 0 ? desc->work_a : desc->work_b;
          for (int64_t q = 0; q < desc->n_sub; ++q) {
            const auto& sd = p->subs[q];
            const uint64_t ps = (uint64_t)((sd.ext[0] * sd.ext[1] + 3) & ~3LL), ez = (uint64_t)sd.ext[2];
            const uint64_t dims[3] = {ps, ez, 3};
            const uint64_t strides[2] = {ps * 8, ps * ez * 8};
            const uint32_t box[3] = {8, LCXR, 3};
            if (encode_tensor_map_f64(&maps[w * desc->n_sub + q], base + sd.ws_off, 3, dims, strides, box)) {
              free_plan(p);
              return -1;
            }
          }
        }
        if (upload(maps, &p->d_lcolmaps)) {
          free_plan(p);
          return -1;
        }
      }
    }
  }
  p->n_fwd = (int)fwd.size();
  p->n_inv = (int)inv.size();
  p->n_col = (int)col.size();
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, dev);
  if (upload(fwd, &p->d_fwd_items) || upload(inv, &p->d_inv_items) || upload(col, &p->d_col_items) ||
      upload(p->ymat, &p->d_ymat) || upload(p->zmat, &p->d_zmat)) {
    free_plan(p);
    return -1;
  }
  // rotation groups: one C^-1 / Y / Z / GEMM per group, n = all member columns
  p->gcols.assign(desc->n_shape, 0);
  for (int64_t s2 = 0; s2 < desc->n_shape; ++s2) {
    const auto& sh = p->shapes[s2];
    const int64_t g = sh.group;
    FMP_REQUIRE(g >= 0 && g < desc->n_shape && p->shapes[g].group == g && p->shapes[g].m == sh.m &&
                    p->shapes[g].ld == sh.ld && (g == s2 || (sh.rowmap_off >= 0 && desc->rowmap)),
                "shape %lld: invalid rotation group %lld", (long long)s2, (long long)g);
    p->gcols[g] += (int)(p->first[s2 + 1] - p->first[s2]);
  }
  {  // grouped GEMM tables: one shape record per extended shape, tiles bucketed by configuration
    const char* gm = getenv("FMP_GEMM");
    std::string gmode = gm ? gm : "ozaki";   // cublas | own | ozaki
    p->use_cublas = gmode == "cublas";
    p->use_ozaki = gmode == "ozaki";
    std::vector<GemmShape> gs;
    std::vector<GemmTile> gt[3];
    for (int64_t s2 = 0; s2 < desc->n_shape; ++s2) {
      const auto& sh = p->shapes[s2];
      const int n = p->gcols[s2];
      gs.push_back(GemmShape{p->cinv[s2], p->ymat[s2], p->zmat[s2], (int)sh.m, n, (int)sh.ld});
      if (n == 0) continue;
      const int cfg = gemm_config_of(n), mt = gemm_tile_m(cfg), nt = gemm_tile_n(cfg);
      for (int i0 = 0; i0 < sh.m; i0 += mt)
        for (int n0 = 0; n0 < n; n0 += nt) gt[cfg].push_back(GemmTile{(int)s2, i0, n0, 0});
    }
    if (upload(gs, &p->d_gshapes) || upload(gt[0], &p->d_gtiles[0]) || upload(gt[1], &p->d_gtiles[1]) ||
        upload(gt[2], &p->d_gtiles[2]) || gemm_setup()) {
      free_plan(p);
      return -1;
    }
    for (int c = 0; c < 3; ++c) p->n_gtiles[c] = (int)gt[c].size();
  }
  {  // padded forward factors of the face kernels (k_faces / k_corr): [U^T_n, V^T_n] per extent
    const int pm = (int)p->d.pmax, NTf = pm <= 24 ? 3 : (pm <= 40 ? 5 : 9), N = 8 * NTf, S = N + 4;
    std::vector<int64_t> off;
    std::vector<int> ext;
    for (const auto& sh : p->shapes)
      for (int a = 0; a < 3; ++a) {
        const int n = (int)sh.ext[a];
        FMP_REQUIRE(n > 0 && n < 80 && n <= N, "face factors: extent %d", n);
        if (std::find(ext.begin(), ext.end(), n) != ext.end()) continue;
        p->pad_slot[n] = (unsigned char)(ext.size() / 2);
        ext.push_back(n);
        off.push_back(sh.ut_off[a]);
        ext.push_back(n);
        off.push_back(sh.vt_off[a]);
      }
    int64_t* d_off = nullptr;
    int* d_ext = nullptr;
    if (cudaMalloc(&p->facepad, sizeof(double) * (size_t)N * S * ext.size()) != cudaSuccess || upload(off, &d_off) ||
        upload(ext, &d_ext)) {
      cudaFree(d_off);
      cudaFree(d_ext);
      free_plan(p);
      FMP_REQUIRE(false, "face factor padding: allocation failed");
    }
    k_pad_factors<<<dim3(8, (unsigned)ext.size()), 256>>>(p->d.factors, d_off, d_ext, (int)ext.size(), N, S, p->facepad);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaFree(d_off);
    cudaFree(d_ext);
    FMP_CHECK_CUDA(e);
  }
  bool have_cinv = desc->alpha != 0.0;
  for (const double* c : p->cinv) have_cinv = have_cinv && c != nullptr;
  if (p->use_ozaki && have_cinv) {   // slices of C^-1 (setup), buffers for the slices of Y
    if (ozaki_setup()) { free_plan(p); return -1; }
    std::vector<OzShape> os;
    std::vector<OzSlice> sa, sb;
    for (int64_t s2 = 0; s2 < desc->n_shape; ++s2) {
      const auto& sh = p->shapes[s2];
      if (sh.group != s2) {   // member of a rotation group: the canonical shape's GEMM covers it
        os.push_back(OzShape{});
        continue;
      }
      const int m = (int)sh.m, n = p->gcols[s2], kc = ozaki_kchunks(m);
      const int w = ozaki_width(std::max(n, 1));
      int8_t *a = nullptr, *b = nullptr;
      int *ea = nullptr, *eb = nullptr;
      const size_t ab = ozaki_a_bytes(m, kc), bb = ozaki_b_bytes(std::max(n, 1), kc);
      if (cudaMalloc(&a, ab) != cudaSuccess || cudaMalloc(&b, bb) != cudaSuccess ||
          cudaMalloc(&ea, sizeof(int) * m) != cudaSuccess || cudaMalloc(&eb, sizeof(int) * std::max(n, 1)) != cudaSuccess ||
          cudaMemset(b, 0, bb) != cudaSuccess) {   // the stacked rows past S w stay zero
        free_plan(p);
        FMP_REQUIRE(false, "cudaMalloc of Ozaki slices failed");
      }
      p->oz_a.push_back(a);
      p->oz_b.push_back(b);
      p->oz_ea.push_back(ea);
      p->oz_eb.push_back(eb);
      // locality order of the correction rows (both C^-1 axes, Y's K axis, Z's rows)
      int* perm = nullptr;
      // (boxes with an extent < 24, 16^3-class subdomains: no gain, and the gathered Y slicing costs)
      if (!getenv_flag("FMP_OZ_NOPERM") && std::max(sh.ext[0], std::max(sh.ext[1], sh.ext[2])) >= 24) {
        const std::vector<int> h = ozaki_row_order((int)sh.ext[0], (int)sh.ext[1], (int)sh.ext[2]);
        FMP_REQUIRE((int64_t)h.size() == m, "Ozaki row order: %zu rows for m = %d", h.size(), m);
        if (upload(h, &perm)) {
          free_plan(p);
          return -1;
        }
        p->oz_perm.push_back(perm);
      }
      sa.push_back(OzSlice{p->cinv[s2], a, ea, perm, perm, m, (int)sh.ld, m, kc, ozaki_tile_m(), 0, 0, 0, 0, 0});
      if (n > 0)
        sb.push_back(OzSlice{p->ymat[s2], b, eb, nullptr, perm, n, (int)sh.ld, m, kc, w, 1, ozaki_stack_rows(w), 0, 0, 0});
      os.push_back(OzShape{a, ea, b, eb, p->zmat[s2], m, n, (int)sh.ld, kc, w, ozaki_stack_rows(w), nullptr, nullptr,
                           nullptr, perm});
    }
    int64_t ra = 0, qa = 0;
    ozaki_plan_slices(sa.data(), (int)sa.size(), &ra, &qa);
    ozaki_plan_slices(sb.data(), (int)sb.size(), &p->oz_rows, &p->oz_threads);
    OzSlice* d_sa = nullptr;
    if (upload(sa, &d_sa) || upload(sb, &p->d_ozslices)) {
      cudaFree(d_sa);
      free_plan(p);
      return -1;
    }
    p->n_ozslices = (int)sb.size();
    const int rc = ozaki_slice(d_sa, (int)sa.size(), ra, qa, 0);
    cudaDeviceSynchronize();
    cudaFree(d_sa);
    if (rc) { free_plan(p); return -1; }
    FMP_CHECK_CUDA(cudaDeviceSynchronize());
    // chunk lists of the non-zero C^-1 slice blocks (zero-slice skipping), then the schedule
    std::vector<OzLists> lists;
    if (ozaki_chunk_lists(os, &lists, &p->oz) || ozaki_build(os, lists, p->sms, &p->oz)) {
      free_plan(p);
      return -1;
    }
  }
  if (cublasCreate(&p->blas) != CUBLAS_STATUS_SUCCESS) {
    free_plan(p);
    FMP_REQUIRE(false, "cublasCreate failed");
  }
  cublasSetMathMode(p->blas, CUBLAS_DEFAULT_MATH);
  for (int q = 0; q < fmp_precond::kAux; ++q) {
    if (cudaStreamCreateWithFlags(&p->aux[q], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_join[q], cudaEventDisableTiming) != cudaSuccess ||
        cublasCreate(&p->aux_blas[q]) != CUBLAS_STATUS_SUCCESS) {
      free_plan(p);
      FMP_REQUIRE(false, "auxiliary stream setup failed");
    }
    cublasSetStream(p->aux_blas[q], p->aux[q]);
  }
  if (cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess) {
    free_plan(p);
    FMP_REQUIRE(false, "event creation failed");
  }
  for (int64_t s2 = 0; s2 < desc->n_shape; ++s2)
    if (p->gcols[s2] > 0) p->gemm_order.push_back((int)s2);
  std::sort(p->gemm_order.begin(), p->gemm_order.end(), [&](int a, int b) {
    const double fa = (double)p->shapes[a].m * p->shapes[a].m * (double)p->gcols[a];
    const double fb = (double)p->shapes[b].m * p->shapes[b].m * (double)p->gcols[b];
    return fa > fb;
  });
  plane_attr<false, 5>(); plane_attr<true, 5>(); plane_attr<false, 9>(); plane_attr<true, 9>();
  column_attr<1>(); column_attr<2>(); column_attr<3>(); column_attr<4>(); column_attr<5>();
  column_attr<6>(); column_attr<7>(); column_attr<8>(); column_attr<9>();
  cudaFuncSetAttribute(k_plane_fast<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_plane_fast<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_plane_fast<false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_plane_fast<false, 5, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_plane_fast<false, 5, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_plane_fast<false, 3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_plane_fast<false, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_plane_fast<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneFastSmem);
  cudaFuncSetAttribute(k_column_fast<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColFastSmem);
  cudaFuncSetAttribute(k_column_fast<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColFastSmem);
  cudaFuncSetAttribute(k_column_fast_db<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, col_db_smem(CW_WARPS_FWD));
  cudaFuncSetAttribute(k_column_fast_db<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, col_db_smem(CW_WARPS_INV));
  cudaFuncSetAttribute(k_column_fast_db<false, CW_WARPS_FWD, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       col_db_smem(CW_WARPS_FWD));
  cudaFuncSetAttribute(k_column_fast_db<true, CW_WARPS_INV, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       col_db_smem(CW_WARPS_INV));

  {
    const int slot = face_slot((p->max_p + 3) & ~3);
    cudaFuncSetAttribute(k_faces<3, 1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)face_smem_bytes<3>(slot));
    cudaFuncSetAttribute(k_faces<5, 2, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)face_smem_bytes<5>(slot));
    cudaFuncSetAttribute(k_faces<9, 3, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)face_smem_bytes<9>(slot));
  }
  cudaFuncSetAttribute(k_corr<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * FaceMat<3>::WORDS * 8);
  cudaFuncSetAttribute(k_corr<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * FaceMat<5>::WORDS * 8);
  cudaFuncSetAttribute(k_corr<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * FaceMat<9>::WORDS * 8);
  if (p->large) {
#define FMP_LCA(MT)                                                                                              \
  cudaFuncSetAttribute(k_column_large<false, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColLargeSmem); \
  cudaFuncSetAttribute(k_column_large<true, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColLargeSmem);
    FMP_LCA(5) FMP_LCA(6) FMP_LCA(7) FMP_LCA(8) FMP_LCA(9)
#undef FMP_LCA
    cudaFuncSetAttribute(k_plane_large<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneLargeSmem);
    cudaFuncSetAttribute(k_plane_large<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlaneLargeSmem);
  }
  FMP_CHECK_CUDA(cudaGetLastError());
  *out = p;
  return 0;
}

extern "C" int fmp_precond_path(const fmp_precond* p) {
  FMP_REQUIRE(p, "null plan");
  return p->fast ? FMP_PATH_FAST : (p->large ? FMP_PATH_LARGE : FMP_PATH_GENERAL);
}

extern "C" int fmp_precond_ozaki_stats(const fmp_precond* p, double* out, int n) {
  FMP_REQUIRE(p && out, "null argument");
  const double v[2] = {p->use_ozaki ? p->oz.kept_slices : 1.0, p->use_ozaki ? p->oz.kept_mma : 1.0};
  for (int i = 0; i < n && i < 2; ++i) out[i] = v[i];
  return n < 2 ? n : 2;
}

extern "C" int fmp_precond_destroy(fmp_precond* p) {
  free_plan(p);
  return 0;
}

static int column_pass(fmp_precond* p, bool inv, const double* src, double* dst, const double* corr,
                       cudaStream_t st) {
  if (p->fast) {
    FastColArgs a{};
    a.subs = p->d.subs;
    a.items = p->d_fcol;
    a.n_items = p->n_fcol;
    a.src = src;
    a.dst = dst;
    a.factors = p->d.factors;
    a.corr = corr;
    if (inv && getenv_flag("FMP_COL_NO_CORR")) a.corr = nullptr;   // timing diagnostic only: wrong results
    a.pmax = (int)p->d.pmax;
    a.alpha = p->d.alpha;
    a.et = p->et;
    // forward: CTA-contiguous item ranges, warps interleaved inside the CTA (measured 0.235 ->
    // 0.227 ms at cfg4); inverse: warps interleaved over the whole launch (CTA ranges: 0.264 ->
    // 0.273 ms)
    a.interleave = getenv_flag("FMP_COL_CONTIG") ? 0 : (inv ? 1 : 2);
    a.no_rem = getenv_flag("FMP_COL_NO_REM") ? 1 : 0;
    a.maps = p->d_colmaps ? p->d_colmaps + (src == p->d.work_a ? 0 : p->d.n_sub) : nullptr;
    if (a.maps && src != p->d.work_a && src != p->d.work_b) a.maps = nullptr;
    a.unroll = a.maps != nullptr && inv ? 1 : 0;   // measured: inverse 0.273 -> 0.268 ms, forward no gain
    if (inv && getenv_flag("FMP_COL_SINGLE")) {
      const int grid = std::min(p->sms, (p->n_fcol + CW_WARPS - 1) / CW_WARPS);
      k_column_fast<true><<<grid, CW_WARPS * 32, kColFastSmem, st>>>(a);
    } else {
      const bool small = std::max(p->max_ex, std::max(p->max_ey, p->max_ez)) <= 24;
      const int nwarp = inv ? CW_WARPS_INV : CW_WARPS_FWD;
      const int grid = std::min(p->sms, (p->n_fcol + nwarp - 1) / nwarp);
#define FMP_COLF(I, S) \
  FMP_CHECK_CUDA(launch_pdl(k_column_fast_db<I, I ? CW_WARPS_INV : CW_WARPS_FWD, S>, grid, nwarp * 32, col_db_smem(nwarp), st, a));
      if (inv && small) { FMP_COLF(true, 3) }
      else if (inv) { FMP_COLF(true, 5) }
      else if (small) { FMP_COLF(false, 3) }
      else { FMP_COLF(false, 5) }
#undef FMP_COLF
    }
    FMP_CHECK_LAUNCH();
    return 0;
  }
  if (p->large) {
    for (const auto& gr : p->lcol) {
      LargeColArgs a{};
      a.subs = p->d.subs;
      a.shapes = p->d.shapes;
      a.items = p->d_lcol + gr.off;
      a.n_items = gr.n;
      a.src = src;
      a.dst = dst;
      a.factors = p->d.factors;
      a.ut = gr.ut;
      a.vt = gr.vt;
      a.ez = gr.ez;
      a.corr = corr;
      a.pmax = (int)p->d.pmax;
      a.alpha = p->d.alpha;
      a.maps = p->d_lcolmaps ? p->d_lcolmaps + (src == p->d.work_a ? 0 : p->d.n_sub) : nullptr;
      if (a.maps && src != p->d.work_a && src != p->d.work_b) a.maps = nullptr;
      const int grid = std::min(p->sms, (gr.n + LCW - 1) / LCW);
      const int mt = inv ? gr.mt_inv : gr.mt_fwd;
#define FMP_LCL(MT)                                                                     \
  case MT:                                                                              \
    if (inv)                                                                            \
      k_column_large<true, MT><<<grid, LCW * 32, kColLargeSmem, st>>>(a);               \
    else                                                                                \
      k_column_large<false, MT><<<grid, LCW * 32, kColLargeSmem, st>>>(a);              \
    break;
      switch (mt) {
        FMP_LCL(5) FMP_LCL(6) FMP_LCL(7) FMP_LCL(8) FMP_LCL(9)
        default: FMP_REQUIRE(false, "unsupported large column tile count %d", mt);
      }
#undef FMP_LCL
      FMP_CHECK_LAUNCH();
    }
    return 0;
  }
  ColArgs a{};
  a.subs = p->d.subs;
  a.shapes = p->d.shapes;
  a.factors = p->d.factors;
  a.items = p->d_col_items;
  a.n_items = p->n_col;
  a.src = src;
  a.dst = dst;
  a.corr = corr;
  a.pmax = (int)p->d.pmax;
  const int grid = std::min(p->n_col, 2 * p->sms);
#define FMP_COL(MT)                                                                   \
  case MT:                                                                            \
    if (inv)                                                                          \
      k_column<MT, true><<<grid, CW * 32, ColSmem<MT>::bytes, st>>>(a);               \
    else                                                                              \
      k_column<MT, false><<<grid, CW * 32, ColSmem<MT>::bytes, st>>>(a);              \
    break;
  switch (column_mt(p)) {
    FMP_COL(1) FMP_COL(2) FMP_COL(3) FMP_COL(4) FMP_COL(5) FMP_COL(6) FMP_COL(7) FMP_COL(8) FMP_COL(9)
    default: FMP_REQUIRE(false, "unsupported z extent");
  }
#undef FMP_COL
  FMP_CHECK_LAUNCH();
  return 0;
}

// the fused Krylov vector update of the forward plane pass (FastPlaneArgs::lc_kind)
struct LincombOp {
  int kind = 0;
  const double* r = nullptr;
  const double* v = nullptr;
  double beta = 0.0, gamma = 0.0;
  double* out = nullptr;
};

static int plane_pass(fmp_precond* p, const fmp_block* blk, bool inv, int mode, const double* src, double* dst,
                      cudaStream_t st, int part = FMP_PART_ALL, const LincombOp& lc = LincombOp()) {
  if (p->fast) {
    FastPlaneArgs a{};
    a.subs = p->d.subs;
    a.items = inv ? p->d_finv : p->d_ffwd;
    a.n_items = inv ? p->n_finv : p->n_ffwd;
    if (!inv && part == FMP_PART_INTERIOR) a.n_items = p->n_ffwd_int;
    if (!inv && part == FMP_PART_BOUNDARY) {
      a.items += p->n_ffwd_int;
      a.n_items -= p->n_ffwd_int;
    }
    if (a.n_items == 0) return 0;
    a.g = make_geo(blk);
    a.src = src;
    a.dst = dst;
    a.factors = p->d.factors;
    a.mode = mode;
    a.et = p->et;
    a.interleave = getenv_flag("FMP_PLANE_CONTIG") ? 0 : 1;   // round-robin planes (DRAM page locality)
    a.lc_kind = inv ? 0 : lc.kind;
    a.lc_prefetch = getenv_flag("FMP_LC_PREFETCH") ? 1 : 0;
    a.lc_r = lc.r;
    a.lc_v = lc.v;
    a.lc_beta = lc.beta;
    a.lc_gamma = lc.gamma;
    a.lc_out = lc.out;
    CUtensorMap tm{};
    a.tma_rows = 0;
    if (!inv && mode != FMP_SOLVE_FACES && (blk->bx & 1) == 0 && ((uintptr_t)src & 15) == 0 &&
        !getenv_flag("FMP_PLANE_NO_TMA")) {
      // the block field as a 4-D tensor (x, y, z, component); box = one haloed subdomain plane
      const uint64_t dims[4] = {(uint64_t)blk->bx, (uint64_t)blk->by, (uint64_t)blk->bz, 3};
      const uint64_t strides[3] = {(uint64_t)blk->bx * 8, (uint64_t)(blk->bx * blk->by) * 8,
                                   (uint64_t)(blk->bx * blk->by * blk->bz) * 8};
      const uint32_t box[4] = {PXS, (uint32_t)p->max_ey, 1, 1};
      if (int e = encode_tensor_map_f64(&tm, src, 4, dims, strides, box)) return e;
      a.tma_rows = p->max_ey;
    }
    const int grid = std::min(p->sms, (a.n_items + PW_WARPS - 1) / PW_WARPS);
    const bool small = std::max(p->max_ex, std::max(p->max_ey, p->max_ez)) <= 24;
    if (inv && small)
      FMP_CHECK_CUDA(launch_pdl(k_plane_fast<true, 3>, grid, PW_WARPS * 32, kPlaneFastSmem, st, tm, a));
    else if (inv)
      FMP_CHECK_CUDA(launch_pdl(k_plane_fast<true>, grid, PW_WARPS * 32, kPlaneFastSmem, st, tm, a));
    else if (small)
      FMP_CHECK_CUDA(launch_pdl(a.lc_kind == 0 ? k_plane_fast<false, 3> : (a.lc_kind == 1 ? k_plane_fast<false, 3, 1> : k_plane_fast<false, 3, 2>),
                                grid, PW_WARPS * 32, kPlaneFastSmem, st, tm, a));
    else
      FMP_CHECK_CUDA(launch_pdl(a.lc_kind == 0 ? k_plane_fast<false> : (a.lc_kind == 1 ? k_plane_fast<false, 5, 1> : k_plane_fast<false, 5, 2>),
                                grid, PW_WARPS * 32, kPlaneFastSmem, st, tm, a));
    FMP_CHECK_LAUNCH();
    return 0;
  }
  if (p->large && !getenv_flag("FMP_NO_LARGE_PLANE")) {
    const int dir = inv ? 1 : 0;
    LargePlaneArgs a{};
    a.subs = p->d.subs;
    a.ctas = p->d_lpc[dir];
    a.items = p->d_lpi[dir];
    a.g = make_geo(blk);
    a.src = src;
    a.dst = dst;
    a.factors = p->d.factors;
    a.mode = mode;
    CUtensorMap tm{};
    a.tma_rows = 0;
    if (!inv && mode != FMP_SOLVE_FACES && (blk->bx & 1) == 0 && ((uintptr_t)src & 15) == 0 &&
        !getenv_flag("FMP_PLANE_NO_TMA")) {
      const uint64_t dims[4] = {(uint64_t)blk->bx, (uint64_t)blk->by, (uint64_t)blk->bz, 3};
      const uint64_t strides[3] = {(uint64_t)blk->bx * 8, (uint64_t)(blk->bx * blk->by) * 8,
                                   (uint64_t)(blk->bx * blk->by * blk->bz) * 8};
      const uint32_t box[4] = {LSM, (uint32_t)p->max_ey, 1, 1};
      if (int e = encode_tensor_map_f64(&tm, src, 4, dims, strides, box)) return e;
      a.tma_rows = p->max_ey;
    }
    if (inv)
      k_plane_large<true><<<p->n_lpc[dir], LPG * 128, kPlaneLargeSmem, st>>>(tm, a);
    else
      k_plane_large<false><<<p->n_lpc[dir], LPG * 128, kPlaneLargeSmem, st>>>(tm, a);
    FMP_CHECK_LAUNCH();
    return 0;
  }
  PlaneArgs a{};
  a.subs = p->d.subs;
  a.shapes = p->d.shapes;
  a.factors = p->d.factors;
  a.items = inv ? p->d_inv_items : p->d_fwd_items;
  a.n_items = inv ? p->n_inv : p->n_fwd;
  a.g = make_geo(blk);
  a.src = src;
  a.dst = dst;
  a.mode = mode;
  const int grid = std::min(a.n_items, 2 * p->sms);
  if (plane_nt(p) == 5) {
    if (inv) k_plane<true, 5><<<grid, PW * 32, PlaneSmem<5>::bytes, st>>>(a);
    else k_plane<false, 5><<<grid, PW * 32, PlaneSmem<5>::bytes, st>>>(a);
  } else {
    if (inv) k_plane<true, 9><<<grid, PW * 32, PlaneSmem<9>::bytes, st>>>(a);
    else k_plane<false, 9><<<grid, PW * 32, PlaneSmem<9>::bytes, st>>>(a);
  }
  FMP_CHECK_LAUNCH();
  return 0;
}

static int precond_apply(fmp_precond* p, const fmp_block* blk, int mode, int part, const double* r, double* z,
                         void* stream, const LincombOp& lc = LincombOp());

// the fused forms need the fast kernels and a block without ghosts (ghost planes of the input
// would have to be formed from the operands' ghosts); FACES mode reads compact fields.  Plans
// of 16^3-class subdomains (extents <= 24) run the two-pass form: their planes carry 1.4x halo
// re-reads against little DMMA work, and fusing measured 3% slower (cfg5_sd16: 24.3 -> 25.0 ms
// per step)
static bool fusable(const fmp_precond* p, const fmp_block* blk, int mode) {
  bool ghosts = false;
  for (int q = 0; q < 6; ++q) ghosts |= blk->ghost[q] != nullptr;
  const bool small = std::max(p->max_ex, std::max(p->max_ey, p->max_ez)) <= 24;
  return p->fast && !small && !ghosts && mode != FMP_SOLVE_FACES && !getenv_flag("FMP_NO_FUSED_LINCOMB");
}

extern "C" int fmp_precond_apply(fmp_precond* p, const fmp_block* blk, int mode, const double* r, double* z,
                                 void* stream) {
  return precond_apply(p, blk, mode, FMP_PART_ALL, r, z, stream);
}

extern "C" int fmp_precond_apply_part(fmp_precond* p, const fmp_block* blk, int mode, int part, const double* r,
                                      double* z, void* stream) {
  FMP_REQUIRE(part >= FMP_PART_ALL && part <= FMP_PART_BOUNDARY, "bad part %d", part);
  return precond_apply(p, blk, mode, part, r, z, stream);
}

extern "C" int fmp_precond_apply_lincomb(fmp_precond* p, const fmp_block* blk, int mode, const double* r,
                                         const double* v, double beta, double* s, double* z, void* stream) {
  FMP_REQUIRE(p && blk && r && v && s, "null argument");
  if (!fusable(p, blk, mode)) {   // the two-pass form
    const int64_t n = 3 * blk->bx * blk->by * blk->bz;
    if (int e = fmp_vec_lincomb(n, 1.0, r, beta, v, s, stream)) return e;
    return precond_apply(p, blk, mode, FMP_PART_ALL, s, z, stream);
  }
  LincombOp lc;
  lc.kind = 1;
  lc.v = v;
  lc.beta = beta;
  lc.out = s;
  return precond_apply(p, blk, mode, FMP_PART_ALL, r, z, stream, lc);
}

extern "C" int fmp_precond_apply_bicg_p(fmp_precond* p, const fmp_block* blk, int mode, const double* r,
                                        const double* p_old, const double* v, double beta, double omega,
                                        double* p_new, double* z, void* stream) {
  FMP_REQUIRE(p && blk && r && p_old && v && p_new, "null argument");
  FMP_REQUIRE(p_new != p_old && p_new != r && p_new != v, "p_new must not alias an operand");
  if (!fusable(p, blk, mode)) {   // the two-pass form (fmp_bicg_p updates in place: copy first)
    const int64_t n = 3 * blk->bx * blk->by * blk->bz;
    FMP_CHECK_CUDA(cudaMemcpyAsync(p_new, p_old, n * sizeof(double), cudaMemcpyDeviceToDevice, as_stream(stream)));
    if (int e = fmp_bicg_p(n, r, p_new, v, beta, omega, stream)) return e;
    return precond_apply(p, blk, mode, FMP_PART_ALL, p_new, z, stream);
  }
  LincombOp lc;
  lc.kind = 2;
  lc.r = r;
  lc.v = v;
  lc.beta = beta;
  lc.gamma = -omega;
  lc.out = p_new;
  return precond_apply(p, blk, mode, FMP_PART_ALL, p_old, z, stream, lc);
}

static int precond_apply(fmp_precond* p, const fmp_block* blk, int mode, int part, const double* r, double* z,
                         void* stream, const LincombOp& lc) {
  FMP_REQUIRE(p && blk, "null argument");
  FMP_REQUIRE(mode >= FMP_SOLVE_WOODBURY && mode <= FMP_SOLVE_FACES, "bad solve mode %d", mode);
  cudaStream_t st = as_stream(stream);
  double* wa = p->d.work_a;
  double* wb = p->d.work_b;
  auto mark = [&](int i) {
    if (p->profile) cudaEventRecord(p->stage_ev[i], st);
  };
  // Only the forward plane pass reads the input field (and its ghosts); every later kernel reads
  // the workspaces.  The interior part is that pass over the subdomains that read no ghost; the
  // boundary part is the pass over the others and everything after it.  (The general kernels and
  // FACES mode run whole in the boundary part.)
  const bool split = p->fast && mode != FMP_SOLVE_FACES;
  if (part != FMP_PART_BOUNDARY) mark(0);   // split: stage 0 spans interior pass, ghost wait, boundary pass
  if (part == FMP_PART_INTERIOR) return split ? plane_pass(p, blk, false, mode, r, wa, st, FMP_PART_INTERIOR) : 0;
  if (int e = plane_pass(p, blk, false, mode, r, wa, st, split ? part : FMP_PART_ALL, lc)) return e;
  mark(1);
  if (int e = column_pass(p, false, wa, wb, nullptr, st)) return e;
  mark(2);
  const int pm = (int)p->d.pmax;
  FaceArgs fa{p->d.subs, p->d.shapes, p->d.factors, wb, p->d.corr, p->d_ymat, p->d_zmat, pm, (p->max_p + 3) & ~3,
              p->d.rowmap, p->facepad, {}};
  fa.bulk_factors = getenv_flag("FMP_FACE_NO_BULK") ? 0 : 1;
  memcpy(fa.pad_slot, p->pad_slot, sizeof(fa.pad_slot));
  if (mode != FMP_SOLVE_EXACT) {
    const dim3 fg(3, (unsigned)p->d.n_sub);
    const int slot = face_slot(fa.max_ps);
    if (pm <= 24)   // 16^3-class subdomains: 3 DMMA tiles per padded extent
      FMP_CHECK_CUDA(launch_pdl(k_faces<3, 1, 3>, fg, FACE_THREADS, face_smem_bytes<3>(slot), st, fa));
    else if (pm <= 40)
      FMP_CHECK_CUDA(launch_pdl(k_faces<5, 2, 5>, fg, FACE_THREADS, face_smem_bytes<5>(slot), st, fa));
    else
      FMP_CHECK_CUDA(launch_pdl(k_faces<9, 3, 9>, fg, FACE_THREADS, face_smem_bytes<9>(slot), st, fa));
    FMP_CHECK_LAUNCH();
  }
  mark(3);
  if (mode == FMP_SOLVE_FACES) return 0;
  if (mode == FMP_SOLVE_WOODBURY) {
    if (!p->use_ozaki) mark(4);
    if (p->use_cublas) {
      // one DGEMM per shape; shapes spread over auxiliary streams (forked from / joined into
      // `st`) so the HBM-bound small-n products overlap the compute-bound large ones
      FMP_CHECK_CUDA(cudaEventRecord(p->ev_fork, st));
      const int naux = std::min<int>(fmp_precond::kAux, (int)p->gemm_order.size());
      for (int q = 0; q < naux; ++q) FMP_CHECK_CUDA(cudaStreamWaitEvent(p->aux[q], p->ev_fork, 0));
      const double one = 1.0, zero = 0.0;
      for (size_t o = 0; o < p->gemm_order.size(); ++o) {
        const int s = p->gemm_order[o];
        const int m = (int)p->shapes[s].m, ld = (int)p->shapes[s].ld;
        const int ncol = p->gcols[s];
        // C^-1 is row-major [m][ld]; OP_T makes cuBLAS use it as is.
        cublasStatus_t bs = cublasDgemm(p->aux_blas[o % naux], CUBLAS_OP_T, CUBLAS_OP_N, m, ncol, m, &one,
                                        p->cinv[s], ld, p->ymat[s], ld, &zero, p->zmat[s], ld);
        FMP_REQUIRE(bs == CUBLAS_STATUS_SUCCESS, "cublasDgemm failed (%d)", (int)bs);
      }
      for (int q = 0; q < naux; ++q) {
        FMP_CHECK_CUDA(cudaEventRecord(p->ev_join[q], p->aux[q]));
        FMP_CHECK_CUDA(cudaStreamWaitEvent(st, p->ev_join[q], 0));
      }
    } else if (p->use_ozaki) {
      FMP_REQUIRE(p->oz.shapes != nullptr, "Ozaki GEMM requested but the plan has no C^-1");
      if (int e = ozaki_slice(p->d_ozslices, p->n_ozslices, p->oz_rows, p->oz_threads, st)) return e;
      mark(4);
      if (int e = ozaki_launch(p->oz, st)) return e;
    } else {
      for (int c = 0; c < 3; ++c)
        if (int e = gemm_launch(c, p->d_gshapes, p->d_gtiles[c], p->n_gtiles[c], p->sms, st)) return e;
    }
    mark(5);
    if (pm <= 24)
      FMP_CHECK_CUDA(launch_pdl(k_corr<3>, dim3(6, (unsigned)p->d.n_sub), FACE_THREADS, 4 * FaceMat<3>::WORDS * sizeof(double), st, fa));
    else if (pm <= 40)
      FMP_CHECK_CUDA(launch_pdl(k_corr<5>, dim3(6, (unsigned)p->d.n_sub), FACE_THREADS, 4 * FaceMat<5>::WORDS * sizeof(double), st, fa));
    else
      FMP_CHECK_CUDA(launch_pdl(k_corr<9>, dim3(6, (unsigned)p->d.n_sub), FACE_THREADS, 4 * FaceMat<9>::WORDS * sizeof(double), st, fa));
    FMP_CHECK_LAUNCH();
  }
  mark(6);
  if (int e = column_pass(p, true, wb, wa, mode == FMP_SOLVE_WOODBURY ? p->d.corr : nullptr, st)) return e;
  mark(7);
  if (int e = plane_pass(p, blk, true, mode, wa, z, st)) return e;
  mark(8);
  return 0;
}

extern "C" int fmp_precond_profile(fmp_precond* p, int enable) {
  FMP_REQUIRE(p, "null plan");
  if (enable)
    for (auto& e : p->stage_ev)
      if (!e) FMP_CHECK_CUDA(cudaEventCreate(&e));
  p->profile = enable != 0;
  return 0;
}

extern "C" int fmp_precond_stage_ms(fmp_precond* p, float* ms, int n) {
  FMP_REQUIRE(p && ms && p->profile, "stage timing not enabled on this plan");
  FMP_CHECK_CUDA(cudaEventSynchronize(p->stage_ev[FMP_PRECOND_STAGES]));
  const int k = std::min(n, FMP_PRECOND_STAGES);
  for (int i = 0; i < k; ++i) FMP_CHECK_CUDA(cudaEventElapsedTime(&ms[i], p->stage_ev[i], p->stage_ev[i + 1]));
  return k;
}

extern "C" int fmp_precond_restrict(fmp_precond* p, const fmp_block* blk, const double* r, double* out,
                                    void* stream) {
  FMP_REQUIRE(p && blk && r && out, "null argument");
  dim3 grid(p->max_ez, 3, (unsigned)p->d.n_sub);
  k_restrict<<<grid, 256, 0, as_stream(stream)>>>(p->d.subs, make_geo(blk), r, out);
  FMP_CHECK_LAUNCH();
  return 0;
}
