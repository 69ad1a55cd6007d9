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
#include <vector>
#include <cublas_v2.h>
#include "common.cuh"

namespace fmp {

__host__ __device__ constexpr int pad8(int n) { return (n + 7) & ~7; }
__host__ __device__ constexpr int pad4(int n) { return (n + 3) & ~3; }
// Row stride (doubles) for an operand with pad8(n) columns: == 4 (mod 8) so the
// DMMA fragment loads (8 rows x 4 cols per warp) hit 16 distinct 8-byte banks.
__host__ __device__ constexpr int sstride(int n) { return pad8(n) + 4; }

struct SubD {
  int ex, ey, ez, lx, ly, lz, ox, oy, oz, wx, wy, wz, shape, column;
  int64_t ws_off, in_off;
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
  return d;
}

// Forward factor of component c along axis a: U^T on the component's own axis, V^T on
// the other two (ref:transform.py:120-132).  Row-major n x n; inverse = transpose.
__device__ __forceinline__ const double* fwd_factor(const double* factors, const fmp_shape& sh, int c, int a) {
  return factors + (a == c ? sh.ut_off[a] : sh.vt_off[a]);
}

// C[m][n] = sum_k A(m,k) B(k,n) over 8x8 DMMA tiles distributed round-robin over warps.
// A(m,k) = a[m*sa + k] (or a[k*sa + m] if AT); B(k,n) = b[k*sb + n] (or b[n*sb + k] if BT).
template <bool AT, bool BT>
__device__ __forceinline__ void smem_gemm(const double* __restrict__ a, int sa, const double* __restrict__ b, int sb,
                                          double* __restrict__ c, int sc, int m8, int n8, int k4, int warp,
                                          int nwarps, int lane) {
  const int g = lane >> 2, t = lane & 3;
  for (int tile = warp; tile < m8 * n8; tile += nwarps) {
    const int mt = tile / n8, nt = tile - mt * n8;
    const int m = mt * 8 + g, n = nt * 8 + g;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < k4; ++kk) {
      const int k = kk * 4 + t;
      const double av = AT ? a[k * sa + m] : a[m * sa + k];
      const double bv = BT ? b[n * sb + k] : b[k * sb + n];
      dmma884(d0, d1, av, bv);
    }
    double* cp = c + (mt * 8 + g) * sc + nt * 8 + 2 * t;
    cp[0] = d0;
    cp[1] = d1;
  }
}

// ---------------------------------------------------------------- K1 / K4: plane passes
struct PlaneArgs {
  const fmp_subdomain* subs;
  const fmp_shape* shapes;
  const double* factors;
  Geo g;
  const double* src;
  double* dst;
  int mode;  // FMP_SOLVE_*
  int ppc;   // planes per CTA
};

// Load an n x n factor (row-major, rows r < n) into smem with stride s, zero padded to pad8.
__device__ __forceinline__ void load_factor(double* dst, int s, const double* __restrict__ f, int n) {
  const int P = pad8(n);
  for (int q = threadIdx.x; q < P * s; q += blockDim.x) {
    const int r = q / s, c = q - r * s;
    dst[q] = (r < n && c < n) ? __ldg(f + r * n + c) : 0.0;
  }
}

// Restriction S_i^gamma: point (c, k, j, i) of the extended box read from the block field,
// its ghost shell (neighbour GPUs) or the global zero ghost (ref:schwarz.py:237-250).
__device__ __forceinline__ double restrict_point(const Geo& g, const double* __restrict__ src, const SubD& d,
                                                 bool inside, int c, int k, int j, int i) {
  if (inside) return __ldg(src + fidx(g, c, d.lz + k, d.ly + j, d.lx + i));
  return fetch(g, src, c, d.lz + k, d.ly + j, d.lx + i);
}

__device__ __forceinline__ bool ext_inside(const Geo& g, const SubD& d) {
  return d.lx >= 0 && d.ly >= 0 && d.lz >= 0 && d.lx + d.ex <= g.bx && d.ly + d.ey <= g.by && d.lz + d.ez <= g.bz;
}

// Extended vectors of every subdomain, [c][k][j][i] at ws_off: the reference Exchanger's
// output (ref:schwarz.py:217-257), produced with the same addressing as K1.
__global__ void k_restrict(const fmp_subdomain* subs, Geo g, const double* __restrict__ src,
                           double* __restrict__ out) {
  const SubD d = load_sub(subs + blockIdx.z);
  const int c = blockIdx.y, k = blockIdx.x;
  if (k >= d.ez) return;
  const bool inside = ext_inside(g, d);
  const int64_t P = (int64_t)d.ex * d.ey;
  double* o = out + d.ws_off + (c * d.ez + k) * P;
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int r = q / d.ex, col = q - r * d.ex;
    o[q] = restrict_point(g, src, d, inside, c, k, r, col);
  }
}

// INV = false (K1): X = r restricted to plane k of the extended box; out = Fy X Fx^T -> work
// INV = true  (K4): X = work plane k; out = Fy^T X Fx; owned part -> block field z
template <bool INV>
__global__ void __launch_bounds__(128) k_plane(PlaneArgs A) {
  extern __shared__ double smem[];
  const SubD d = load_sub(A.subs + blockIdx.z);
  const fmp_shape sh = A.shapes[d.shape];
  const int c = blockIdx.y;
  const int nplanes = INV ? d.wz : d.ez;
  const int kbeg = blockIdx.x * A.ppc;
  if (kbeg >= nplanes) return;
  const int kend = min(kbeg + A.ppc, nplanes);
  const int ex = d.ex, ey = d.ey, PX = pad8(ex), PY = pad8(ey), SXs = sstride(ex), SYs = sstride(ey);
  double* sFx = smem;               // [PX][SXs]
  double* sFy = sFx + PX * SXs;     // [PY][SYs]
  double* sX = sFy + PY * SYs;      // [PY][SXs]
  double* sT = sX + PY * SXs;       // [PY][SXs]
  load_factor(sFx, SXs, fwd_factor(A.factors, sh, c, 0), ex);
  load_factor(sFy, SYs, fwd_factor(A.factors, sh, c, 1), ey);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t P = (int64_t)ex * ey;
  const int64_t V = P * d.ez;
  // source addressing
  const bool inside = ext_inside(A.g, d);
  for (int kk = kbeg; kk < kend; ++kk) {
    const int k = INV ? d.oz + kk : kk;
    // ---- load plane into sX (zero padded)
    for (int q = threadIdx.x; q < PY * SXs; q += blockDim.x) {
      const int r = q / SXs, col = q - r * SXs;
      double v = 0.0;
      if (r < ey && col < ex) {
        if (INV) {
          v = A.src[d.ws_off + (c * d.ez + k) * P + r * ex + col];
        } else if (A.mode == FMP_SOLVE_FACES) {
          v = A.src[d.in_off + c * V + k * P + r * ex + col];
        } else {
          v = restrict_point(A.g, A.src, d, inside, c, k, r, col);
        }
      }
      sX[q] = v;
    }
    __syncthreads();
    if (!INV) {
      // T[j][a] = sum_i X[j][i] Fx[a][i];   O[b][a] = sum_j Fy[b][j] T[j][a]
      smem_gemm<false, true>(sX, SXs, sFx, SXs, sT, SXs, PY / 8, PX / 8, pad4(ex) / 4, warp, nw, lane);
      __syncthreads();
      smem_gemm<false, false>(sFy, SYs, sT, SXs, sX, SXs, PY / 8, PX / 8, pad4(ey) / 4, warp, nw, lane);
    } else {
      // T[b][i] = sum_a X[b][a] Fx[a][i];   O[j][i] = sum_b Fy[b][j] T[b][i]
      smem_gemm<false, false>(sX, SXs, sFx, SXs, sT, SXs, PY / 8, PX / 8, pad4(ex) / 4, warp, nw, lane);
      __syncthreads();
      smem_gemm<true, false>(sFy, SYs, sT, SXs, sX, SXs, PY / 8, PX / 8, pad4(ey) / 4, warp, nw, lane);
    }
    __syncthreads();
    if (!INV) {
      double* out = A.dst + d.ws_off + (c * d.ez + k) * P;
      for (int q = threadIdx.x; q < P; q += blockDim.x) {
        const int r = q / ex, col = q - r * ex;
        out[q] = sX[r * SXs + col];
      }
    } else {
      for (int q = threadIdx.x; q < d.wy * d.wx; q += blockDim.x) {
        const int r = q / d.wx, col = q - r * d.wx;
        A.dst[fidx(A.g, c, d.lz + k, d.ly + d.oy + r, d.lx + d.ox + col)] = sX[(d.oy + r) * SXs + d.ox + col];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K2 / K3: column passes
constexpr int TP = 64;  // columns (flattened (j,i) plane positions) per CTA

struct ColArgs {
  const fmp_subdomain* subs;
  const fmp_shape* shapes;
  const double* factors;
  const double* src;
  double* dst;
  const double* corr;  // K3 only, may be null (no correction)
  int pmax;
  double alpha;
};

// B^-1 y at a transformed point with singular-value triplet s (ref:subdomain.py:145-153):
// B^-1 = q I + (1 - q) u u^T, q = 1/(1 + alpha |s|^2), u = s/|s|.
__device__ __forceinline__ void block_solve(double sx, double sy, double sz, double alpha, double& y0, double& y1,
                                            double& y2) {
  const double s2 = sx * sx + sy * sy + sz * sz;
  const double q = 1.0 / (1.0 + alpha * s2);
  const double proj = (1.0 - q) * (sx * y0 + sy * y1 + sz * y2) / s2;
  y0 = q * y0 + proj * sx;
  y1 = q * y1 + proj * sy;
  y2 = q * y2 + proj * sz;
}

// INV = false (K2): X[c][k][p] = work; y^ = B^-1 (Fz X) -> dst
// INV = true  (K3): X[c][k~][p] = y^ (minus the folded Woodbury term); out = Fz^T X -> dst
template <int MT, bool INV>
__global__ void __launch_bounds__(256) k_column(ColArgs A) {
  extern __shared__ double smem[];
  const SubD d = load_sub(A.subs + blockIdx.y);
  const fmp_shape sh = A.shapes[d.shape];
  const int ex = d.ex, ey = d.ey, ez = d.ez;
  const int P = ex * ey;
  const int p0 = blockIdx.x * TP;
  if (p0 >= P) return;
  const int PZ = pad8(ez), SZs = sstride(ez), SC = TP + 4;
  double* sX = smem;                   // [3][PZ][SC]
  double* sF = sX + 3 * PZ * SC;       // [2][PZ][SZs]: V^T_z (components x, y), U^T_z (component z)
  load_factor(sF, SZs, A.factors + sh.vt_off[2], ez);
  load_factor(sF + PZ * SZs, SZs, A.factors + sh.ut_off[2], ez);
  const int64_t V = (int64_t)P * ez;
  const double* src = A.src + d.ws_off;
  for (int q = threadIdx.x; q < 3 * PZ * SC; q += blockDim.x) {
    const int cc = q / (PZ * SC), rem = q - cc * PZ * SC, r = rem / SC, col = rem - r * SC;
    double v = 0.0;
    if (r < ez && col < TP && p0 + col < P) v = src[cc * V + (int64_t)r * P + p0 + col];
    sX[q] = v;
  }
  const double* Sx = A.factors + sh.s_off[0];
  const double* Sy = A.factors + sh.s_off[1];
  const double* Sz = A.factors + sh.s_off[2];
  __syncthreads();
  if (INV && A.corr) {
    // y^ -= B^-1 (G Q Z): per component two rank-structured face terms (see K6)
    const double* cb = A.corr + (int64_t)blockIdx.y * 6 * A.pmax * A.pmax;
    const int pm = A.pmax, pm2 = pm * pm;
    const double* Fx0 = A.factors + sh.ut_off[0];  // comp x on axis x uses U^T, others V^T
    const double* Vx = A.factors + sh.vt_off[0];
    const double* Uy = A.factors + sh.ut_off[1];
    const double* Vy = A.factors + sh.vt_off[1];
    const double* Uz = A.factors + sh.ut_off[2];
    const double* Vz = A.factors + sh.vt_off[2];
    (void)Fx0;
    for (int q = threadIdx.x; q < ez * TP; q += blockDim.x) {
      const int cz = q / TP, col = q - cz * TP;
      const int p = p0 + col;
      if (p >= P) continue;
      const int b = p / ex, a = p - b * ex;
      // comp x: Fz=V_z, Fy=V_y:  Fz[cz][0] * G_x[b][a] + Fy[b][0] * F_x[cz][a]
      double dx = Vz[cz * ez] * cb[0 * pm2 + b * pm + a] + Vy[b * ey] * cb[1 * pm2 + cz * pm + a];
      // comp y: Fz=V_z, Fx=V_x:  Fz[cz][0] * G_y[b][a] + Fx[a][0] * F_y[cz][b]
      double dy = Vz[cz * ez] * cb[2 * pm2 + b * pm + a] + Vx[a * ex] * cb[3 * pm2 + cz * pm + b];
      // comp z: Fy=V_y, Fx=V_x:  Fy[b][0] * G_z[cz][a] + Fx[a][0] * F_z[cz][b]
      double dz = Vy[b * ey] * cb[4 * pm2 + cz * pm + a] + Vx[a * ex] * cb[5 * pm2 + cz * pm + b];
      (void)Uy; (void)Uz;
      block_solve(Sx[a], Sy[b], Sz[cz], A.alpha, dx, dy, dz);
      sX[(0 * PZ + cz) * SC + col] -= dx;
      sX[(1 * PZ + cz) * SC + col] -= dy;
      sX[(2 * PZ + cz) * SC + col] -= dz;
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int nt = warp;  // 8 warps x 8 columns = TP
  const int m8 = PZ / 8, k4 = pad4(ez) / 4;
  double acc[3][MT][2];
#pragma unroll
  for (int cc = 0; cc < 3; ++cc)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[cc][mt][0] = acc[cc][mt][1] = 0.0;
  const double* Fv = sF;
  const double* Fu = sF + PZ * SZs;
  for (int kk = 0; kk < k4; ++kk) {
    const int k = kk * 4 + t;
    const double b0 = sX[(0 * PZ + k) * SC + nt * 8 + g];
    const double b1 = sX[(1 * PZ + k) * SC + nt * 8 + g];
    const double b2 = sX[(2 * PZ + k) * SC + nt * 8 + g];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt < m8) {
        const int m = mt * 8 + g;
        const double av = INV ? Fv[k * SZs + m] : Fv[m * SZs + k];
        const double au = INV ? Fu[k * SZs + m] : Fu[m * SZs + k];
        dmma884(acc[0][mt][0], acc[0][mt][1], av, b0);
        dmma884(acc[1][mt][0], acc[1][mt][1], av, b1);
        dmma884(acc[2][mt][0], acc[2][mt][1], au, b2);
      }
    }
  }
  if (!INV) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt < m8) {
        const int cz = mt * 8 + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int p = p0 + nt * 8 + 2 * t + h;
          if (cz < ez && p < P) {
            const int b = p / ex, a = p - b * ex;
            block_solve(Sx[a], Sy[b], Sz[cz], A.alpha, acc[0][mt][h], acc[1][mt][h], acc[2][mt][h]);
          }
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int cc = 0; cc < 3; ++cc)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
      if (mt < m8) {
        double* o = sX + (cc * PZ + mt * 8 + g) * SC + nt * 8 + 2 * t;
        o[0] = acc[cc][mt][0];
        o[1] = acc[cc][mt][1];
      }
  __syncthreads();
  double* dst = A.dst + d.ws_off;
  const int ncol = min(TP, P - p0);
  for (int q = threadIdx.x; q < 3 * ez * TP; q += blockDim.x) {
    const int cc = q / (ez * TP), rem = q - cc * ez * TP, r = rem / TP, col = rem - r * TP;
    if (col < ncol) dst[cc * V + (int64_t)r * P + p0 + col] = sX[(cc * PZ + r) * SC + col];
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
};

__device__ __forceinline__ int ext_of(const SubD& d, int a) { return a == 0 ? d.ex : (a == 1 ? d.ey : d.ez); }

// K5: Y[:, col] = e0 on the two faces per component, e0 = G^-1 y^ evaluated only there.
// Projection along the face normal with weights F_n[t][0] (inverse factor row 0), then
// a 2-D inverse transform over the in-plane axes.
__global__ void __launch_bounds__(256) k_faces(FaceArgs A) {
  extern __shared__ double smem[];
  const SubD d = load_sub(A.subs + blockIdx.y);
  const fmp_shape sh = A.shapes[d.shape];
  const int c = blockIdx.x;
  const int ex = d.ex, ey = d.ey, ez = d.ez, P = ex * ey;
  const int pm = A.pmax, pm2 = pm * pm;
  double* sPlane = smem;          // [ey][ex]
  double* sA = sPlane + pm2;      // primary projection   [u1][v1] (transformed indices)
  double* sB = sA + pm2;          // secondary projection [u2][v2]
  double* sT = sB + pm2;          // temp
  const FaceGeo fg = face_geo(c);
  const double* wn1 = fwd_factor(A.factors, sh, c, fg.n1);
  const double* wn2 = fwd_factor(A.factors, sh, c, fg.n2);
  const int nn1 = ext_of(d, fg.n1), nn2 = ext_of(d, fg.n2);
  const double* src = A.yhat + d.ws_off + (int64_t)c * P * ez;
  for (int q = threadIdx.x; q < pm2; q += blockDim.x) sA[q] = 0.0;
  for (int cz = 0; cz < ez; ++cz) {
    __syncthreads();
    for (int q = threadIdx.x; q < P; q += blockDim.x) sPlane[q] = src[(int64_t)cz * P + q];
    __syncthreads();
    // primary face
    if (fg.n1 == 2) {  // z-normal: sA[b][a] += w[cz] * plane[b][a]
      const double w = __ldg(wn1 + cz * nn1);
      for (int q = threadIdx.x; q < P; q += blockDim.x) sA[(q / ex) * pm + q % ex] += w * sPlane[q];
    } else {  // c = z: y-normal: sA[cz][a] = sum_b w[b] plane[b][a]
      for (int a = threadIdx.x; a < ex; a += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < ey; ++b) s += __ldg(wn1 + b * nn1) * sPlane[b * ex + a];
        sA[cz * pm + a] = s;
      }
    }
    // secondary face
    if (fg.n2 == 1) {  // c = x: y-normal: sB[cz][a] = sum_b w[b] plane[b][a]
      for (int a = threadIdx.x; a < ex; a += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < ey; ++b) s += __ldg(wn2 + b * nn2) * sPlane[b * ex + a];
        sB[cz * pm + a] = s;
      }
    } else {  // x-normal: sB[cz][b] = sum_a w[a] plane[b][a]
      for (int b = threadIdx.x; b < ey; b += blockDim.x) {
        double s = 0.0;
        for (int a = 0; a < ex; ++a) s += __ldg(wn2 + a * nn2) * sPlane[b * ex + a];
        sB[cz * pm + b] = s;
      }
    }
  }
  __syncthreads();
  // 2-D inverse transforms: E[u][v] = sum_tu Fu[tu][u] sum_tv Fv[tv][v] Proj[tu][tv]
  double* Y = A.ymat[d.shape] + (int64_t)d.column * sh.m;
  int base = 0;
  for (int q = 0; q < c; ++q) base += (int)sh.m_comp[q];
  for (int f = 0; f < 2; ++f) {
    const int ua = f == 0 ? fg.u1 : fg.u2, va = f == 0 ? fg.v1 : fg.v2;
    const int nu = ext_of(d, ua), nv = ext_of(d, va);
    const double* Fu = fwd_factor(A.factors, sh, c, ua);
    const double* Fv = fwd_factor(A.factors, sh, c, va);
    const double* Pj = f == 0 ? sA : sB;
    for (int q = threadIdx.x; q < nu * nv; q += blockDim.x) {  // T[tu][v] = sum_tv Pj[tu][tv] Fv[tv][v]
      const int tu = q / nv, v = q - tu * nv;
      double s = 0.0;
      for (int tv = 0; tv < nv; ++tv) s += Pj[tu * pm + tv] * __ldg(Fv + tv * nv + v);
      sT[tu * pm + v] = s;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nu * nv; q += blockDim.x) {  // E[u][v] = sum_tu Fu[tu][u] T[tu][v]
      const int u = q / nv, v = q - u * nv;
      const int row = face_row(c, f, u, v, ex, ey);
      if (row < 0) continue;
      double s = 0.0;
      for (int tu = 0; tu < nu; ++tu) s += __ldg(Fu + tu * nu + u) * sT[tu * pm + v];
      Y[base + row] = s;
    }
    __syncthreads();
  }
}

// K6: from Z (C^-1 Y) build, per component and face, the forward-transformed face plane
// Proj[tu][tv] = sum_{u,v} Fu[tu][u] Fv[tv][v] Zface[u][v]  -> corr planes (see K3).
__global__ void __launch_bounds__(256) k_corr(FaceArgs A) {
  extern __shared__ double smem[];
  const SubD d = load_sub(A.subs + blockIdx.y);
  const fmp_shape sh = A.shapes[d.shape];
  const int c = blockIdx.x;
  const int ex = d.ex, ey = d.ey;
  const int pm = A.pmax, pm2 = pm * pm;
  double* sZ = smem;       // [u][v]
  double* sT = sZ + pm2;   // [u][tv]
  const FaceGeo fg = face_geo(c);
  const double* Z = A.zmat[d.shape] + (int64_t)d.column * sh.m;
  int base = 0;
  for (int q = 0; q < c; ++q) base += (int)sh.m_comp[q];
  for (int f = 0; f < 2; ++f) {
    const int ua = f == 0 ? fg.u1 : fg.u2, va = f == 0 ? fg.v1 : fg.v2;
    const int nu = ext_of(d, ua), nv = ext_of(d, va);
    const double* Fu = fwd_factor(A.factors, sh, c, ua);
    const double* Fv = fwd_factor(A.factors, sh, c, va);
    for (int q = threadIdx.x; q < nu * nv; q += blockDim.x) {
      const int u = q / nv, v = q - u * nv;
      const int row = face_row(c, f, u, v, ex, ey);
      sZ[u * pm + v] = row < 0 ? 0.0 : Z[base + row];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nu * nv; q += blockDim.x) {  // T[u][tv] = sum_v Z[u][v] Fv[tv][v]
      const int u = q / nv, tv = q - u * nv;
      double s = 0.0;
      for (int v = 0; v < nv; ++v) s += sZ[u * pm + v] * __ldg(Fv + tv * nv + v);
      sT[u * pm + tv] = s;
    }
    __syncthreads();
    double* out = A.corr + ((int64_t)blockIdx.y * 6 + c * 2 + f) * pm2;
    for (int q = threadIdx.x; q < nu * nv; q += blockDim.x) {  // Proj[tu][tv] = sum_u Fu[tu][u] T[u][tv]
      const int tu = q / nv, tv = q - tu * nv;
      double s = 0.0;
      for (int u = 0; u < nu; ++u) s += __ldg(Fu + tu * nu + u) * sT[u * pm + tv];
      out[tu * pm + tv] = s;
    }
    __syncthreads();
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
  cublasHandle_t blas = nullptr;
  int max_ex = 1, max_ey = 1, max_ez = 1, max_p = 1, max_wz = 1;
};

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
  for (const auto& s : p->subs) {
    p->max_ex = std::max<int>(p->max_ex, (int)s.ext[0]);
    p->max_ey = std::max<int>(p->max_ey, (int)s.ext[1]);
    p->max_ez = std::max<int>(p->max_ez, (int)s.ext[2]);
    p->max_p = std::max<int>(p->max_p, (int)(s.ext[0] * s.ext[1]));
    p->max_wz = std::max<int>(p->max_wz, (int)s.own[2]);
  }
  const int mx = std::max(p->max_ex, std::max(p->max_ey, p->max_ez));
  if (mx > 72 || mx > desc->pmax) {
    delete p;
    FMP_REQUIRE(false, "extended extent %d exceeds the supported maximum 72 (or pmax %lld)", mx,
                (long long)desc->pmax);
  }
  if (cudaMalloc(&p->d_ymat, sizeof(double*) * desc->n_shape) != cudaSuccess ||
      cudaMalloc(&p->d_zmat, sizeof(double*) * desc->n_shape) != cudaSuccess) {
    delete p;
    FMP_REQUIRE(false, "cudaMalloc of pointer tables failed");
  }
  cudaMemcpy(p->d_ymat, p->ymat.data(), sizeof(double*) * desc->n_shape, cudaMemcpyHostToDevice);
  cudaMemcpy(p->d_zmat, p->zmat.data(), sizeof(double*) * desc->n_shape, cudaMemcpyHostToDevice);
  if (cublasCreate(&p->blas) != CUBLAS_STATUS_SUCCESS) {
    cudaFree(p->d_ymat);
    cudaFree(p->d_zmat);
    delete p;
    FMP_REQUIRE(false, "cublasCreate failed");
  }
  cublasSetMathMode(p->blas, CUBLAS_DEFAULT_MATH);
  // shared-memory opt-in for the largest configuration we may launch
  cudaFuncSetAttribute(k_plane<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_plane<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_faces, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_corr, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  *out = p;
  return 0;
}

extern "C" int fmp_precond_destroy(fmp_precond* p) {
  if (!p) return 0;
  if (p->blas) cublasDestroy(p->blas);
  cudaFree(p->d_ymat);
  cudaFree(p->d_zmat);
  delete p;
  return 0;
}

template <int MT>
static int launch_column(bool inv, dim3 grid, size_t smem, cudaStream_t st, const ColArgs& a) {
  if (inv) {
    cudaFuncSetAttribute(k_column<MT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_column<MT, true><<<grid, 256, smem, st>>>(a);
  } else {
    cudaFuncSetAttribute(k_column<MT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_column<MT, false><<<grid, 256, smem, st>>>(a);
  }
  FMP_CHECK_LAUNCH();
  return 0;
}

static int column_pass(fmp_precond* p, bool inv, const double* src, double* dst, const double* corr,
                       cudaStream_t st) {
  ColArgs a{p->d.subs, p->d.shapes, p->d.factors, src, dst, corr, (int)p->d.pmax, p->d.alpha};
  const int PZ = pad8(p->max_ez);
  const size_t smem = (size_t)(3 * PZ * (TP + 4) + 2 * PZ * sstride(p->max_ez)) * sizeof(double);
  dim3 grid((p->max_p + TP - 1) / TP, (unsigned)p->d.n_sub);
  switch (PZ / 8) {
    case 1: return launch_column<1>(inv, grid, smem, st, a);
    case 2: return launch_column<2>(inv, grid, smem, st, a);
    case 3: return launch_column<3>(inv, grid, smem, st, a);
    case 4: return launch_column<4>(inv, grid, smem, st, a);
    case 5: return launch_column<5>(inv, grid, smem, st, a);
    case 6: return launch_column<6>(inv, grid, smem, st, a);
    case 7: return launch_column<7>(inv, grid, smem, st, a);
    case 8: return launch_column<8>(inv, grid, smem, st, a);
    case 9: return launch_column<9>(inv, grid, smem, st, a);
  }
  FMP_REQUIRE(false, "unsupported z extent");
}

static int plane_pass(fmp_precond* p, const fmp_block* blk, bool inv, int mode, const double* src, double* dst,
                      cudaStream_t st) {
  PlaneArgs a;
  a.subs = p->d.subs;
  a.shapes = p->d.shapes;
  a.factors = p->d.factors;
  a.g = make_geo(blk);
  a.src = src;
  a.dst = dst;
  a.mode = mode;
  a.ppc = 2;
  const int PX = pad8(p->max_ex), PY = pad8(p->max_ey);
  const size_t smem =
      (size_t)(PX * sstride(p->max_ex) + PY * sstride(p->max_ey) + 2 * PY * sstride(p->max_ex)) * sizeof(double);
  const int planes = inv ? p->max_wz : p->max_ez;
  dim3 grid((planes + a.ppc - 1) / a.ppc, 3, (unsigned)p->d.n_sub);
  if (inv)
    k_plane<true><<<grid, 128, smem, st>>>(a);
  else
    k_plane<false><<<grid, 128, smem, st>>>(a);
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_precond_apply(fmp_precond* p, const fmp_block* blk, int mode, const double* r, double* z,
                                 void* stream) {
  FMP_REQUIRE(p && blk, "null argument");
  FMP_REQUIRE(mode >= FMP_SOLVE_WOODBURY && mode <= FMP_SOLVE_FACES, "bad solve mode %d", mode);
  cudaStream_t st = as_stream(stream);
  double* wa = p->d.work_a;
  double* wb = p->d.work_b;
  if (int e = plane_pass(p, blk, false, mode, r, wa, st)) return e;
  if (int e = column_pass(p, false, wa, wb, nullptr, st)) return e;
  const int pm = (int)p->d.pmax;
  FaceArgs fa{p->d.subs, p->d.shapes, p->d.factors, wb, p->d.corr, p->d_ymat, p->d_zmat, pm};
  if (mode != FMP_SOLVE_EXACT) {
    k_faces<<<dim3(3, (unsigned)p->d.n_sub), 256, 4 * pm * pm * sizeof(double), st>>>(fa);
    FMP_CHECK_LAUNCH();
  }
  if (mode == FMP_SOLVE_FACES) return 0;
  if (mode == FMP_SOLVE_WOODBURY) {
    cublasSetStream(p->blas, st);
    const double one = 1.0, zero = 0.0;
    for (int64_t s = 0; s < p->d.n_shape; ++s) {
      const int m = (int)p->shapes[s].m;
      const int ncol = (int)(p->first[s + 1] - p->first[s]);
      if (ncol == 0) continue;
      // C^-1 is stored row-major (the reference's ndarray); OP_T makes cuBLAS use it as is.
      cublasStatus_t bs = cublasDgemm(p->blas, CUBLAS_OP_T, CUBLAS_OP_N, m, ncol, m, &one, p->cinv[s], m,
                                      p->ymat[s], m, &zero, p->zmat[s], m);
      FMP_REQUIRE(bs == CUBLAS_STATUS_SUCCESS, "cublasDgemm failed (%d)", (int)bs);
    }
    k_corr<<<dim3(3, (unsigned)p->d.n_sub), 256, 2 * pm * pm * sizeof(double), st>>>(fa);
    FMP_CHECK_LAUNCH();
  }
  if (int e = column_pass(p, true, wb, wa, mode == FMP_SOLVE_WOODBURY ? p->d.corr : nullptr, st)) return e;
  return plane_pass(p, blk, true, mode, wa, z, st);
}

extern "C" int fmp_precond_restrict(fmp_precond* p, const fmp_block* blk, const double* r, double* out,
                                    void* stream) {
  FMP_REQUIRE(p && blk && r && out, "null argument");
  dim3 grid(p->max_ez, 3, (unsigned)p->d.n_sub);
  k_restrict<<<grid, 256, 0, as_stream(stream)>>>(p->d.subs, make_geo(blk), r, out);
  FMP_CHECK_LAUNCH();
  return 0;
}
