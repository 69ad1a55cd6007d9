// Matrix-free double-curl stencils (K7, K13).
//
// A = I + alpha (C_b C_f + Lambda) equals I + alpha C_b C_f evaluated on the box padded
// with one layer of zeros, with the intermediate curl also evaluated on the low ghost
// layer (checked against ref:operators.py:167-175 and
// the CSR of ref:operators.py:201-238 in tests/test_stencil_gpu.py).  So the kernel
// needs no Lambda branch: the zero ghost (global boundary) or the neighbour ghost
// (GPU-block faces, fmp_block) is all it reads.  with_boundary=False subtracts
// alpha*Lambda*x explicitly.
//
// Roofline: HBM-bound, 48 B per owned point (read x: 24 B, write y: 24 B);
// mode 3 (true residual) reads x and b (48 B) and writes nothing.
#include "common.cuh"

namespace fmp {


template <bool GEN>
struct Loader {
  const Geo& g;
  const double* __restrict__ f;
  __device__ __forceinline__ double operator()(int c, int k, int j, int i) const {
    if (GEN) return fetch(g, f, c, k, j, i);
    return __ldg(f + fidx(g, c, k, j, i));
  }
};

// The 13-point bracket of Appendix A: (C_b C_f + Lambda) x at (i,j,k) for all components.
template <bool GEN>
__device__ __forceinline__ void bracket(const Loader<GEN>& L, int k, int j, int i, double& tx, double& ty,
                                        double& tz, double& ex, double& ey, double& ez) {
  ex = L(0, k, j, i);
  ey = L(1, k, j, i);
  ez = L(2, k, j, i);
  const double ex_jm = L(0, k, j - 1, i), ex_jp = L(0, k, j + 1, i);
  const double ex_km = L(0, k - 1, j, i), ex_kp = L(0, k + 1, j, i);
  const double ex_im = L(0, k, j, i - 1), ex_im_jp = L(0, k, j + 1, i - 1), ex_im_kp = L(0, k + 1, j, i - 1);
  const double ey_ip = L(1, k, j, i + 1), ey_im = L(1, k, j, i - 1);
  const double ey_km = L(1, k - 1, j, i), ey_kp = L(1, k + 1, j, i);
  const double ey_jm = L(1, k, j - 1, i), ey_ip_jm = L(1, k, j - 1, i + 1), ey_jm_kp = L(1, k + 1, j - 1, i);
  const double ez_ip = L(2, k, j, i + 1), ez_im = L(2, k, j, i - 1);
  const double ez_jp = L(2, k, j + 1, i), ez_jm = L(2, k, j - 1, i);
  const double ez_km = L(2, k - 1, j, i), ez_ip_km = L(2, k - 1, j, i + 1), ez_jp_km = L(2, k - 1, j + 1, i);
  tx = 4.0 * ex - ex_jm - ex_jp - ex_km - ex_kp + ey_ip - ey - ey_ip_jm + ey_jm + ez_ip - ez - ez_ip_km + ez_km;
  ty = 4.0 * ey - ey_im - ey_ip - ey_km - ey_kp + ez_jp - ez - ez_jp_km + ez_km + ex_jp - ex - ex_im_jp + ex_im;
  tz = 4.0 * ez - ez_im - ez_ip - ez_jm - ez_jp + ex_kp - ex - ex_im_kp + ex_im + ey_kp - ey - ey_jm_kp + ey_jm;
}

// ---------------------------------------------------------------- SpMV: 2.5-D blocked z-march
// A CTA owns a 32 x 8 (x, y) column tile and marches a z-range.  Planes k-1, k, k+1 of all
// three components (tile + 1-cell halo) sit in a 4-slot shared-memory ring; plane k+2 streams
// in with cp.async while plane k is computed, so every x value is read from HBM about once
// (halo rows/columns come from L2) and the 25 neighbour reads per point hit shared memory.
constexpr int TX = 32, TY = 8;                         // column tile
constexpr int HX = TX + 2, HY = TY + 2, PLANE = HX * HY;  // haloed plane (per component)
constexpr int NSLOT = 5;   // planes k-1, k, k+1 in use, k+2 and k+3 in flight

__device__ __forceinline__ void spmv_issue_plane(const Geo& g, const double* __restrict__ x, double* slot, int i0,
                                                 int j0, int k) {
  for (int q = threadIdx.x; q < 3 * PLANE; q += TX * TY) {
    const int c = q / PLANE, rem = q - c * PLANE, r = rem / HX, col = rem - r * HX;
    cp_async8(slot + q, point_ptr(g, x, c, k, j0 - 1 + r, i0 - 1 + col), x);
  }
}

// Work is split in "plane units" (one z-plane of one column tile): CTA b takes the contiguous
// unit range [b*U/G, (b+1)*U/G) -- whole tiles or pieces of at most two -- so the grid is an
// exact multiple of the SM count with no partial last wave.
template <int MODE>
__global__ void __launch_bounds__(TX* TY) k_spmv(Geo g, double alpha, int bnd, const double* __restrict__ x,
                                                  double* __restrict__ y, const double* __restrict__ w,
                                                  double* __restrict__ partials, int tiles_x, int tiles_y) {
  __shared__ __align__(16) double ring[NSLOT][3 * PLANE];
  __shared__ double red[TX * TY / 32];
  const int tid = threadIdx.x, lx = tid % TX, ly = tid / TX;
  double acc0 = 0.0, acc1 = 0.0;
  const int64_t V = (int64_t)g.bx * g.by * g.bz;
  const int64_t units = (int64_t)tiles_x * tiles_y * g.bz;
  const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
  for (int64_t u = u0; u < u1;) {
    const int tile = (int)(u / g.bz);
    const int k0 = (int)(u - (int64_t)tile * g.bz);
    const int64_t left = u1 - u;
    const int k1 = (int)(k0 + left < g.bz ? k0 + left : g.bz);
    u += k1 - k0;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int i0 = tx * TX, j0 = ty * TY;
    const int i = i0 + lx, j = j0 + ly;
    const bool active = i < g.bx && j < g.by;
    const int gi = g.gx0 + i, gj = g.gy0 + j;
    __syncthreads();   // ring reuse across segments
    for (int kk = k0 - 1; kk <= k0 + 2; ++kk) {   // one commit group per plane
      if (kk <= k1) spmv_issue_plane(g, x, ring[(kk - k0 + 1) % NSLOT], i0, j0, kk);
      cp_async_commit();
    }
    for (int k = k0; k < k1; ++k) {
      cp_async_wait<1>();   // planes up to k+1 landed (k+2 may still be in flight)
      __syncthreads();      // ... for everyone; slot of k-2 is free
      if (k + 3 <= k1) spmv_issue_plane(g, x, ring[(k + 3 - k0 + 1) % NSLOT], i0, j0, k + 3);
      cp_async_commit();
      if (!active) continue;
      const double* pm = ring[(k - 1 - k0 + 1) % NSLOT];
      const double* p0 = ring[(k - k0 + 1) % NSLOT];
      const double* pp = ring[(k + 1 - k0 + 1) % NSLOT];
      const int o = (ly + 1) * HX + lx + 1;
#define EX(P, dj, di) P[0 * PLANE + o + (dj) * HX + (di)]
#define EY(P, dj, di) P[1 * PLANE + o + (dj) * HX + (di)]
#define EZ(P, dj, di) P[2 * PLANE + o + (dj) * HX + (di)]
      const double ex = EX(p0, 0, 0), ey = EY(p0, 0, 0), ez = EZ(p0, 0, 0);
      // Appendix A: (C_b C_f + Lambda) x on the zero-ghost padded box
      double tx = 4.0 * ex - EX(p0, -1, 0) - EX(p0, 1, 0) - EX(pm, 0, 0) - EX(pp, 0, 0) + EY(p0, 0, 1) - ey -
                  EY(p0, -1, 1) + EY(p0, -1, 0) + EZ(p0, 0, 1) - ez - EZ(pm, 0, 1) + EZ(pm, 0, 0);
      double ty = 4.0 * ey - EY(p0, 0, -1) - EY(p0, 0, 1) - EY(pm, 0, 0) - EY(pp, 0, 0) + EZ(p0, 1, 0) - ez -
                  EZ(pm, 1, 0) + EZ(pm, 0, 0) + EX(p0, 1, 0) - ex - EX(p0, 1, -1) + EX(p0, 0, -1);
      double tz = 4.0 * ez - EZ(p0, 0, -1) - EZ(p0, 0, 1) - EZ(p0, -1, 0) - EZ(p0, 1, 0) + EX(pp, 0, 0) - ex -
                  EX(pp, 0, -1) + EX(p0, 0, -1) + EY(pp, 0, 0) - ey - EY(pp, -1, 0) + EY(p0, -1, 0);
#undef EX
#undef EY
#undef EZ
      if (!bnd) {
        const int gk = g.gz0 + k;
        tx -= ((gj == 0) + (gk == 0)) * ex;
        ty -= ((gi == 0) + (gk == 0)) * ey;
        tz -= ((gi == 0) + (gj == 0)) * ez;
      }
      const double yx = ex + alpha * tx, yy = ey + alpha * ty, yz = ez + alpha * tz;
      const int64_t oi = fidx(g, 0, k, j, i);
      if (MODE == 3) {
        const double rx = w[oi] - yx, ry = w[oi + V] - yy, rz = w[oi + 2 * V] - yz;
        acc0 += rx * rx + ry * ry + rz * rz;
      } else {
        y[oi] = yx;
        y[oi + V] = yy;
        y[oi + 2 * V] = yz;
        if (MODE >= 1) acc0 += yx * w[oi] + yy * w[oi + V] + yz * w[oi + 2 * V];
        if (MODE == 2) acc1 += yx * yx + yy * yy + yz * yz;
      }
    }
    cp_async_wait<0>();
  }
  if (MODE >= 1) {
    const double s0 = block_sum<TX * TY>(acc0, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s0;
    if (MODE == 2) {
      const double s1 = block_sum<TX * TY>(acc1, red);
      if (threadIdx.x == 0) partials[gridDim.x + blockIdx.x] = s1;
    }
  }
}

// ---------------------------------------------------------------- curls and CN stencils
template <int KIND>  // 0 forward, 1 backward
__device__ __forceinline__ void curl_at(const Geo& g, const double* __restrict__ f, int k, int j, int i, double& cx,
                                        double& cy, double& cz) {
  if (KIND == 0) {  // D^f u(i) = u(i+1) - u(i), zero beyond the high face (ref:operators.py:94-96)
    const double ex = fetch(g, f, 0, k, j, i), ey = fetch(g, f, 1, k, j, i), ez = fetch(g, f, 2, k, j, i);
    cx = (fetch(g, f, 2, k, j + 1, i) - ez) - (fetch(g, f, 1, k + 1, j, i) - ey);
    cy = (fetch(g, f, 0, k + 1, j, i) - ex) - (fetch(g, f, 2, k, j, i + 1) - ez);
    cz = (fetch(g, f, 1, k, j, i + 1) - ey) - (fetch(g, f, 0, k, j + 1, i) - ex);
  } else {  // D^b u(i) = u(i) - u(i-1), zero before the low face (ref:operators.py:97-99)
    const double ex = fetch(g, f, 0, k, j, i), ey = fetch(g, f, 1, k, j, i), ez = fetch(g, f, 2, k, j, i);
    cx = (ez - fetch(g, f, 2, k, j - 1, i)) - (ey - fetch(g, f, 1, k - 1, j, i));
    cy = (ex - fetch(g, f, 0, k - 1, j, i)) - (ez - fetch(g, f, 2, k, j, i - 1));
    cz = (ey - fetch(g, f, 1, k, j, i - 1)) - (ex - fetch(g, f, 0, k, j - 1, i));
  }
}

template <int KIND>
__global__ void k_curl(Geo g, const double* __restrict__ f, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= g.bx) return;
  double cx, cy, cz;
  curl_at<KIND>(g, f, k, j, i, cx, cy, cz);
  const int64_t o = fidx(g, 0, k, j, i), V = (int64_t)g.bx * g.by * g.bz;
  out[o] = cx;
  out[o + V] = cy;
  out[o + 2 * V] = cz;
}

// R = E + dt*curl_b(H) - alpha*(C_b C_f E), alpha = dt^2/4  (ref:cn_driver.py:54-59)
__global__ void k_cn_rhs(Geo gE, Geo gH, double dt, const double* __restrict__ E, const double* __restrict__ H,
                         double* __restrict__ R) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= gE.bx) return;
  const double alpha = dt * dt / 4.0;
  double hx, hy, hz;
  curl_at<1>(gH, H, k, j, i, hx, hy, hz);
  const Loader<true> L{gE, E};
  double tx, ty, tz, ex, ey, ez;
  bracket<true>(L, k, j, i, tx, ty, tz, ex, ey, ez);
  const int gi = gE.gx0 + i, gj = gE.gy0 + j, gk = gE.gz0 + k;
  tx -= ((gj == 0) + (gk == 0)) * ex;  // C_b C_f without Lambda
  ty -= ((gi == 0) + (gk == 0)) * ey;
  tz -= ((gi == 0) + (gj == 0)) * ez;
  const int64_t o = fidx(gE, 0, k, j, i), V = (int64_t)gE.bx * gE.by * gE.bz;
  R[o] = (ex + dt * hx) - alpha * tx;
  R[o + V] = (ey + dt * hy) - alpha * ty;
  R[o + 2 * V] = (ez + dt * hz) - alpha * tz;
}

// H_new = H - (0.5 dt) (curl_f(E_new) + curl_f(E_old))  (ref:cn_driver.py:90-91)
__global__ void k_cn_h(Geo gN, Geo gO, double hdt, const double* __restrict__ H, const double* __restrict__ En,
                       const double* __restrict__ Eo, double* __restrict__ Hn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= gN.bx) return;
  double ax, ay, az, bx, by, bz;
  curl_at<0>(gN, En, k, j, i, ax, ay, az);
  curl_at<0>(gO, Eo, k, j, i, bx, by, bz);
  const int64_t o = fidx(gN, 0, k, j, i), V = (int64_t)gN.bx * gN.by * gN.bz;
  Hn[o] = H[o] - hdt * (ax + bx);
  Hn[o + V] = H[o + V] - hdt * (ay + by);
  Hn[o + 2 * V] = H[o + 2 * V] - hdt * (az + bz);
}

}  // namespace fmp

using namespace fmp;

static int check_block(const fmp_block* b) {
  FMP_REQUIRE(b && b->bx >= 1 && b->by >= 1 && b->bz >= 1, "invalid block extents");
  FMP_REQUIRE(b->gx0 >= 0 && b->gy0 >= 0 && b->gz0 >= 0 && b->gx0 + b->bx <= b->nx && b->gy0 + b->by <= b->ny &&
                  b->gz0 + b->bz <= b->nz,
              "block outside the global box");
  FMP_REQUIRE(b->bx * b->by <= (int64_t)1 << 31, "block plane too large");
  return 0;
}

extern "C" int fmp_stencil_apply(const fmp_block* blk, double alpha, int boundary, int mode, const double* x,
                                 double* y, const double* w, double* dots, double* scratch, void* stream) {
  if (int e = check_block(blk)) return e;
  FMP_REQUIRE(mode >= 0 && mode <= 3, "bad stencil mode %d", mode);
  FMP_REQUIRE(mode == 0 || (w && dots && scratch), "mode %d needs w, dots and scratch", mode);
  const Geo g = make_geo(blk);
  const int tx = (g.bx + TX - 1) / TX, ty = (g.by + TY - 1) / TY;
  const int64_t units = (int64_t)tx * ty * g.bz;
  // one full wave: SMs x resident CTAs (smem-limited to 5 of 41 KB), fewer for tiny blocks
  const int64_t want = (int64_t)kNumSM * 5;
  const int grid = (int)(units / 8 < want ? (units / 8 > 0 ? units / 8 : 1) : want);
  cudaStream_t st = as_stream(stream);
  switch (mode) {
    case 0: k_spmv<0><<<grid, TX * TY, 0, st>>>(g, alpha, boundary, x, y, w, scratch, tx, ty); break;
    case 1: k_spmv<1><<<grid, TX * TY, 0, st>>>(g, alpha, boundary, x, y, w, scratch, tx, ty); break;
    case 2: k_spmv<2><<<grid, TX * TY, 0, st>>>(g, alpha, boundary, x, y, w, scratch, tx, ty); break;
    case 3: k_spmv<3><<<grid, TX * TY, 0, st>>>(g, alpha, boundary, x, y, w, scratch, tx, ty); break;
  }
  FMP_CHECK_LAUNCH();
  if (mode >= 1) return finish_reduce(scratch, grid, mode == 2 ? 2 : 1, dots, st);
  return 0;
}

extern "C" int fmp_curl(const fmp_block* blk, int kind, const double* x, double* out, void* stream) {
  if (int e = check_block(blk)) return e;
  const Geo g = make_geo(blk);
  dim3 grid((g.bx + 127) / 128, g.by, g.bz);
  if (kind == 0)
    k_curl<0><<<grid, 128, 0, as_stream(stream)>>>(g, x, out);
  else
    k_curl<1><<<grid, 128, 0, as_stream(stream)>>>(g, x, out);
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_cn_rhs(const fmp_block* blkE, const fmp_block* blkH, double dt, const double* E, const double* H,
                          double* R, void* stream) {
  if (int e = check_block(blkE)) return e;
  const Geo gE = make_geo(blkE), gH = make_geo(blkH);
  dim3 grid((gE.bx + 127) / 128, gE.by, gE.bz);
  k_cn_rhs<<<grid, 128, 0, as_stream(stream)>>>(gE, gH, dt, E, H, R);
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_cn_h_update(const fmp_block* blkNew, const fmp_block* blkOld, double dt, const double* H,
                               const double* E_new, const double* E_old, double* H_new, void* stream) {
  if (int e = check_block(blkNew)) return e;
  const Geo gN = make_geo(blkNew), gO = make_geo(blkOld);
  dim3 grid((gN.bx + 127) / 128, gN.by, gN.bz);
  k_cn_h<<<grid, 128, 0, as_stream(stream)>>>(gN, gO, 0.5 * dt, H, E_new, E_old, H_new);
  FMP_CHECK_LAUNCH();
  return 0;
}
