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
#include "tma.cuh"
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <vector>

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
      if (!(bnd & FMP_STENCIL_LAMBDA)) {
        const int gk = g.gz0 + k;
        tx -= ((gj == 0) + (gk == 0)) * ex;
        ty -= ((gi == 0) + (gk == 0)) * ey;
        tz -= ((gi == 0) + (gj == 0)) * ez;
      }
      const bool id = !(bnd & FMP_STENCIL_NO_IDENTITY);
      const double yx = id ? ex + alpha * tx : alpha * tx, yy = id ? ey + alpha * ty : alpha * ty,
                   yz = id ? ez + alpha * tz : alpha * tz;
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

// curl at one point (used by the CN stencils and the CN right-hand side mode of the z-march)
template <int KIND, bool GEN>  // 0 forward, 1 backward
__device__ __forceinline__ void curl_at(const Loader<GEN>& L, int k, int j, int i, double& cx, double& cy,
                                        double& cz) {
  const double ex = L(0, k, j, i), ey = L(1, k, j, i), ez = L(2, k, j, i);
  if (KIND == 0) {  // D^f u(i) = u(i+1) - u(i), zero beyond the high face (ref:operators.py:94-96)
    cx = (L(2, k, j + 1, i) - ez) - (L(1, k + 1, j, i) - ey);
    cy = (L(0, k + 1, j, i) - ex) - (L(2, k, j, i + 1) - ez);
    cz = (L(1, k, j, i + 1) - ey) - (L(0, k, j + 1, i) - ex);
  } else {  // D^b u(i) = u(i) - u(i-1), zero before the low face (ref:operators.py:97-99)
    cx = (ez - L(2, k, j - 1, i)) - (ey - L(1, k - 1, j, i));
    cy = (ex - L(0, k - 1, j, i)) - (ez - L(2, k, j, i - 1));
    cz = (ey - L(1, k, j, i - 1)) - (ex - L(0, k, j - 1, i));
  }
}
// ---------------------------------------------------------------- SpMV, TMA z-march (sm_100a)
// Warp-specialised.  A producer warp streams each haloed plane of all three components
// ([3][SY+2][SX+4] doubles, 16 KB) into a 4-slot shared-memory ring with ONE TMA box load per
// plane; cells outside the block (the zero-ghost physical boundary) are the TMA unit's
// out-of-bounds zero fill, so there is no boundary code.  Eight consumer warps wait on the
// slot's "full" mbarrier, compute, and release the slot on its "empty" mbarrier; no CTA-wide
// barrier in the loop, so consumers and producer drift freely within the ring.
// GPU-block faces with neighbour ghosts are patched in shared memory after the plane lands.
// Work: units (z-chunk of L planes) x (64 x 8 column tile), z-chunk-major, handed out by an
// atomic counter to a grid of exactly the resident CTAs, so CTAs that run concurrently hold
// neighbouring tiles of the same z range and the halo rows/planes they share are L2 hits.
constexpr int SX = 64, SY = 8;
constexpr int SXR = SX + 4, SYH = SY + 2;          // smem row: logical i0-2 .. i0+SX+1
constexpr int SPL = SXR * SYH, SPLANE = 3 * SPL;   // doubles per component plane / per plane
constexpr int SSLOT = (SPLANE + 15) / 16 * 16;      // slot stride: TMA destinations are 128-byte aligned
constexpr int SCONS = 8;                            // consumer warps
constexpr int STHREADS = (SCONS + 1) * 32;
constexpr uint32_t kPlaneBytes = SPLANE * 8;
// [ring: NS x SSLOT doubles][2 x NS mbarriers][NS unit ids (int64)][2 x SCONS reduction words]
constexpr int spmv_bulk_smem(int ns) { return (ns * SSLOT + 3 * ns + 2 * SCONS) * (int)sizeof(double); }

struct BulkSpmvArgs {
  Geo g;
  const double* x;
  double* y;
  const double* w;
  double* partials;
  unsigned long long* counter;   // [fetch, done]: dynamic unit scheduler, zero between launches
  const int* ulist;              // units of this launch (nullptr: all units 0 .. units-1)
  int64_t nlaunch;               // units handed out by this launch
  double alpha;
  int bnd, tiles_x, tiles_y, L, nzc, ghosts;
  int wpf;   // modes 1-3: L2 prefetch distance (planes) of the w operand, 0 = off
  int wlate; // modes 1-3: w read after the stencil (FMP_SPMV_WLATE=1, A/B)
  // mode 4 (CN right-hand side, fmp_cn_rhs): y = (x + dt curl_b(h)) - alpha C_b C_f x with x = E
  // streamed through the ring, h = H read per point (its ghosts in gh), bnd = 0 (no Lambda)
  Geo gh;
  const double* h;
  double dt;
};

template <int MODE, int SNSLOT>
__global__ void __launch_bounds__(STHREADS, SNSLOT <= 4 ? 3 : 2) k_spmv_bulk(const __grid_constant__ CUtensorMap tm, BulkSpmvArgs A) {
  extern __shared__ __align__(128) double ring[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + SNSLOT * SSLOT);
  uint64_t* empty = full + SNSLOT;
  int64_t* slot_unit = reinterpret_cast<int64_t*>(empty + SNSLOT);   // unit of a unit's first load, -1 = done
  double* red = reinterpret_cast<double*>(slot_unit + SNSLOT);
  const Geo& g = A.g;
  const int tid = threadIdx.x, warp = tid >> 5, lx = tid & 31;
  const int ntiles = A.tiles_x * A.tiles_y;
  const int64_t units = (int64_t)ntiles * A.nzc;
  const int64_t V = (int64_t)g.bx * g.by * g.bz;
  if (tid == 0) {
    tma_prefetch_desc(&tm);
    for (int s = 0; s < SNSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SCONS);
    }
    fence_mbar_init();
  }
  pdl_trigger();
  pdl_wait();   // x (and the scheduler counters) belong to the previous kernels on the stream
  __syncthreads();
  auto nplanes = [&](int64_t u) { return min(A.L, g.bz - (int)(u / ntiles) * A.L); };

  if (warp == SCONS) {
    // ---------------- producer: takes units from the global counter (z-chunk-major order, so
    // the CTAs in flight hold neighbouring tiles of the same z range) and streams planes
    // k0-1 .. k0+np of each; the unit id rides with the unit's first plane
    int64_t q = 0;
    for (;;) {
      unsigned long long f = 0;
      if (lx == 0) f = atomicAdd(A.counter, 1ull);
      f = __shfl_sync(0xffffffffu, f, 0);
      if ((int64_t)f >= A.nlaunch) {   // tell the consumers: a "unit" of -1 in the next slot
        const int s = (int)(q % SNSLOT);
        if (q >= SNSLOT) mbar_wait(&empty[s], (uint32_t)(((q / SNSLOT) - 1) & 1));
        if (lx == 0) {
          slot_unit[s] = -1;
          mbar_arrive(&full[s]);
          __threadfence();   // the last CTA out re-arms the scheduler for the next launch
          if (atomicAdd(A.counter + 1, 1ull) == gridDim.x - 1) {
            A.counter[0] = 0;
            A.counter[1] = 0;
          }
        }
        break;
      }
      const int64_t u = A.ulist ? (int64_t)A.ulist[f] : (int64_t)f;
      const int tile = (int)(u % ntiles), zc = (int)(u / ntiles);
      const int i0 = (tile % A.tiles_x) * SX, j0 = (tile / A.tiles_x) * SY, k0 = zc * A.L;
      const int np = nplanes(u);
      for (int m = 0; m < np + 2; ++m, ++q) {
        const int s = (int)(q % SNSLOT), k = k0 - 1 + m;
        if (q >= SNSLOT) mbar_wait(&empty[s], (uint32_t)(((q / SNSLOT) - 1) & 1));
        if (lx == 0) {
          if (m == 0) slot_unit[s] = u;
          mbar_expect_tx(&full[s], kPlaneBytes);
        }
        __syncwarp();
        // one TMA box per plane; cells outside the block (negative or beyond-the-end
        // coordinates) are zero-filled by the TMA unit = the zero-ghost boundary.  The box
        // starts at x = i0 - 2: tile-mode boxes need a 16-byte aligned inner coordinate
        // (negative ones are fine), tools/tma_test.cu
        if (lx == 0) tma_load_4d(ring + s * SSLOT, &tm, i0 - 2, j0 - 1, k, 0, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers: 8 warps, row ly = warp, points i0 + lane and i0 + lane + 32.
  // Plane k-1 is never re-read from shared memory: the five values the stencil needs from it
  // were read from plane k one step earlier and are carried in registers (20 shared loads per
  // point instead of 25).  So only planes k and k+1 are held; plane k is released after the step.
  // Fused dot products: one partial per UNIT (not per CTA), summed over the 8 consumer warps in a
  // fixed order, so the result does not depend on which CTA the scheduler gave a unit to and the
  // final fixed-order reduction over units is deterministic.
  const int ly = warp;
  int64_t qbase = 0;   // load index of the current unit's first plane (k0 - 1)
  for (;;) {
    double acc0 = 0.0, acc1 = 0.0;
    mbar_wait(&full[qbase % SNSLOT], (uint32_t)((qbase / SNSLOT) & 1));
    const int64_t u = slot_unit[qbase % SNSLOT];
    if (u < 0) break;
    const int tile = (int)(u % ntiles), zc = (int)(u / ntiles);
    const int i0 = (tile % A.tiles_x) * SX, j0 = (tile / A.tiles_x) * SY, k0 = zc * A.L;
    const int np = nplanes(u);
    // neighbour ghosts: halo cells outside the block in x / y (ii in [0, xa) u [xb, SX+2),
    // jj in [0, ya) u [yb, SYH)) and whole planes outside it in z are overwritten by fetch()
    const int xa = i0 == 0 ? 1 : 0, xb = min(SX + 2, g.bx - i0 + 1), nxs = xa + (SX + 2 - xb);
    const int ya = j0 == 0 ? 1 : 0, yb = min(SYH, g.by - j0 + 1), nys = ya + (SYH - yb);
    const bool edge = A.ghosts && (nxs > 0 || nys > 0 || k0 == 0 || k0 + np == g.bz);
    double pe[2], pf[2], ph[2], pq[2], pr[2];   // plane k-1: ex, ey, ez, ez(i+1), ez(j+1)
    for (int jz = 0; jz < np; ++jz) {
      const int64_t q0 = qbase + jz;
      for (int h = (jz == 0 ? 0 : 2); h < 3; ++h)
        mbar_wait(&full[(q0 + h) % SNSLOT], (uint32_t)(((q0 + h) / SNSLOT) & 1));
      if (edge) {
        const int ct = tid, nct = SCONS * 32;
        for (int h = (jz == 0 ? 0 : 2); h < 3; ++h) {
          const int k = k0 + jz - 1 + h;
          double* P = ring + ((q0 + h) % SNSLOT) * SSLOT;
          if (k < 0 || k >= g.bz) {
            for (int e = ct; e < 3 * SYH * (SX + 2); e += nct) {
              const int c = e / (SYH * (SX + 2)), r = e - c * (SYH * (SX + 2)), jj = r / (SX + 2), ii = r - jj * (SX + 2);
              P[c * SPL + jj * SXR + ii + 1] = fetch(g, A.x, c, k, j0 - 1 + jj, i0 - 1 + ii);
            }
            continue;
          }
          if (nxs > 0)
            for (int e = ct; e < 3 * SYH * nxs; e += nct) {
              const int c = e / (SYH * nxs), r = e - c * (SYH * nxs), jj = r / nxs, qq = r - jj * nxs;
              const int ii = qq < xa ? qq : xb + (qq - xa);
              P[c * SPL + jj * SXR + ii + 1] = fetch(g, A.x, c, k, j0 - 1 + jj, i0 - 1 + ii);
            }
          if (nys > 0)
            for (int e = ct; e < 3 * nys * (SX + 2); e += nct) {
              const int c = e / (nys * (SX + 2)), r = e - c * (nys * (SX + 2)), qq = r / (SX + 2), ii = r - qq * (SX + 2);
              const int jj = qq < ya ? qq : yb + (qq - ya);
              P[c * SPL + jj * SXR + ii + 1] = fetch(g, A.x, c, k, j0 - 1 + jj, i0 - 1 + ii);
            }
        }
        fence_proxy_async();
        asm volatile("bar.sync 1, %0;\n" ::"n"(SCONS * 32) : "memory");   // consumers only
      }
      const double* p0 = ring + ((q0 + 1) % SNSLOT) * SSLOT;
      const double* pp = ring + ((q0 + 2) % SNSLOT) * SSLOT;
      const int k = k0 + jz, j = j0 + ly;
      // modes 1-3: this plane's w operand, loaded before the stencil so its latency overlaps the
      // shared-memory reads and arithmetic (FMP_SPMV_WLATE=1: loaded after, A/B)
      double wv[2][3];
      if (MODE == 4) {   // curl_b(H) of this plane's two points, ahead of the stencil likewise
#pragma unroll
        for (int hx = 0; hx < 2; ++hx) {
          const int i = i0 + lx + 32 * hx;
          wv[hx][0] = wv[hx][1] = wv[hx][2] = 0.0;
          if (i < g.bx && j < g.by) {
            if (i >= 1 && j >= 1 && k >= 1)
              curl_at<1>(Loader<false>{A.gh, A.h}, k, j, i, wv[hx][0], wv[hx][1], wv[hx][2]);
            else
              curl_at<1>(Loader<true>{A.gh, A.h}, k, j, i, wv[hx][0], wv[hx][1], wv[hx][2]);
          }
        }
      }
      if (MODE >= 1 && MODE <= 3 && !A.wlate) {
#pragma unroll
        for (int hx = 0; hx < 2; ++hx) {
          const int i = i0 + lx + 32 * hx;
          const bool in = i < g.bx && j < g.by;
          const int64_t oi = in ? fidx(g, 0, k, j, i) : 0;
#pragma unroll
          for (int c = 0; c < 3; ++c) wv[hx][c] = in ? A.w[oi + c * V] : 0.0;
        }
      }
#define EX(P, dj, di) P[0 * SPL + o + (dj) * SXR + (di)]
#define EY(P, dj, di) P[1 * SPL + o + (dj) * SXR + (di)]
#define EZ(P, dj, di) P[2 * SPL + o + (dj) * SXR + (di)]
#pragma unroll
      for (int hx = 0; hx < 2; ++hx) {
        const int i = i0 + lx + 32 * hx;
        const int o = (ly + 1) * SXR + lx + 32 * hx + 2;
        if (jz == 0) {   // unit start: prime the carried plane k0-1 values
          const double* pm_ = ring + (q0 % SNSLOT) * SSLOT;
          pe[hx] = EX(pm_, 0, 0);
          pf[hx] = EY(pm_, 0, 0);
          ph[hx] = EZ(pm_, 0, 0);
          pq[hx] = EZ(pm_, 0, 1);
          pr[hx] = EZ(pm_, 1, 0);
        }
        const double ex = EX(p0, 0, 0), ey = EY(p0, 0, 0), ez = EZ(p0, 0, 0);
        const double ez_ip = EZ(p0, 0, 1), ez_jp = EZ(p0, 1, 0), ex_im = EX(p0, 0, -1), ey_jm = EY(p0, -1, 0);
        const double nx = EX(pp, 0, 0), ny = EY(pp, 0, 0);
        // Appendix A: (C_b C_f + Lambda) x on the zero-ghost padded box
        double tx = 4.0 * ex - EX(p0, -1, 0) - EX(p0, 1, 0) - pe[hx] - nx + EY(p0, 0, 1) - ey - EY(p0, -1, 1) +
                    ey_jm + ez_ip - ez - pq[hx] + ph[hx];
        double ty = 4.0 * ey - EY(p0, 0, -1) - EY(p0, 0, 1) - pf[hx] - ny + ez_jp - ez - pr[hx] + ph[hx] +
                    EX(p0, 1, 0) - ex - EX(p0, 1, -1) + ex_im;
        double tz = 4.0 * ez - EZ(p0, 0, -1) - ez_ip - EZ(p0, -1, 0) - ez_jp + nx - ex - EX(pp, 0, -1) + ex_im + ny -
                    ey - EY(pp, -1, 0) + ey_jm;
        pe[hx] = ex;
        pf[hx] = ey;
        ph[hx] = ez;
        pq[hx] = ez_ip;
        pr[hx] = ez_jp;
        if (i >= g.bx || j >= g.by) continue;
        if (!(A.bnd & FMP_STENCIL_LAMBDA)) {
          const int gi = g.gx0 + i, gj = g.gy0 + j, gk = g.gz0 + k;
          tx -= ((gj == 0) + (gk == 0)) * ex;
          ty -= ((gi == 0) + (gk == 0)) * ey;
          tz -= ((gi == 0) + (gj == 0)) * ez;
        }
        const bool id = !(A.bnd & FMP_STENCIL_NO_IDENTITY);
        const double yx = id ? ex + A.alpha * tx : A.alpha * tx, yy = id ? ey + A.alpha * ty : A.alpha * ty,
                     yz = id ? ez + A.alpha * tz : A.alpha * tz;
        const int64_t oi = fidx(g, 0, k, j, i);
        if (MODE >= 1 && MODE <= 3 && A.wpf > 0 && k + A.wpf < g.bz) {   // w of a later plane of this column into L2
          const double* wn = A.w + oi + (int64_t)A.wpf * g.bx * g.by;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(wn));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(wn + V));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(wn + 2 * V));
        }
        if (MODE == 4) {   // ref:cn_driver.py:54-59, same evaluation order as k_cn_rhs
          __stcs(A.y + oi, (ex + A.dt * wv[hx][0]) - A.alpha * tx);
          __stcs(A.y + oi + V, (ey + A.dt * wv[hx][1]) - A.alpha * ty);
          __stcs(A.y + oi + 2 * V, (ez + A.dt * wv[hx][2]) - A.alpha * tz);
        } else if (MODE == 3) {
          const double w0 = A.wlate ? A.w[oi] : wv[hx][0], w1 = A.wlate ? A.w[oi + V] : wv[hx][1],
                       w2 = A.wlate ? A.w[oi + 2 * V] : wv[hx][2];
          const double rx = w0 - yx, ry = w1 - yy, rz = w2 - yz;
          acc0 += rx * rx + ry * ry + rz * rz;
        } else {
          __stcs(A.y + oi, yx);   // streaming stores: keep L2 for the halo planes and rows
          __stcs(A.y + oi + V, yy);
          __stcs(A.y + oi + 2 * V, yz);
          if (MODE >= 1) {
            const double w0 = A.wlate ? A.w[oi] : wv[hx][0], w1 = A.wlate ? A.w[oi + V] : wv[hx][1],
                         w2 = A.wlate ? A.w[oi + 2 * V] : wv[hx][2];
            acc0 += yx * w0 + yy * w1 + yz * w2;
          }
          if (MODE == 2) acc1 += yx * yx + yy * yy + yz * yz;
        }
      }
#undef EX
#undef EY
#undef EZ
      __syncwarp();
      if (lx == 0) {   // release plane k (and plane k-1 after the first step, k+1 after the last)
        mbar_arrive(&empty[(q0 + 1) % SNSLOT]);
        if (jz == 0) mbar_arrive(&empty[q0 % SNSLOT]);
        if (jz == np - 1) mbar_arrive(&empty[(q0 + 2) % SNSLOT]);
      }
    }
    qbase += np + 2;
    if (MODE >= 1 && MODE <= 3) {   // this unit's partial(s): consumer-only reduction (named barrier 1)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
        acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
      }
      if (lx == 0) {
        red[warp] = acc0;
        red[SCONS + warp] = acc1;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(SCONS * 32) : "memory");
      if (tid == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w2 = 0; w2 < SCONS; ++w2) {
          s0 += red[w2];
          s1 += red[SCONS + w2];
        }
        A.partials[u] = s0;
        if (MODE == 2) A.partials[units + u] = s1;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(SCONS * 32) : "memory");
    }
  }
}

// ---------------------------------------------------------------- curls and CN stencils
// A point whose stencil stays inside the block reads with plain loads (Loader<false>); only the
// block's surface layer goes through fetch() (global zero boundary, neighbour ghosts).
__device__ __forceinline__ bool inner(const Geo& g, int k, int j, int i) {
  return i >= 1 && j >= 1 && k >= 1 && i + 1 < g.bx && j + 1 < g.by && k + 1 < g.bz;
}
// 2-D thread blocks (32 x 8): the j-neighbours a thread reads were just read by its block
constexpr int CBX = 32, CBY = 8;

template <int KIND>
__global__ void __launch_bounds__(CBX* CBY) k_curl(Geo g, const double* __restrict__ f, double* __restrict__ out) {
  const int i = blockIdx.x * CBX + threadIdx.x, j = blockIdx.y * CBY + threadIdx.y, k = blockIdx.z;
  if (i >= g.bx || j >= g.by) return;
  double cx, cy, cz;
  if (inner(g, k, j, i))
    curl_at<KIND>(Loader<false>{g, f}, k, j, i, cx, cy, cz);
  else
    curl_at<KIND>(Loader<true>{g, f}, k, j, i, cx, cy, cz);
  const int64_t o = fidx(g, 0, k, j, i), V = (int64_t)g.bx * g.by * g.bz;
  out[o] = cx;
  out[o + V] = cy;
  out[o + 2 * V] = cz;
}

// R = E + dt*curl_b(H) - alpha*(C_b C_f E), alpha = dt^2/4  (ref:cn_driver.py:54-59)
__global__ void __launch_bounds__(CBX* CBY) k_cn_rhs(Geo gE, Geo gH, double dt, const double* __restrict__ E,
                                                    const double* __restrict__ H, double* __restrict__ R) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * CBX + threadIdx.x, j = blockIdx.y * CBY + threadIdx.y, k = blockIdx.z;
  if (i >= gE.bx || j >= gE.by) return;
  const double alpha = dt * dt / 4.0;
  double hx, hy, hz, tx, ty, tz, ex, ey, ez;
  if (inner(gE, k, j, i)) {
    curl_at<1>(Loader<false>{gH, H}, k, j, i, hx, hy, hz);
    bracket<false>(Loader<false>{gE, E}, k, j, i, tx, ty, tz, ex, ey, ez);
  } else {
    curl_at<1>(Loader<true>{gH, H}, k, j, i, hx, hy, hz);
    bracket<true>(Loader<true>{gE, E}, k, j, i, tx, ty, tz, ex, ey, ez);
  }
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
__global__ void __launch_bounds__(CBX* CBY) k_cn_h(Geo gN, Geo gO, double hdt, const double* __restrict__ H,
                                                  const double* __restrict__ En, const double* __restrict__ Eo,
                                                  double* __restrict__ Hn) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * CBX + threadIdx.x, j = blockIdx.y * CBY + threadIdx.y, k = blockIdx.z;
  if (i >= gN.bx || j >= gN.by) return;
  double ax, ay, az, bx, by, bz;
  if (inner(gN, k, j, i)) {
    curl_at<0>(Loader<false>{gN, En}, k, j, i, ax, ay, az);
    curl_at<0>(Loader<false>{gO, Eo}, k, j, i, bx, by, bz);
  } else {
    curl_at<0>(Loader<true>{gN, En}, k, j, i, ax, ay, az);
    curl_at<0>(Loader<true>{gO, Eo}, k, j, i, bx, by, bz);
  }
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

// z-chunk length: minimise rounds x (planes + 2 halo planes) for the resident grid
static void spmv_chunking(int64_t ntiles, int bz, int64_t resident, int* L_out, int* nzc_out) {
  int bestL = bz;
  double best = 1e300;
  for (int L = 4; L <= 64; ++L) {
    const int Lc = std::min(L, bz);
    const int64_t nzc = (bz + Lc - 1) / Lc, units = ntiles * nzc;
    const int64_t rounds = (units + resident - 1) / resident;
    const double cost = (double)rounds * (Lc + 2);
    if (cost < best - 1e-9) { best = cost; bestL = Lc; }
    if (Lc == bz) break;
  }
  *L_out = bestL;
  *nzc_out = (bz + bestL - 1) / bestL;
}

static bool bulk_ok(const fmp_block* b, const double* x) {
  return b->bx % 2 == 0 && ((uintptr_t)x & 15) == 0 && b->bx <= ((int64_t)1 << 31) &&
         b->by <= ((int64_t)1 << 31) && b->bz <= ((int64_t)1 << 31) && !getenv_flag("FMP_SPMV_LEGACY");
}

// Units of one part of the SpMV (z-chunk x column tile, in scheduler order): FMP_PART_INTERIOR =
// units that read no neighbour ghost cell, FMP_PART_BOUNDARY = the others.  A unit covers
// i in [i0-1, i0+SX], j in [j0-1, j0+SY], k in [k0-1, k0+np]; it reads a ghost slab when that range
// leaves the block on a side whose ghost pointer is set.  Lists are built once per geometry and
// kept on the device (one small allocation per distinct (device, block, chunking, ghost mask)).
static int unit_list(const Geo& g, int tiles_x, int tiles_y, int L, int nzc, int part, const int** out,
                     int64_t* count) {
  static std::mutex mu;
  static std::map<std::vector<int64_t>, std::pair<int*, int64_t>> cache;
  int dev = 0;
  FMP_CHECK_CUDA(cudaGetDevice(&dev));
  int mask = 0;
  for (int q = 0; q < 6; ++q) mask |= (g.ghost[q] != nullptr) << q;
  const std::vector<int64_t> key{dev, g.bx, g.by, g.bz, L, nzc, mask, part};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<int> units;
    const int64_t ntiles = (int64_t)tiles_x * tiles_y;
    for (int64_t u = 0; u < ntiles * nzc; ++u) {
      const int tile = (int)(u % ntiles), zc = (int)(u / ntiles);
      const int i0 = (tile % tiles_x) * SX, j0 = (tile / tiles_x) * SY, k0 = zc * L;
      const int np = std::min(L, g.bz - k0);
      const bool ghost = (i0 == 0 && (mask & 1)) || (i0 + SX >= g.bx && (mask & 2)) || (j0 == 0 && (mask & 4)) ||
                         (j0 + SY >= g.by && (mask & 8)) || (k0 == 0 && (mask & 16)) ||
                         (k0 + np >= g.bz && (mask & 32));
      if (ghost == (part == FMP_PART_BOUNDARY)) units.push_back((int)u);
    }
    int* d = nullptr;
    if (!units.empty()) {
      FMP_CHECK_CUDA(cudaMalloc(&d, units.size() * sizeof(int)));
      FMP_CHECK_CUDA(cudaMemcpy(d, units.data(), units.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    it = cache.emplace(key, std::make_pair(d, (int64_t)units.size())).first;
  }
  *out = it->second.first;
  *count = it->second.second;
  return 0;
}

static int stencil_apply(const fmp_block* blk, double alpha, int boundary, int mode, int part, const double* x,
                         double* y, const double* w, double* dots, double* scratch, void* stream,
                         const fmp_block* blkH = nullptr, const double* H = nullptr, double dt = 0.0);

extern "C" int fmp_stencil_apply(const fmp_block* blk, double alpha, int boundary, int mode, const double* x,
                                 double* y, const double* w, double* dots, double* scratch, void* stream) {
  return stencil_apply(blk, alpha, boundary, mode, FMP_PART_ALL, x, y, w, dots, scratch, stream);
}

extern "C" int fmp_stencil_apply_part(const fmp_block* blk, double alpha, int boundary, int mode, int part,
                                      const double* x, double* y, const double* w, double* dots, double* scratch,
                                      void* stream) {
  FMP_REQUIRE(part >= FMP_PART_ALL && part <= FMP_PART_BOUNDARY, "bad part %d", part);
  return stencil_apply(blk, alpha, boundary, mode, part, x, y, w, dots, scratch, stream);
}

static int stencil_apply(const fmp_block* blk, double alpha, int boundary, int mode, int part, const double* x,
                         double* y, const double* w, double* dots, double* scratch, void* stream,
                         const fmp_block* blkH, const double* H, double dt) {
  if (int e = check_block(blk)) return e;
  FMP_REQUIRE((mode >= 0 && mode <= 3) || (mode == 4 && blkH && H), "bad stencil mode %d", mode);
  FMP_REQUIRE(boundary >= 0 && boundary <= 3, "bad stencil boundary flags %d", boundary);
  const bool reduces = mode >= 1 && mode <= 3;   // modes with fused dot products
  FMP_REQUIRE(!reduces || (w && dots && scratch), "mode %d needs w, dots and scratch", mode);
  const Geo g = make_geo(blk);
  cudaStream_t st = as_stream(stream);
  if (bulk_ok(blk, x)) {
    // the smem attribute and the occupancy are per device: set them once on each device used
    static int resident4s[64] = {}, resident6s[64] = {};
    int cur = 0;
    FMP_CHECK_CUDA(cudaGetDevice(&cur));
    FMP_REQUIRE(cur < 64, "device index %d out of range", cur);
    int& resident4 = resident4s[cur];
    int& resident6 = resident6s[cur];
    if (!resident4) {
#define FMP_SPMV_ATTR(M, N)                                                                            \
  FMP_CHECK_CUDA(cudaFuncSetAttribute(k_spmv_bulk<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                      spmv_bulk_smem(N)));
      FMP_SPMV_ATTR(0, 4) FMP_SPMV_ATTR(1, 4) FMP_SPMV_ATTR(2, 4) FMP_SPMV_ATTR(3, 4) FMP_SPMV_ATTR(4, 4)
      FMP_SPMV_ATTR(0, 6) FMP_SPMV_ATTR(1, 6) FMP_SPMV_ATTR(2, 6) FMP_SPMV_ATTR(3, 6) FMP_SPMV_ATTR(4, 6)
#undef FMP_SPMV_ATTR
      int r = 0;
      FMP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_spmv_bulk<0, 4>, STHREADS, spmv_bulk_smem(4)));
      resident4 = std::max(1, r);
      FMP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_spmv_bulk<0, 6>, STHREADS, spmv_bulk_smem(6)));
      resident6 = std::max(1, r);
    }
    const int ns = getenv_flag("FMP_SPMV_NS6") ? 6 : 4;
    const int resident_per_sm = ns == 4 ? resident4 : resident6;
    BulkSpmvArgs a{};
    a.g = g;
    a.x = x;
    a.y = y;
    a.w = w;
    a.partials = scratch;
    a.alpha = alpha;
    a.bnd = boundary;
    if (mode == 4) {
      a.gh = make_geo(blkH);
      a.h = H;
      a.dt = dt;
    }
    a.tiles_x = (g.bx + SX - 1) / SX;
    a.tiles_y = (g.by + SY - 1) / SY;
    a.ghosts = 0;
    for (int q = 0; q < 6; ++q) a.ghosts |= g.ghost[q] != nullptr;
    // the w operand of the fused dots / residual is read per point after the stencil, so its DRAM
    // latency sits in every consumer step; prefetching the next plane's w into L2 hides it
    // (bench.py: 2434 -> 2463 MDoF/s at cfg4; FMP_SPMV_WPF=0 turns it off)
    a.wpf = getenv("FMP_SPMV_WPF") ? atoi(getenv("FMP_SPMV_WPF")) : 1;
    a.wlate = getenv_flag("FMP_SPMV_WLATE") ? 1 : 0;
    // [fetch, done] counter pairs of the unit scheduler, zero at rest (each launch re-arms its
    // own pair).  A ring of pairs, so launches in flight on different streams or devices of this
    // process never share one (per device: the ring is allocated on the current device).
    constexpr int kCounterRing = 64;
    static unsigned long long* counters[64] = {};
    static std::atomic<unsigned> next_pair{0};
    int dev = 0;
    FMP_CHECK_CUDA(cudaGetDevice(&dev));
    FMP_REQUIRE(dev < 64, "device index %d out of range", dev);
    if (!counters[dev]) {
      unsigned long long* c = nullptr;
      FMP_CHECK_CUDA(cudaMalloc(&c, 2 * kCounterRing * sizeof(unsigned long long)));
      FMP_CHECK_CUDA(cudaMemset(c, 0, 2 * kCounterRing * sizeof(unsigned long long)));
      counters[dev] = c;
    }
    a.counter = counters[dev] + 2 * (next_pair.fetch_add(1, std::memory_order_relaxed) % kCounterRing);
    const int64_t ntiles = (int64_t)a.tiles_x * a.tiles_y;
    const int64_t resident = (int64_t)kNumSM * resident_per_sm;
    spmv_chunking(ntiles, g.bz, resident, &a.L, &a.nzc);
    if (reduces)   // one partial per unit (two in mode 2) must fit the scratch: longer chunks
      while (ntiles * a.nzc > kScratchDoubles / 2 && a.L < g.bz) {
        a.L = std::min(g.bz, 2 * a.L);
        a.nzc = (g.bz + a.L - 1) / a.L;
      }
    const int64_t units = ntiles * a.nzc;
    FMP_REQUIRE(!reduces || units <= kScratchDoubles / 2, "block too large for the SpMV reduction scratch");
    a.ulist = nullptr;
    a.nlaunch = units;
    if (part != FMP_PART_ALL) {
      if (int e = unit_list(g, a.tiles_x, a.tiles_y, a.L, a.nzc, part, &a.ulist, &a.nlaunch)) return e;
    }
    const int grid = (int)std::min<int64_t>(a.nlaunch, resident);
    if (grid > 0) {
    CUtensorMap tm;
    const uint64_t dims[4] = {(uint64_t)g.bx, (uint64_t)g.by, (uint64_t)g.bz, 3};
    const uint64_t strides[3] = {(uint64_t)g.bx * 8, (uint64_t)g.bx * g.by * 8, (uint64_t)g.bx * g.by * g.bz * 8};
    const uint32_t box[4] = {SXR, SYH, 1, 3};
    if (int e = encode_tensor_map_f64(&tm, x, 4, dims, strides, box)) return e;
#define FMP_SPMV_GO(N)                                                                                   \
  switch (mode) {                                                                                        \
    case 0: FMP_CHECK_CUDA(launch_pdl(k_spmv_bulk<0, N>, grid, STHREADS, spmv_bulk_smem(N), st, tm, a)); break;                \
    case 1: FMP_CHECK_CUDA(launch_pdl(k_spmv_bulk<1, N>, grid, STHREADS, spmv_bulk_smem(N), st, tm, a)); break;                \
    case 2: FMP_CHECK_CUDA(launch_pdl(k_spmv_bulk<2, N>, grid, STHREADS, spmv_bulk_smem(N), st, tm, a)); break;                \
    case 3: FMP_CHECK_CUDA(launch_pdl(k_spmv_bulk<3, N>, grid, STHREADS, spmv_bulk_smem(N), st, tm, a)); break;                \
    case 4: FMP_CHECK_CUDA(launch_pdl(k_spmv_bulk<4, N>, grid, STHREADS, spmv_bulk_smem(N), st, tm, a)); break;                \
  }
    if (ns == 4) {
      FMP_SPMV_GO(4)
    } else {
      FMP_SPMV_GO(6)
    }
#undef FMP_SPMV_GO
    FMP_CHECK_LAUNCH();
    }
    // the interior part leaves its per-unit partials in scratch; the boundary part adds its own
    // and reduces all of them in the fixed unit order
    if (reduces && part != FMP_PART_INTERIOR) return finish_reduce(scratch, (int)units, mode == 2 ? 2 : 1, dots, st);
    return 0;
  }
  FMP_REQUIRE(mode != 4, "CN right-hand side mode needs the bulk path");
  if (part == FMP_PART_INTERIOR) return 0;   // the thread-per-point fallback runs whole in the boundary part
  const int tx = (g.bx + TX - 1) / TX, ty = (g.by + TY - 1) / TY;
  const int64_t units = (int64_t)tx * ty * g.bz;
  // one full wave: SMs x resident CTAs (smem-limited to 5 of 41 KB), fewer for tiny blocks
  const int64_t want = (int64_t)kNumSM * 5;
  const int grid = (int)(units / 8 < want ? (units / 8 > 0 ? units / 8 : 1) : want);
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
  const dim3 grid((g.bx + CBX - 1) / CBX, (g.by + CBY - 1) / CBY, g.bz), block(CBX, CBY);
  if (kind == 0)
    k_curl<0><<<grid, block, 0, as_stream(stream)>>>(g, x, out);
  else
    k_curl<1><<<grid, block, 0, as_stream(stream)>>>(g, x, out);
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_cn_rhs(const fmp_block* blkE, const fmp_block* blkH, double dt, const double* E, const double* H,
                          double* R, void* stream) {
  if (int e = check_block(blkE)) return e;
  if (bulk_ok(blkE, E) && !getenv_flag("FMP_CN_RHS_POINT"))   // E through the TMA z-march ring (mode 4)
    return stencil_apply(blkE, dt * dt / 4.0, 0, 4, FMP_PART_ALL, E, R, nullptr, nullptr, nullptr, stream, blkH, H, dt);
  const Geo gE = make_geo(blkE), gH = make_geo(blkH);
  const dim3 grid((gE.bx + CBX - 1) / CBX, (gE.by + CBY - 1) / CBY, gE.bz), block(CBX, CBY);
  FMP_CHECK_CUDA(launch_pdl(k_cn_rhs, grid, block, 0, as_stream(stream), gE, gH, dt, E, H, R));
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_cn_h_update(const fmp_block* blkNew, const fmp_block* blkOld, double dt, const double* H,
                               const double* E_new, const double* E_old, double* H_new, void* stream) {
  if (int e = check_block(blkNew)) return e;
  const Geo gN = make_geo(blkNew), gO = make_geo(blkOld);
  const dim3 grid((gN.bx + CBX - 1) / CBX, (gN.by + CBY - 1) / CBY, gN.bz), block(CBX, CBY);
  FMP_CHECK_CUDA(launch_pdl(k_cn_h, grid, block, 0, as_stream(stream), gN, gO, 0.5 * dt, H, E_new, E_old, H_new));
  FMP_CHECK_LAUNCH();
  return 0;
}
