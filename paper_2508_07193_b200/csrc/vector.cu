// Krylov vector kernels (K8) and the deterministic reduction tail (K9's on-device half).
//
// Elementwise updates reproduce numpy's evaluation of the reference expressions
// (ref:krylov.py:114-136): every product and every sum is rounded on its own
// (__dmul_rn/__dadd_rn forbid FMA contraction), so equal inputs give equal bits.
// Roofline: HBM-bound; bytes per double = 8 x (vectors read + written).
#include <cstdarg>
#include <cstring>
#include <algorithm>
#include "common.cuh"

namespace fmp {

static thread_local char g_err[512] = "";
std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

// the vector kernels' launches with programmatic serialisation (FMP_NO_PDL_VEC=1: ordinary, A/B)
static bool vec_pdl() {
  static const bool on = pdl_on() && !getenv_flag("FMP_NO_PDL_VEC");
  return on;
}

// ---------------------------------------------------------------- reduction tail
template <int ND>
__global__ void __launch_bounds__(1024) k_finish(const double* __restrict__ partials, int count, double* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[32];
#pragma unroll
  for (int q = 0; q < ND; ++q) {
    double v = 0.0;
    for (int b = threadIdx.x; b < count; b += blockDim.x) v += partials[q * count + b];
    v = block_sum<1024>(v, red);
    if (threadIdx.x == 0) out[q] = v;
  }
}

int finish_reduce(const double* partials, int count, int nd, double* out, cudaStream_t st) {
  if (nd == 1)
    FMP_CHECK_CUDA(launch_k(vec_pdl(), k_finish<1>, 1, 1024, 0, st, partials, count, out));
  else
    FMP_CHECK_CUDA(launch_k(vec_pdl(), k_finish<2>, 1, 1024, 0, st, partials, count, out));
  FMP_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------- elementwise
__global__ void k_lincomb(int64_t n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                          double* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = add_rn(mul_rn(a, x[q]), mul_rn(b, y[q]));
}

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    y[q] = add_rn(y[q], mul_rn(a, x[q]));
}

__global__ void k_scale(int64_t n, double a, const double* __restrict__ x, double* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = mul_rn(a, x[q]);
}

__global__ void __launch_bounds__(kVecThreads) k_dot(int64_t n, const double* __restrict__ x,
                                                     const double* __restrict__ y, double* __restrict__ partials) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[kVecThreads / 32];
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    acc = fma(x[q], y[q], acc);
  acc = block_sum<kVecThreads>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

// p = 1.0*r + beta*(1.0*p + (-omega)*v)     (ref:krylov.py:181-182)
__global__ void k_bicg_p(int64_t n, const double* __restrict__ r, double* __restrict__ p,
                         const double* __restrict__ v, double beta, double momega) {
  pdl_trigger();
  pdl_wait();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double p1 = add_rn(p[q], mul_rn(momega, v[q]));
    p[q] = add_rn(r[q], mul_rn(beta, p1));
  }
}

// x += alpha*p_hat; x += omega*s_hat; r = 1.0*s + (-omega)*t; rho_next partial = (r_shadow, r)
// (ref:krylov.py:213-215 and the next iteration's krylov.py:171).  XZERO: x is zero on entry (the
// first iteration): the zero is a literal, so x is written without being read or pre-filled,
// with the same rounding (0.0 + a == a, +0.0 for a == -0.0, as when a stored zero is read)
template <bool XZERO>
__global__ void __launch_bounds__(kVecThreads) k_bicg_xr(int64_t n, double* __restrict__ x,
                                                         const double* __restrict__ ph,
                                                         const double* __restrict__ sh,
                                                         const double* __restrict__ s,
                                                         const double* __restrict__ t, double* __restrict__ r,
                                                         const double* __restrict__ rs, double alpha,
                                                         double omega, double* __restrict__ partials) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[kVecThreads / 32];
  double acc = 0.0;
  const double momega = -omega;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double xv = add_rn(XZERO ? 0.0 : x[q], mul_rn(alpha, ph[q]));
    x[q] = add_rn(xv, mul_rn(omega, sh[q]));
    const double rv = add_rn(s[q], mul_rn(momega, t[q]));
    r[q] = rv;
    acc = fma(rs[q], rv, acc);
  }
  acc = block_sum<kVecThreads>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

// y += a*x, then partial of (z, y_new)   (one MGS step of ref:krylov.py:301-309 fused with the
// next step's inner product; z = y gives the norm that ends the sweep)
__global__ void __launch_bounds__(kVecThreads) k_axpy_dot(int64_t n, double a, const double* __restrict__ x,
                                                          double* y, const double* z,
                                                          double* __restrict__ partials) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[kVecThreads / 32];
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double yv = add_rn(y[q], mul_rn(a, x[q]));
    y[q] = yv;
    acc = fma(z == y ? yv : z[q], yv, acc);
  }
  acc = block_sum<kVecThreads>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

// out = x; out += c_0 v_0; out += c_1 v_1; ...  in that order, each product and sum rounded
// (the reference's copy + axpy_into loop, ref:krylov.py:348-350), one pass over memory
constexpr int kCombineMax = 32;
struct CombineArgs {
  const double* v[kCombineMax];
  double c[kCombineMax];
  int k;
};
// x and out alias for every chunk after the first (fmp_vec_combine, k > kCombineMax): no
// __restrict__ on them; each element is read before it is written by the same thread.
__global__ void k_combine(int64_t n, const double* x, const CombineArgs A, double* out) {
  pdl_trigger();
  pdl_wait();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double t = x[q];
    for (int i = 0; i < A.k; ++i) t = add_rn(t, mul_rn(A.c[i], A.v[i][q]));
    out[q] = t;
  }
}

static inline int vec_grid(int64_t n) {
  const int64_t need = (n + kVecThreads - 1) / kVecThreads;
  return (int)(need < kVecGrid ? (need > 0 ? need : 1) : kVecGrid);
}

}  // namespace fmp

using namespace fmp;

extern "C" int fmp_abi_version(void) { return FMP_ABI_VERSION; }

extern "C" int fmp_last_error(char* buf, size_t len) {
  if (!buf || !len) return -1;
  strncpy(buf, g_err, len - 1);
  buf[len - 1] = 0;
  return 0;
}

extern "C" int64_t fmp_reduce_scratch_doubles(void) { return kScratchDoubles; }

extern "C" int64_t fmp_launch_count(void) { return g_launches.load(); }

extern "C" int fmp_vec_lincomb(int64_t n, double a, const double* x, double b, const double* y, double* out,
                               void* stream) {
  if (n <= 0) return 0;
  FMP_CHECK_CUDA(launch_k(vec_pdl(), k_lincomb, vec_grid(n), kVecThreads, 0, as_stream(stream), n, a, x, b, y, out));
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_vec_axpy(int64_t n, double a, const double* x, double* y, void* stream) {
  if (n <= 0) return 0;
  FMP_CHECK_CUDA(launch_k(vec_pdl(), k_axpy, vec_grid(n), kVecThreads, 0, as_stream(stream), n, a, x, y));
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_vec_scale(int64_t n, double a, const double* x, double* out, void* stream) {
  if (n <= 0) return 0;
  FMP_CHECK_CUDA(launch_k(vec_pdl(), k_scale, vec_grid(n), kVecThreads, 0, as_stream(stream), n, a, x, out));
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_vec_dot(int64_t n, const double* x, const double* y, double* out, double* scratch, void* stream) {
  const int grid = vec_grid(n);
  cudaStream_t st = as_stream(stream);
  FMP_CHECK_CUDA(launch_k(vec_pdl(), k_dot, grid, kVecThreads, 0, st, n, x, y, scratch));
  FMP_CHECK_LAUNCH();
  return finish_reduce(scratch, grid, 1, out, st);
}

extern "C" int fmp_vec_axpy_dot(int64_t n, double a, const double* x, double* y, const double* z, double* dots,
                                double* scratch, void* stream) {
  const int grid = vec_grid(n);
  cudaStream_t st = as_stream(stream);
  FMP_CHECK_CUDA(launch_k(vec_pdl(), k_axpy_dot, grid, kVecThreads, 0, st, n, a, x, y, z, scratch));
  FMP_CHECK_LAUNCH();
  return finish_reduce(scratch, grid, 1, dots, st);
}

extern "C" int fmp_vec_combine(int64_t n, const double* x, int k, const double* const* v, const double* coef,
                               double* out, void* stream) {
  FMP_REQUIRE(k >= 0 && (k == 0 || (v && coef)), "bad combine arguments");
  if (n <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  const double* src = x;
  for (int i0 = 0; i0 < k || i0 == 0; i0 += kCombineMax) {   // chunks of kCombineMax terms, in order
    CombineArgs a{};
    a.k = std::min(kCombineMax, k - i0);
    for (int i = 0; i < a.k; ++i) {
      a.v[i] = v[i0 + i];
      a.c[i] = coef[i0 + i];
    }
    FMP_CHECK_CUDA(launch_k(vec_pdl(), k_combine, vec_grid(n), kVecThreads, 0, st, n, src, a, out));
    FMP_CHECK_LAUNCH();
    src = out;
    if (k == 0) break;
  }
  return 0;
}

extern "C" int fmp_bicg_p(int64_t n, const double* r, double* p, const double* v, double beta, double omega,
                          void* stream) {
  if (n <= 0) return 0;
  FMP_CHECK_CUDA(launch_k(vec_pdl(), k_bicg_p, vec_grid(n), kVecThreads, 0, as_stream(stream), n, r, p, v, beta, -omega));
  FMP_CHECK_LAUNCH();
  return 0;
}

static int bicg_xr(bool xzero, int64_t n, double* x, const double* p_hat, const double* s_hat, const double* s,
                   const double* t, double* r, const double* r_shadow, double alpha, double omega, double* dots,
                   double* scratch, void* stream) {
  const int grid = vec_grid(n);
  cudaStream_t st = as_stream(stream);
  FMP_CHECK_CUDA(launch_k(vec_pdl(), xzero ? k_bicg_xr<true> : k_bicg_xr<false>, grid, kVecThreads, 0, st, n, x, p_hat,
                          s_hat, s, t, r, r_shadow, alpha, omega, scratch));
  FMP_CHECK_LAUNCH();
  return finish_reduce(scratch, grid, 1, dots, st);
}

extern "C" int fmp_bicg_xr(int64_t n, double* x, const double* p_hat, const double* s_hat, const double* s,
                           const double* t, double* r, const double* r_shadow, double alpha, double omega,
                           double* dots, double* scratch, void* stream) {
  return bicg_xr(false, n, x, p_hat, s_hat, s, t, r, r_shadow, alpha, omega, dots, scratch, stream);
}

extern "C" int fmp_bicg_xr0(int64_t n, double* x, const double* p_hat, const double* s_hat, const double* s,
                            const double* t, double* r, const double* r_shadow, double alpha, double omega,
                            double* dots, double* scratch, void* stream) {
  return bicg_xr(true, n, x, p_hat, s_hat, s, t, r, r_shadow, alpha, omega, dots, scratch, stream);
}
