// Shared device helpers for libflashmp_b200 (sm_100a).
#pragma once
#include <atomic>
#include <utility>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../include/flashmp_b200.h"

namespace fmp {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
#define FMP_CHECK_CUDA(call)                                                        \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ::fmp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return -1;                                                                    \
    }                                                                               \
  } while (0)
// Every kernel launch of this library is followed by FMP_CHECK_LAUNCH(), which also counts
// it (fmp_launch_count) so benchmarks can report how many of OUR kernels ran.
extern std::atomic<int64_t> g_launches;
#define FMP_CHECK_LAUNCH()                                        \
  do {                                                            \
    ::fmp::g_launches.fetch_add(1, std::memory_order_relaxed);    \
    FMP_CHECK_CUDA(cudaGetLastError());                           \
  } while (0)
#define FMP_REQUIRE(cond, ...)                                                      \
  do {                                                                              \
    if (!(cond)) { ::fmp::set_error(__VA_ARGS__); return -2; }                      \
  } while (0)

inline bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] == '1';
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- programmatic dependent launch
// The hot-path kernels are launched with programmatic stream serialisation: a kernel may start
// (its CTAs load their resident factor tables, initialise barriers, prefetch tensor maps) while
// its predecessor on the stream is still finishing, and blocks in pdl_wait() until the
// predecessor has completed and its writes are visible.  Every kernel launched by launch_pdl()
// calls pdl_wait() in every CTA before touching data another kernel writes (and before its own
// global writes), so completion stays transitively ordered along the stream.  pdl_trigger()
// lets the successor launch once every CTA of this grid has started.  FMP_NO_PDL=1: ordinary
// launches (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" :::); }

inline bool pdl_on() {
  static const bool on = !getenv_flag("FMP_NO_PDL");
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  return launch_k(pdl_on(), kern, grid, block, smem, st, std::forward<Args>(args)...);
}

constexpr int kNumSM = 148;
// Fixed persistent-grid sizes keep every reduction's partial order independent of n.
constexpr int kVecGrid = 4 * kNumSM;      // vector kernels: 592 CTAs x 256 threads
constexpr int kVecThreads = 256;
constexpr int kStencilGrid = 8 * kNumSM;  // stencil: 1184 CTAs x 128 threads
constexpr int64_t kScratchDoubles = 16384;

// ---------------------------------------------------------------- field access
// Block-local read with the ghost shell of fmp_block (see flashmp_b200.h).
struct Geo {
  int bx, by, bz;
  int gx0, gy0, gz0;
  int nx, ny, nz;
  int P;
  const double* ghost[6];
};

inline Geo make_geo(const fmp_block* b) {
  Geo g;
  g.bx = (int)b->bx; g.by = (int)b->by; g.bz = (int)b->bz;
  g.gx0 = (int)b->gx0; g.gy0 = (int)b->gy0; g.gz0 = (int)b->gz0;
  g.nx = (int)b->nx; g.ny = (int)b->ny; g.nz = (int)b->nz;
  g.P = (int)b->halo;
  for (int q = 0; q < 6; ++q) g.ghost[q] = b->ghost[q];
  return g;
}

__device__ __forceinline__ int64_t fidx(const Geo& g, int c, int k, int j, int i) {
  return (((int64_t)c * g.bz + k) * g.by + j) * g.bx + i;
}

// Generic accessor: handles points outside the block (global zero ghost or neighbour ghosts).
__device__ __forceinline__ double fetch(const Geo& g, const double* __restrict__ f, int c, int k, int j,
                                        int i) {
  if ((unsigned)i < (unsigned)g.bx && (unsigned)j < (unsigned)g.by && (unsigned)k < (unsigned)g.bz)
    return __ldg(f + fidx(g, c, k, j, i));
  const int gi = g.gx0 + i, gj = g.gy0 + j, gk = g.gz0 + k;
  if ((unsigned)gi >= (unsigned)g.nx || (unsigned)gj >= (unsigned)g.ny || (unsigned)gk >= (unsigned)g.nz)
    return 0.0;
  const int P = g.P;
  if (i < 0 || i >= g.bx) {
    const double* s = i < 0 ? g.ghost[0] : g.ghost[1];
    if (!s) return 0.0;
    const int ii = i < 0 ? i + P : i - g.bx;
    return __ldg(s + ((((int64_t)c * (g.bz + 2 * P) + (k + P)) * (g.by + 2 * P) + (j + P)) * P + ii));
  }
  if (j < 0 || j >= g.by) {
    const double* s = j < 0 ? g.ghost[2] : g.ghost[3];
    if (!s) return 0.0;
    const int jj = j < 0 ? j + P : j - g.by;
    return __ldg(s + ((((int64_t)c * (g.bz + 2 * P) + (k + P)) * P + jj) * g.bx + i));
  }
  const double* s = k < 0 ? g.ghost[4] : g.ghost[5];
  if (!s) return 0.0;
  const int kk = k < 0 ? k + P : k - g.bz;
  return __ldg(s + ((((int64_t)c * P + kk) * g.by + j) * g.bx + i));
}

// Address of a block-local point for async copies: nullptr means "reads as zero"
// (outside the global box, or a missing ghost slab).  Same rules as fetch().
__device__ __forceinline__ const double* point_ptr(const Geo& g, const double* f, int c, int k, int j, int i) {
  if ((unsigned)i < (unsigned)g.bx && (unsigned)j < (unsigned)g.by && (unsigned)k < (unsigned)g.bz)
    return f + fidx(g, c, k, j, i);
  const int gi = g.gx0 + i, gj = g.gy0 + j, gk = g.gz0 + k;
  if ((unsigned)gi >= (unsigned)g.nx || (unsigned)gj >= (unsigned)g.ny || (unsigned)gk >= (unsigned)g.nz)
    return nullptr;
  const int P = g.P;
  if (i < 0 || i >= g.bx) {
    const double* s = i < 0 ? g.ghost[0] : g.ghost[1];
    if (!s) return nullptr;
    const int ii = i < 0 ? i + P : i - g.bx;
    return s + ((((int64_t)c * (g.bz + 2 * P) + (k + P)) * (g.by + 2 * P) + (j + P)) * P + ii);
  }
  if (j < 0 || j >= g.by) {
    const double* s = j < 0 ? g.ghost[2] : g.ghost[3];
    if (!s) return nullptr;
    const int jj = j < 0 ? j + P : j - g.by;
    return s + ((((int64_t)c * (g.bz + 2 * P) + (k + P)) * P + jj) * g.bx + i);
  }
  const double* s = k < 0 ? g.ghost[4] : g.ghost[5];
  if (!s) return nullptr;
  const int kk = k < 0 ? k + P : k - g.bz;
  return s + ((((int64_t)c * P + kk) * g.by + j) * g.bx + i);
}

// ---------------------------------------------------------------- cp.async (LDGSTS)
// 8-byte async global->shared copy; src == nullptr zero-fills the destination (the copy then
// reads 0 bytes from `valid`, any mapped global address).
__device__ __forceinline__ void cp_async8(double* dst, const double* src, const double* valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = src ? 8 : 0;
  const void* s = src ? (const void*)src : (const void*)valid;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(s), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------- numpy-faithful rounding
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// ---------------------------------------------------------------- reductions
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* smem) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) smem[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < NT / 32 ? smem[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// Final fixed-order reduction of `count` partial vectors of width `nd` (partials[q*count + b]).
int finish_reduce(const double* partials, int count, int nd, double* out, cudaStream_t st);

// ---------------------------------------------------------------- FP64 tensor-core MMA
// mma.sync m8n8k4 f64 (DMMA). Fragment maps (verified on B200, tools/fp64_probe.cu):
//  A(8x4):  lane -> (row g = lane>>2, col t = lane&3)
//  B(4x8):  lane -> (row t, col g)
//  C(8x8):  lane -> (row g, cols 2t, 2t+1)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace fmp
