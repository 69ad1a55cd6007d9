// Multi-GPU ghost-shell exchange: pack and unpack kernels (K10; replaces the reference's
// in-process Exchanger messages, ref:schwarz.py:217-257).
//
// A block's ghost shell (width P, layout in fmp_block) is filled in three phases -- z faces,
// then y faces extended over the z ghosts, then x faces extended over both -- so edges and
// corners arrive without diagonal messages.  Every slab a rank sends is produced by ONE pack
// launch that reads its owned field and the ghosts of the earlier phases through fetch(), the
// same accessor the stencil and subdomain kernels use, so the slab holds exactly what the
// neighbour's kernels will read.  Each slab carries a trailing tag (epoch * 3 + phase); the
// receiver's unpack checks it, so a lost or stale message is detected on the device and
// reported through a host-mapped status word (raised as CommunicationError by the host).
//
// Roofline: HBM-bound copies, 16 B per slab element (read + write); the slabs are 1-3 % of a
// 256^3 block per phase and overlap interior work (fmp_precond_apply_part / fmp_stencil_apply_part).
#include "common.cuh"
#include <algorithm>

namespace fmp {

struct SlabGeo {
  int n3, n2, n1;      // slab extents (slowest .. fastest) after the component index
  int k0, j0, i0;      // block-local coordinates of slab element (0, 0, 0)
};

static SlabGeo slab_geo(const fmp_block* b, int phase, int side) {
  const int P = (int)b->halo, bx = (int)b->bx, by = (int)b->by, bz = (int)b->bz;
  SlabGeo s{};
  if (phase == 0) {          // z: (3, P, by, bx), own planes [0, P) or [bz - P, bz)
    s = {P, by, bx, side ? bz - P : 0, 0, 0};
  } else if (phase == 1) {   // y: (3, bz + 2P, P, bx), own rows, extended over the z ghosts
    s = {bz + 2 * P, P, bx, -P, side ? by - P : 0, 0};
  } else {                   // x: (3, bz + 2P, by + 2P, P), own columns, extended over y and z ghosts
    s = {bz + 2 * P, by + 2 * P, P, -P, -P, side ? bx - P : 0};
  }
  return s;
}

__global__ void k_halo_pack(Geo g, SlabGeo s, const double* __restrict__ x, double* __restrict__ out, double tag,
                            int64_t n) {
  const int64_t per_c = (int64_t)s.n3 * s.n2 * s.n1;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q / per_c);
    int64_t r = q - c * per_c;
    const int a3 = (int)(r / ((int64_t)s.n2 * s.n1));
    r -= (int64_t)a3 * s.n2 * s.n1;
    const int a2 = (int)(r / s.n1), a1 = (int)(r - (int64_t)a2 * s.n1);
    out[q] = fetch(g, x, c, s.k0 + a3, s.j0 + a2, s.i0 + a1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = tag;
}

__global__ void k_halo_unpack(const double* __restrict__ in, double* __restrict__ ghost, int64_t n, double tag,
                              int* status, int bit) {
  if (in != ghost)
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= n; q += (int64_t)gridDim.x * blockDim.x)
      ghost[q] = in[q];
  if (blockIdx.x == 0 && threadIdx.x == 0 && in[n] != tag && status) atomicOr(status, bit);
}

}  // namespace fmp

using namespace fmp;

static int halo_check(const fmp_block* b, int phase, int side) {
  FMP_REQUIRE(b && b->bx >= 1 && b->by >= 1 && b->bz >= 1, "invalid block extents");
  FMP_REQUIRE(phase >= 0 && phase <= 2 && (side == 0 || side == 1), "bad halo phase %d / side %d", phase, side);
  FMP_REQUIRE(b->halo >= 1 && b->halo <= b->bx && b->halo <= b->by && b->halo <= b->bz,
              "halo width %lld outside [1, block extent]", (long long)b->halo);
  return 0;
}

extern "C" int64_t fmp_halo_slab_doubles(const fmp_block* blk, int phase) {
  if (halo_check(blk, phase, 0)) return -2;
  const SlabGeo s = slab_geo(blk, phase, 0);
  return 3 * (int64_t)s.n3 * s.n2 * s.n1;
}

extern "C" int fmp_halo_pack(const fmp_block* blk, int phase, int side, const double* x, double* out, double tag,
                             void* stream) {
  if (int e = halo_check(blk, phase, side)) return e;
  FMP_REQUIRE(x && out, "null field or slab");
  const SlabGeo s = slab_geo(blk, phase, side);
  const int64_t n = 3 * (int64_t)s.n3 * s.n2 * s.n1;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 4 * kNumSM);
  k_halo_pack<<<grid, 256, 0, as_stream(stream)>>>(make_geo(blk), s, x, out, tag, n);
  FMP_CHECK_LAUNCH();
  return 0;
}

extern "C" int fmp_halo_unpack(const fmp_block* blk, int phase, int side, const double* in, double tag, int* status,
                               void* stream) {
  if (int e = halo_check(blk, phase, side)) return e;
  const int slot = (phase == 0 ? 4 : phase == 1 ? 2 : 0) + side;
  double* ghost = const_cast<double*>(blk->ghost[slot]);
  FMP_REQUIRE(in && ghost, "halo unpack needs the received slab and ghost slot %d", slot);
  const SlabGeo s = slab_geo(blk, phase, side);
  const int64_t n = 3 * (int64_t)s.n3 * s.n2 * s.n1;
  const int grid = in == ghost ? 1 : (int)std::min<int64_t>((n + 256) / 256, 4 * kNumSM);
  k_halo_unpack<<<grid, 256, 0, as_stream(stream)>>>(in, ghost, n, tag, status, 1 << slot);
  FMP_CHECK_LAUNCH();
  return 0;
}
