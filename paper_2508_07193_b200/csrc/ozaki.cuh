// Host interface of the Ozaki INT8 tensor-core Woodbury GEMM (ozaki.cu), used by precond.cu.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace fmp {

struct OzShape {
  const int8_t* A;   // tiled slices of C^-1: [mtile][kchunk][S][128 x 32 B]
  const int* eA;     // [m] row exponents of C^-1
  const int8_t* B;   // tiled slices of Y: [ntile][kchunk][2 K halves][R stacked rows x 16 B]
  const int* eB;     // [n] row exponents of Y^T
  double* Z;         // [n][ld]
  int m, n, ld, kchunks, w, R;   // w: column-tile width (multiple of 8, <= 72); R = pad16(S w) stacked B rows
  // Zero-slice skipping: the K chunks of row tile mt whose C^-1 slices are not all zero are
  // klist[koff[mt] .. koff[mt+1]) (ascending), kp0 the number of leading all-zero slices of each
  // (those slices and their MMAs are skipped: their digits contribute exactly zero).
  const uint16_t* klist;
  const uint8_t* kp0;
  const int* koff;
  // Row/column order of the GEMM (ozaki_row_order): position i of the sliced C^-1 / of the K axis
  // is correction row perm[i]; Z is written back through it.  null = identity.
  const int* perm;
};
// Host copy of one shape's chunk lists (ozaki_chunk_lists -> ozaki_build).
struct OzLists {
  std::vector<uint16_t> klist;
  std::vector<uint8_t> kp0;
  std::vector<int> koff;
};
// One work item: list entries [k0, k1) of row tile mt (K chunks klist[koff[mt] + j]), column
// tile nt.  A tile whose list is split into nseg > 1 segments (load balance, or more than 16384
// K terms: int32 headroom) writes per-segment FP64 partials to partial slots slot0 + seg; the last
// segment to finish sums them in segment order (deterministic) into Z.  nseg == 1: the item
// writes Z directly.
struct OzItem {
  int shape, mt, nt, k0, k1, seg, nseg, slot0;
};
// Device tables of one batched Ozaki GEMM (all rotation groups of a plan).
struct OzPlan {
  OzShape* shapes = nullptr;
  OzItem* items = nullptr;
  int* offs = nullptr;        // CTA b runs items [offs[b], offs[b+1])
  double* zpart = nullptr;    // [slots][OZ_WMAX][128] partial results of split tiles
  int* counters = nullptr;    // [slots] arrivals per split tile (slot0), zero at rest
  uint16_t* klist = nullptr;  // chunk lists of all shapes (OzShape::klist / kp0 / koff point in)
  uint8_t* kp0 = nullptr;
  int* koff = nullptr;
  int grid = 0, n_items = 0, n_slots = 0;
  double kept_slices = 1.0;   // fraction of C^-1 slice blocks streamed (diagnostics)
  double kept_mma = 1.0;      // fraction of the dense MMA work (28 slice products) issued
};
// One operand to slice: rows x kvalid doubles (row stride ld) -> tiles of height T.
struct OzSlice {
  const double* src;
  int8_t* dst;
  int* exps;
  const int* rperm;   // row r of the operand is source row rperm[r] (null = identity)
  const int* kperm;   // K position k is source column kperm[k] (null = identity)
  int rows, ld, kvalid, kchunks, T, stacked;   // stacked = 1: slices stacked along N (B operand)
  int R;              // stacked: rows per K half of a (tile, kchunk) block (>= S * T, zero padding)
  int64_t row0, q0;   // prefix offsets of this operand in the batched exponent / digit grids
  int64_t prow0;      // prefix of padded rows (tile multiples) in the batched slicing grid
};

int ozaki_setup();
int ozaki_kchunks(int m);
int ozaki_tile_m();
int ozaki_width(int n);                       // column-tile width for n columns
int ozaki_stack_rows(int w);                  // R: stacked B rows of a column tile of width w
size_t ozaki_a_bytes(int m, int kchunks);
size_t ozaki_b_bytes(int n, int kchunks);
// Fill row0/q0/prow0 of a batch; returns the total rows and padded rows (the slicing grid).
void ozaki_plan_slices(OzSlice* s, int count, int64_t* rows, int64_t* padded_rows);
int ozaki_slice(const OzSlice* d_slices, int count, int64_t rows, int64_t padded_rows, cudaStream_t st);
// After the C^-1 slices exist: per row tile, the K chunks with a non-zero slice and their
// leading all-zero slice counts (FMP_OZ_DENSE=1: every chunk, no skipping); uploads the lists
// into `plan` and points the shapes at them.  Returns 0 or -1.
int ozaki_chunk_lists(std::vector<OzShape>& shapes, std::vector<OzLists>* lists, OzPlan* plan);
// Locality order of the m correction rows of a box (ex, ey, ez): the rows (reference order:
// component-major, ascending linear index) sorted by the Morton code of their point (i, j, k),
// component last, so the points C^-1 couples strongly -- the same or nearby places, every
// component -- share 128-row tiles and 32-column chunks, and fewer slice blocks are non-zero
// (FMP_OZ_NOPERM=1: reference order).  Returns perm with position -> reference row.
std::vector<int> ozaki_row_order(int ex, int ey, int ez);
// Work items (column tiles x list segments) for the shapes (entries with n == 0 are skipped),
// balanced over `sms` persistent CTAs, uploaded with the partial-slot workspace.  `plan` already
// holds the chunk lists (ozaki_chunk_lists).  Returns 0 or -1.
int ozaki_build(const std::vector<OzShape>& shapes, const std::vector<OzLists>& lists, int sms, OzPlan* plan);
void ozaki_free(OzPlan* p);
int ozaki_launch(const OzPlan& p, cudaStream_t st);

}  // namespace fmp
