// Host interface of the Ozaki INT8 tensor-core Woodbury GEMM (ozaki.cu), used by precond.cu.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace fmp {

struct OzShape {
  const int8_t* A;   // tiled slices of C^-1: [mtile][kchunk][S][128 x 32 B]
  const int* eA;     // [m] row exponents of C^-1
  const int8_t* B;   // tiled slices of Y: [ntile][kchunk][S][w x 32 B]
  const int* eB;     // [n] row exponents of Y^T
  double* Z;         // [n][ld]
  int m, n, ld, kchunks, w, pad;   // w: column-tile width (multiple of 16, S*w <= 512)
};
struct OzTile {
  int shape, mt, nt, kpart;   // kpart: K part (chunks [kpart * 512, ...)) for K > 16384
};
// One operand to slice: rows x kvalid doubles (row stride ld) -> tiles of height T.
struct OzSlice {
  const double* src;
  int8_t* dst;
  int* exps;
  int rows, ld, kvalid, kchunks, T, stacked;   // stacked = 1: slices stacked along N (B operand)
  int64_t row0, q0;   // prefix offsets of this operand in the batched exponent / digit grids
  int64_t prow0;      // prefix of padded rows (tile multiples) in the batched slicing grid
};

int ozaki_setup();
int ozaki_kchunks(int m);
int ozaki_kparts(int kchunks);                 // K parts of <= 16384 bytes (int32 level headroom)
int ozaki_tile_m();
int ozaki_width(int n);                       // column-tile width for n columns
size_t ozaki_a_bytes(int m, int kchunks);
size_t ozaki_b_bytes(int n, int kchunks);
// Fill row0/q0/prow0 of a batch; returns the total rows and padded rows (the slicing grid).
void ozaki_plan_slices(OzSlice* s, int count, int64_t* rows, int64_t* padded_rows);
int ozaki_slice(const OzSlice* d_slices, int count, int64_t rows, int64_t padded_rows, cudaStream_t st);
// tiles reordered into per-CTA lists (CTA b runs tiles [offs[b], offs[b+1])), balanced by cost
void ozaki_schedule(const std::vector<OzShape>& shapes, std::vector<OzTile>& tiles, int grid, std::vector<int>& offs);
int ozaki_launch(const OzShape* shapes, const OzTile* tiles, const int* offs, int grid, cudaStream_t st);

}  // namespace fmp
