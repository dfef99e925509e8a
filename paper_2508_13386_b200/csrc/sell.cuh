// SELL-32 layout of the 3x3-block Hessian (B200 design).
//
// Rows are grouped in slices of 32 consecutive vertices; slice s has L_s = max row length
// block-columns starting at column sl_ptr[s].  Block j of row r (lane l = r % 32) lives at
// position pos = (sl_ptr[r/32] + j) * 32 + l: its column index at col[pos] and its 9 entries at
// vals[((sl_ptr[r/32] + j) * 9 + q) * 32 + l], q = 3 * row_in_block + col_in_block.  A warp
// handling one slice (thread per row) therefore reads every index / value plane with one fully
// coalesced 128 / 256-byte access per block-column, with no shuffles and no dependent row
// pointer chain.  Padding entries (rows shorter than L_s) have col = r and zero values.
#pragma once
#include <stdint.h>

namespace msim {

struct SellView {
  int nv;
  const int32_t *__restrict__ sl_ptr;
  const int32_t *__restrict__ col;
  const double *__restrict__ vals;
};

__device__ __forceinline__ size_t sell_val_index(int c, int q, int lane) {
  return ((size_t)c * 9 + q) * 32 + lane;
}

}  // namespace msim
