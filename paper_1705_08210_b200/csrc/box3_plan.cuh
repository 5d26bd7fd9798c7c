// Tiling of a 3-way interval box (host and device share this code, so the
// C-ABI planner and the kernels can never disagree).
//
// For pivot j (the middle index) the valid (i, k) set is the rectangle
// [i0, min(i1, j)) x [max(k0, j+1), k1). Tiled on its own it leaves one
// ragged row tile and one ragged column tile per pivot -- ~6% of padded cells
// at n = 6000. When the box allows (BM == BN and i0 = k0 mod BM), pivot j is
// paired with its MATE q = i0 + BM*R + (BM-1-r) (R, r = full row tiles and
// ragged rows of j): their ragged rows (r + (BM-1-r) = BM-1) share one
// row-packed tile per clean column tile, and their ragged leading columns
// share one column-packed tile per full row tile. Rows/columns of a packed
// tile carry their own pivot; since min is exact, applying the pivot on the
// column side instead of the row side gives the same n_ijk bit for bit.
#pragma once

#include <stdint.h>

namespace psim {

struct Pivot3 {
  int64_t nrows, ncols, klo;  // rows [i0, i0 + nrows), columns [klo, k1)
  int64_t R, r;               // full row tiles / ragged rows (row tiles aligned at i0)
  int64_t Cc, Kc, w;          // first clean column tile (aligned at k0), clean tiles, ragged
                              // leading columns (the part of tile Cc-1 at or after klo)
  int64_t mate;               // paired pivot or -1
  int64_t tiles;              // single-pivot CTAs this pivot contributes (a pair's on its lower pivot)
  int64_t packed;             // packed (two-pivot) CTAs, likewise; launched as a separate grid
};

__host__ __device__ inline int64_t p3_min(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t p3_max(int64_t a, int64_t b) { return a > b ? a : b; }

__host__ __device__ inline void pivot3_geom(int64_t i0, int64_t i1, int64_t k0, int64_t k1,
                                            int64_t bm, int64_t bn, int64_t j, Pivot3& g) {
  g.klo = p3_max(k0, j + 1);
  g.nrows = p3_max(0, p3_min(i1, j) - i0);
  g.ncols = p3_max(0, k1 - g.klo);
  g.R = g.nrows / bm;
  g.r = g.nrows % bm;
  const int64_t off = g.klo - k0, f = off % bn;
  g.Cc = (off + bn - 1) / bn;
  g.w = f ? p3_min(bn - f, g.ncols) : 0;
  g.Kc = p3_max(0, (k1 - k0 + bn - 1) / bn - g.Cc);
  g.mate = -1;
  g.tiles = 0;
  g.packed = 0;
}

// Tiles of a packed pair (leader g, mate h). Single-pivot CTAs: A/B full
// tiles of each pivot (interleaved), E/F the two corners (ragged rows x
// ragged columns of one pivot). Packed CTAs: C row-packed ragged rows (one
// per clean column tile), D column-packed ragged columns (one per full row
// tile).
__host__ __device__ inline int64_t pair3_single(const Pivot3& g, const Pivot3& h) {
  return 2 * g.R * g.Kc + (g.r > 0 && g.w > 0) + (h.r > 0 && h.w > 0);
}
__host__ __device__ inline int64_t pair3_packed(const Pivot3& g, const Pivot3& h) {
  return (g.r + h.r > 0 ? g.Kc : 0) + (g.w + h.w > 0 ? g.R : 0);
}

__host__ __device__ inline Pivot3 pivot3(int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                                         int64_t k0, int64_t k1, int64_t bm, int64_t bn,
                                         int64_t j) {
  Pivot3 g;
  pivot3_geom(i0, i1, k0, k1, bm, bn, j, g);
  const bool pack = bm == bn && ((i0 - k0) % bm + bm) % bm == 0;
  if (pack && g.nrows > 0 && g.ncols > 0 && j < i1 && j >= k0) {
    const int64_t q = i0 + bm * g.R + (bm - 1 - g.r);
    if (q != j && q >= j0 && q < j1 && q < i1 && q >= k0) {
      Pivot3 h;
      pivot3_geom(i0, i1, k0, k1, bm, bn, q, h);
      if (h.nrows > 0 && h.ncols > 0 && h.R == g.R && h.Cc == g.Cc && h.Kc == g.Kc &&
          g.w + h.w <= bn && g.r + h.r <= bm) {
        g.mate = q;
        g.tiles = q < j ? 0 : pair3_single(g, h);
        g.packed = q < j ? 0 : pair3_packed(g, h);
        return g;
      }
    }
  }
  g.tiles = (g.nrows > 0 && g.ncols > 0) ? ((g.nrows + bm - 1) / bm) * ((g.ncols + bn - 1) / bn)
                                         : 0;
  return g;
}

}  // namespace psim
