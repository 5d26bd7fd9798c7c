// Tiling of a 3-way interval box (host and device share this code, so the
// C-ABI planner and the kernels can never disagree).
//
// For pivot j (the middle index) the valid (i, k) set is the rectangle
// [i0, min(i1, j)) x [max(k0, j+1), k1). Tiled on its own it leaves one
// ragged row tile and one ragged column tile per pivot -- ~6% of padded cells
// at n = 6000. Three layouts remove most of that:
//
// * PAIR (diagonal boxes: BM == BN and i0 = k0 mod BM). Pivot j is paired
//   with its MATE q = i0 + BM*R + (BM-1-r) (R, r = full row tiles and ragged
//   rows of j): their ragged rows (r + (BM-1-r) = BM-1) share one row-packed
//   tile per clean column tile, and their ragged leading columns share one
//   column-packed tile per full row tile.
// * FLAT_COLS (rows independent of j: i1 <= j0, e.g. the face and volume
//   units of the tetrahedral schedule). The (j, k) columns of all pivots are
//   laid end to end and cut into BN-wide tiles; a tile lies inside one pivot
//   (single-pivot CTA) or straddles two (a two-segment CTA). Pivots with
//   fewer than BN columns (the tail of J) keep one ragged tile each.
// * FLAT_ROWS (columns independent of j: j1 <= k0), the transpose: the (i, j)
//   rows are laid end to end; pivots with fewer than BM rows (the head of J)
//   keep one ragged tile each.
//
// Rows/columns of a two-segment tile carry their own pivot; since min is
// exact, applying the pivot on the column side instead of the row side gives
// the same n_ijk bit for bit.
#pragma once

#include <stdint.h>

#include "psim.h"

namespace psim {

enum { kBoxPlain = 0, kBoxPair = 1, kBoxFlatCols = 2, kBoxFlatRows = 3 };

struct Pivot3 {
  int64_t nrows, ncols, klo;  // rows [i0, i0 + nrows), columns [klo, k1)
  int64_t R, r;               // full row tiles / ragged rows (row tiles aligned at i0)
  int64_t Cc, Kc, w;          // first clean column tile (aligned at k0), clean tiles, ragged
                              // leading columns (the part of tile Cc-1 at or after klo)
  int64_t mate;               // paired pivot or -1
  int64_t tiles;              // single-pivot CTAs this pivot contributes (a pair's on its lower pivot)
  int64_t packed;             // packed (two-pivot) CTAs, likewise; launched as a separate grid
  // FLAT_* layouts: j's flattened span [f0, f1) along the flat axis, the tile
  // count across the fixed axis, whether j is on the flat axis at all, and
  // whether j's last tile straddles into pivot j+1 (then owned by j, packed)
  int64_t f0, f1, nfix;
  int flat, cross;
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
  g.f0 = g.f1 = g.nfix = 0;
  g.flat = g.cross = 0;
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

// sum_{x=a}^{b-1} x (0 when b <= a)
__host__ __device__ inline int64_t p3_span_sum(int64_t a, int64_t b) {
  return b > a ? (a + b - 1) * (b - a) / 2 : 0;
}

// Layout of a box (see the header comment). FLAT_COLS and FLAT_ROWS both
// apply to a volume box; take the one whose fixed axis pads less.
__host__ __device__ inline int box3_mode(int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                                         int64_t k0, int64_t k1, int64_t bm, int64_t bn) {
  const bool fc = i1 <= j0 && i1 > i0, fr = j1 <= k0 && k1 > k0;
  if (fc && fr) {
    const int64_t ni = i1 - i0, nk = k1 - k0;
    const int64_t pi = (ni + bm - 1) / bm * bm, pk = (nk + bn - 1) / bn * bn;
    return (pi - ni) * pk <= (pk - nk) * pi ? kBoxFlatCols : kBoxFlatRows;  // waste ratios
  }
  if (fc) return kBoxFlatCols;
  if (fr) return kBoxFlatRows;
  if (bm == bn && ((i0 - k0) % bm + bm) % bm == 0) return kBoxPair;
  return kBoxPlain;
}

// FLAT_COLS: flat pivots are [j0, jf) (ncols(j) >= bn, ncols non-increasing
// in j); F(j) = columns of the flat pivots before j.
__host__ __device__ inline int64_t p3_cols_jf(int64_t j0, int64_t j1, int64_t k0, int64_t k1,
                                              int64_t bn) {
  if (k0 > k1 - bn) return j0;
  return p3_max(j0, p3_min(j1, k1 - bn));
}
__host__ __device__ inline int64_t p3_cols_F(int64_t j0, int64_t k0, int64_t k1, int64_t j) {
  const int64_t a = p3_max(0, p3_min(j, k0) - j0);  // pivots j' < k0: k1 - k0 columns each
  const int64_t s = p3_max(j0, k0);                 // pivots j' >= k0: k1 - 1 - j' columns
  const int64_t m = p3_max(0, j - s);
  return a * (k1 - k0) + m * (k1 - 1) - p3_span_sum(s, j);
}
// FLAT_ROWS: flat pivots are [jh, j1) (nrows(j) >= bm, nrows non-decreasing
// in j); G(j) = rows of the flat pivots before j.
__host__ __device__ inline int64_t p3_rows_jh(int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                                              int64_t bm) {
  if (i1 - i0 < bm) return j1;
  return p3_max(j0, p3_min(j1, i0 + bm));
}
__host__ __device__ inline int64_t p3_rows_G(int64_t i0, int64_t i1, int64_t jh, int64_t j) {
  const int64_t ea = p3_min(j, i1);  // pivots j' < i1: j' - i0 rows
  const int64_t a = p3_max(0, ea - jh);
  const int64_t b = p3_max(0, j - p3_max(jh, i1));  // pivots j' >= i1: i1 - i0 rows
  return p3_span_sum(jh, p3_max(jh, ea)) - a * i0 + b * (i1 - i0);
}

__host__ __device__ inline int64_t p3_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Per-pivot counts of a FLAT_* box (g from pivot3_geom). Returns false when
// j is not on the flat axis (it then takes the plain per-pivot tiling).
__host__ __device__ inline bool pivot3_flat(int mode, int64_t i0, int64_t i1, int64_t j0,
                                            int64_t j1, int64_t k0, int64_t k1, int64_t bm,
                                            int64_t bn, int64_t j, Pivot3& g) {
  if (mode == kBoxFlatCols) {
    const int64_t jf = p3_cols_jf(j0, j1, k0, k1, bn);
    if (j >= jf || g.nrows <= 0) return false;
    g.nfix = p3_cdiv(g.nrows, bm);
    g.f0 = p3_cols_F(j0, k0, k1, j);
    g.f1 = g.f0 + g.ncols;
    g.cross = j + 1 < jf && g.f1 % bn != 0;
    const int64_t starts = p3_cdiv(g.f1, bn) - p3_cdiv(g.f0, bn);
    g.tiles = g.nfix * (starts - g.cross);
    g.packed = g.nfix * g.cross;
  } else {
    const int64_t jh = p3_rows_jh(i0, i1, j0, j1, bm);
    if (j < jh || g.ncols <= 0) return false;
    g.nfix = p3_cdiv(g.ncols, bn);
    g.f0 = p3_rows_G(i0, i1, jh, j);
    g.f1 = g.f0 + g.nrows;
    g.cross = j + 1 < j1 && g.f1 % bm != 0;
    const int64_t starts = p3_cdiv(g.f1, bm) - p3_cdiv(g.f0, bm);
    g.tiles = g.nfix * (starts - g.cross);
    g.packed = g.nfix * g.cross;
  }
  g.flat = 1;
  return true;
}

__host__ __device__ inline Pivot3 pivot3(int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                                         int64_t k0, int64_t k1, int64_t bm, int64_t bn,
                                         int64_t j) {
  Pivot3 g;
  pivot3_geom(i0, i1, k0, k1, bm, bn, j, g);
  const int mode = box3_mode(i0, i1, j0, j1, k0, k1, bm, bn);
  if ((mode == kBoxFlatCols || mode == kBoxFlatRows) &&
      pivot3_flat(mode, i0, i1, j0, j1, k0, k1, bm, bn, j, g))
    return g;
  if (mode == kBoxPair && g.nrows > 0 && g.ncols > 0 && j < i1 && j >= k0) {
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

// One CTA's tile: up to two row segments and two column segments, each with
// its own pivot on the segmented side (side 0: rows carry the pivot, the
// columns are one segment; side 1: columns carry it). A single-pivot tile is
// one row segment and one column segment.
struct Tile3 {
  int64_t p0, p1;      // pivots (global) of segment 0 / 1
  int64_t row0, row1;  // first global row of each row segment
  int64_t col0, col1;  // first global column of each column segment
  int nr0, nr1;        // row segment sizes (nr1 may be 0)
  int nc0, nc1;        // column segment sizes (nc1 may be 0)
  int side;            // 0: pivot per row segment, 1: pivot per column segment
};

// Prefix entry i; on the device a volatile load, so a decode repeated after
// the mainloop is recomputed rather than held live across it.
__host__ __device__ inline int64_t p3_pref(const int64_t* p, int64_t i) {
#ifdef __CUDA_ARCH__
  int64_t v;
  asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(v) : "l"(p + i));
  return v;
#else
  return p[i];
#endif
}

// The tile of CTA t of a box's single-pivot grid (PACKED = false) or
// two-segment grid (PACKED = true); tile_pref = per-pivot CTA prefix of that
// grid (pivot3's tiles / packed). Host copies serve the C-ABI tile query
// (psim_box3_tile), which the CPU tests use to check exact coverage.
template <int BM, int BN, bool PACKED>
__host__ __device__ inline Tile3 box3_decode(const psim_box3_t& b, const int64_t* tile_pref,
                                             int64_t nJ, int64_t t) {
  int64_t lo = 0, hi = nJ;  // largest lo with tile_pref[lo] <= t
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (p3_pref(tile_pref, mid) <= t) lo = mid; else hi = mid;
  }
  const int64_t j = b.j0 + lo;
  int64_t l = t - p3_pref(tile_pref, lo);
  const Pivot3 g = pivot3(b.i0, b.i1, b.j0, b.j1, b.k0, b.k1, BM, BN, j);
  Tile3 d;
  d.p0 = d.p1 = j;
  d.nr1 = d.nc1 = 0;
  d.row1 = d.col1 = 0;
  d.side = 0;
  if (g.flat) {  // FLAT_* layouts (box3_plan.cuh): tiles cut along the flattened axis
    const bool fc = box3_mode(b.i0, b.i1, b.j0, b.j1, b.k0, b.k1, BM, BN) == kBoxFlatCols;
    const int64_t blk = fc ? BN : BM;
    int64_t fix, fs;
    if (PACKED) {  // j's last flat tile, straddling into pivot j+1
      fix = l;
      fs = (p3_cdiv(g.f1, blk) - 1) * blk;
    } else {
      const int64_t nl = p3_cdiv(g.f1, blk) - p3_cdiv(g.f0, blk) - g.cross;
      fix = fc ? l / nl : l % g.nfix;
      fs = (p3_cdiv(g.f0, blk) + (fc ? l % nl : l / g.nfix)) * blk;
    }
    const int seg = (int)p3_min(blk, g.f1 - fs);  // j's part of the tile
    if (fc) {
      d.side = 1;
      d.row0 = b.i0 + fix * BM;
      d.nr0 = (int)p3_min(BM, g.nrows - fix * BM);
      d.col0 = g.klo + (fs - g.f0);
      d.nc0 = seg;
      if (PACKED) {
        d.p1 = j + 1;
        d.col1 = p3_max(b.k0, j + 2);
        d.nc1 = BN - seg;
      }
    } else {
      d.col0 = b.k0 + fix * BN;
      d.nc0 = (int)p3_min(BN, g.ncols - fix * BN);
      d.row0 = b.i0 + (fs - g.f0);
      d.nr0 = seg;
      if (PACKED) {
        d.p1 = j + 1;
        d.row1 = b.i0;
        d.nr1 = BM - seg;
      }
    }
    return d;
  }
  if (g.mate < 0) {  // single pivot: row tiles from i0, column tiles from klo
    const int64_t tiles_k = (g.ncols + BN - 1) / BN;
    const int64_t ti = l / tiles_k, tk = l - ti * tiles_k;
    d.row0 = b.i0 + ti * BM;
    d.col0 = g.klo + tk * BN;
    d.nr0 = (int)p3_min(BM, g.nrows - ti * BM);
    d.nc0 = (int)p3_min(BN, g.ncols - tk * BN);
    return d;
  }
  Pivot3 h;
  pivot3_geom(b.i0, b.i1, b.k0, b.k1, BM, BN, g.mate, h);
  const int64_t q = g.mate;
  auto clean_col = [&](int64_t ci, Tile3& x) {  // clean column tile Cc + ci
    x.col0 = b.k0 + (g.Cc + ci) * BN;
    x.nc0 = (int)p3_min(BN, b.k1 - x.col0);
  };
  if (!PACKED) {
    const int64_t nAB = 2 * g.R * g.Kc;
    if (l < nAB) {  // full tiles of j and q, interleaved (same panels)
      d.p0 = (l & 1) ? q : j;
      const int64_t rc = l >> 1, ri = rc / g.Kc;
      d.row0 = b.i0 + ri * BM;
      d.nr0 = BM;
      clean_col(rc - ri * g.Kc, d);
      return d;
    }
    l -= nAB;
    const bool e_j = g.r > 0 && g.w > 0;
    const bool own = (l == 0 && e_j);  // corner of j, else of q
    const Pivot3& x = own ? g : h;
    d.p0 = own ? j : q;
    d.row0 = b.i0 + g.R * BM;
    d.nr0 = (int)x.r;
    d.col0 = x.klo;
    d.nc0 = (int)x.w;
    return d;
  }
  const int64_t nC = g.r + h.r > 0 ? g.Kc : 0;
  if (l < nC) {  // ragged rows of both pivots in one tile
    d.p1 = q;
    d.row0 = d.row1 = b.i0 + g.R * BM;
    d.nr0 = (int)g.r;
    d.nr1 = (int)h.r;
    clean_col(l, d);
    return d;
  }
  l -= nC;
  {  // ragged leading columns of both pivots in one tile (l < R when g.w + h.w > 0)
    d.side = 1;
    d.p1 = q;
    d.row0 = b.i0 + l * BM;
    d.nr0 = BM;
    d.col0 = g.klo;
    d.nc0 = (int)g.w;
    d.col1 = h.klo;
    d.nc1 = (int)h.w;
  }
  return d;
}

}  // namespace psim
