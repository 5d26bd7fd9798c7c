// 3-way Czekanowski kernel over one interval box of the tetrahedral schedule.
//
// Reference path replaced (one SliceTask3 of run_3way, metrics3.py:131-192):
//   X_j = min(v_j, V_b)        xj_columns            mingemm.py:225-234
//   n'_3 = dense(X_j, V_c)     _blocked_kernel       mingemm.py:94-117, metrics3.py:163
//   Eq. 1 assembly             metrics3.py:167-182   (1.5*(((n_ij+n_ik)+n_jk)-n_ijk)) /
//                                                    ((s_i+s_j)+s_k), canonical i<j<k roles
//   cells / records            metrics3.py:183-191, checksum verify.py:86-96
//
// A box is every (i, j, k) in I x J x K with i < j < k (each schedule unit --
// diagonal-edge sixth, face sixth, volume slice, and their stage sub-ranges
// -- is one such box, see schedule.py:231-263). The kernel pivots on the
// MIDDLE index j: for fixed j the valid (i, k) set is the rectangle
// [i0, min64(i1, j)) x [max(k0, j+1), k1), so no tile is triangular. The
// pivot column is min-combined into the staged A tile in shared memory, and
// the mainloop is exactly the 2-way min-plus mainloop.
//
// Bitwise argument (SURVEY Appendix C rule 8): n_ijk = sum_q min(min(x_j, v_i), v_k)
// in ascending q is role-independent because min is exact; n_ij, n_ik, n_jk
// come from 2-way numerator tables whose entries equal the reference's
// column_sums(Xb) / P_bc bit for bit; the assembly uses canonical roles.
//
// Output layout ("pivot-major"): for j in J, the rectangle rows i, columns k
// row-major, at out_pref[j - j0].
#include "minplus.cuh"
#include "psim_internal.h"

namespace psim {

// Eq. 1 for one triple (metrics3.py:38-44 with canonical roles i<j<k,
// metrics3.py:146, 175-182): local columns ai (block A), jb (B), kc (C).
template <typename T>
__device__ __forceinline__ T czek3_value(const Czek3Box& b, int64_t ai, int64_t jb, int64_t kc,
                                         T n_ijk, bool& zero) {
  const T* SA = static_cast<const T*>(b.SA);
  const T* SB = static_cast<const T*>(b.SB);
  const T* SC = static_cast<const T*>(b.SC);
  const T nij = static_cast<const T*>(b.NAB)[ai + jb * b.ldAB];
  const T nik = static_cast<const T*>(b.NAC)[ai + kc * b.ldAC];
  const T njk = static_cast<const T*>(b.NBC)[jb + kc * b.ldBC];
  const T d = Traits<T>::add(Traits<T>::add(SA[ai], SB[jb]), SC[kc]);
  const T n3 = Traits<T>::sub(Traits<T>::add(Traits<T>::add(nij, nik), njk), n_ijk);
  zero = (d == T(0));
  return zero ? T(0) : Traits<T>::div(Traits<T>::mul(T(1.5), n3), d);
}

// One CTA's tile of a box: pivot j (index lo in the box's J range), the
// tile's rows / cols, and their local columns in blocks A / C.
struct Tile3 {
  int64_t lo, j, ncols, r0, c0, ia, kc, jb;
  int rows, cols;
};

// tile_pref is read with volatile loads (ld_pref) so the second decode after
// the mainloop is recomputed, not kept live in registers across it.
template <class C>
__device__ __forceinline__ Tile3 decode3(const Czek3Box& b, const int64_t* tile_pref, int64_t nJ) {
  Tile3 d;
  // locate pivot j: largest lo with tile_pref[lo] <= blockIdx.x
  const int64_t t = blockIdx.x;
  int64_t lo = 0, hi = nJ;  // invariant tile_pref[lo] <= t < tile_pref[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (ld_pref(tile_pref + mid) <= t) lo = mid; else hi = mid;
  }
  d.lo = lo;
  d.j = b.j0 + lo;
  const int64_t ihi = min64(b.i1, d.j);
  const int64_t klo = max64(b.k0, d.j + 1);
  const int64_t nrows = ihi - b.i0;
  d.ncols = b.k1 - klo;
  const int64_t tiles_k = (d.ncols + C::BN - 1) / C::BN;
  const int64_t lt = t - ld_pref(tile_pref + lo);
  const int64_t ti = lt / tiles_k, tk = lt - ti * tiles_k;
  d.r0 = ti * C::BM;
  d.c0 = tk * C::BN;
  d.rows = (int)min64(C::BM, nrows - d.r0);
  d.cols = (int)min64(C::BN, d.ncols - d.c0);
  d.ia = b.i0 - b.a0 + d.r0;   // local column of the tile's first i in block A
  d.kc = klo - b.c0 + d.c0;    // local column of the tile's first k in block C
  d.jb = d.j - b.b0;           // local column of j in block B
  return d;
}

// RAW = true writes the n_ijk partial sums (field-split path) instead of values.
template <class C, bool RAW>
__global__ void __launch_bounds__(kNT, C::MINB)
    k_czek3(const Czek3Box b, const int64_t* __restrict__ tile_pref,
            const int64_t* __restrict__ out_pref, int64_t nJ) {
  using T = typename C::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);

  T acc[C::TM][C::TN];
  {
    const Tile3 d = decode3<C>(b, tile_pref, nJ);
    minplus_tile<C, true>(static_cast<const T*>(b.VA) + d.ia * b.ldA, b.ldA, d.rows,
                          static_cast<const T*>(b.VC) + d.kc * b.ldC, b.ldC, d.cols,
                          static_cast<const T*>(b.VB) + d.jb * b.ldB, b.n_f, acc, smem);
  }
  // decoded again (measured: keeping the tile state live across the mainloop
  // costs registers and ~4% of the mainloop's issue rate)
  const Tile3 d = decode3<C>(b, tile_pref, nJ);
  const int64_t lo = d.lo, j = d.j, ncols = d.ncols, r0 = d.r0, c0 = d.c0;
  const int64_t ia = d.ia, kc = d.kc, jb = d.jb;
  const int rows = d.rows, cols = d.cols;

  T* out = static_cast<T*>(b.vals);
  const int64_t obase = out_pref[lo];
  const uint64_t nv = (uint64_t)b.n_v;

  const int ty = thread_ty(), tx = thread_tx();
  if (RAW) {
#pragma unroll
    for (int mi = 0; mi < C::TM; ++mi) {
      const int li = ty + 16 * mi;
      if (li >= rows) continue;
      const int64_t orow = obase + (r0 + li) * ncols + c0;
#pragma unroll
      for (int nk = 0; nk < C::TN; ++nk) {
        const int lk = tx + 16 * nk;
        if (lk < cols) out[orow + lk] = acc[mi][nk];
      }
    }
    return;
  }
  Cks c;
#pragma unroll
  for (int mi = 0; mi < C::TM; ++mi) {
    const int li = ty + 16 * mi;
    if (li >= rows) continue;
    const int64_t ai = ia + li;            // local in A
    const int64_t i = b.a0 + ai;           // global
    // triple_index(i, j, k) = base_ij + (k - j - 1), base_ij = C3(n)-C3(n-i)+pair_index(j-i-1, j-i, n-i-1)
    const uint64_t base_ij = choose3(nv) - choose3(nv - (uint64_t)i) +
                             pair_index((uint64_t)(j - i - 1), (uint64_t)(j - i), nv - (uint64_t)i - 1);
    const int64_t orow = obase + (r0 + li) * ncols + c0;
#pragma unroll
    for (int nk = 0; nk < C::TN; ++nk) {
      const int lk = tx + 16 * nk;
      if (lk >= cols) continue;
      const int64_t kcl = kc + lk;          // local in C
      const int64_t k = b.c0 + kcl;         // global
      bool zero;
      const T v = czek3_value<T>(b, ai, jb, kcl, acc[mi][nk], zero);
      if (out) out[orow + lk] = v;
      c.term(base_ij + (uint64_t)(k - j - 1), Traits<T>::bits(v));
      c.deg += zero ? 1ull : 0ull;
    }
  }
  cks_block_flush<kNT>(b.acc, c);
}

// Values + checksum for elements [e0, e1) of a box's pivot-major layout from
// already-folded n_ijk sums (the 3-way field-split path: partial n_ijk ->
// ordered fold over p_f -> this epilogue; metrics3.py:163-182). N3 and vals
// point at element e0. out_pref: the box's per-pivot output prefix (device).
template <typename T>
__global__ void __launch_bounds__(256) k_czek3_from_num(const Czek3Box b,
                                                        const int64_t* __restrict__ out_pref,
                                                        int64_t nJ, const T* __restrict__ N3,
                                                        int64_t e0, int64_t e1, T* __restrict__ vals) {
  Cks c;
  const uint64_t nv = (uint64_t)b.n_v;
  for (int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nJ;  // largest lo with out_pref[lo] <= e
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (out_pref[mid] <= e) lo = mid; else hi = mid;
    }
    const int64_t j = b.j0 + lo;
    const int64_t klo = max64(b.k0, j + 1);
    const int64_t ncols = b.k1 - klo;
    const int64_t off = e - out_pref[lo];
    const int64_t i = b.i0 + off / ncols, k = klo + off % ncols;
    bool zero;
    const T v = czek3_value<T>(b, i - b.a0, j - b.b0, k - b.c0, N3[e - e0], zero);
    if (vals) vals[e - e0] = v;
    c.term(triple_index((uint64_t)i, (uint64_t)j, (uint64_t)k, nv), Traits<T>::bits(v));
    c.deg += zero ? 1ull : 0ull;
  }
  cks_block_flush<256>(b.acc, c);
}

// Per-pivot prefix sums of CTA tiles and output elements for a box, one CTA:
// each thread folds a contiguous j range, then a block scan of the partials.
__global__ void __launch_bounds__(1024) k_box3_prefix(int64_t i0, int64_t i1, int64_t j0,
                                                      int64_t j1, int64_t k0, int64_t k1, int64_t bm, int64_t bn,
                                                      int64_t* __restrict__ tile_pref,
                                                      int64_t* __restrict__ out_pref) {
  __shared__ int64_t s_t[1024], s_o[1024];
  const int64_t nJ = j1 - j0;
  const int64_t per = (nJ + blockDim.x - 1) / blockDim.x;
  const int64_t a = min64(nJ, threadIdx.x * per), e = min64(nJ, a + per);
  auto counts = [&](int64_t jj, int64_t& t, int64_t& o) {
    const int64_t j = j0 + jj;
    const int64_t r = max64(0, min64(i1, j) - i0);
    const int64_t c = max64(0, k1 - max64(k0, j + 1));
    t = ((r + bm - 1) / bm) * ((c + bn - 1) / bn);
    o = r * c;
  };
  int64_t st = 0, so = 0;
  for (int64_t jj = a; jj < e; ++jj) {
    int64_t t, o;
    counts(jj, t, o);
    st += t;
    so += o;
  }
  s_t[threadIdx.x] = st;
  s_o[threadIdx.x] = so;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // inclusive Hillis-Steele scan
    int64_t vt = threadIdx.x >= off ? s_t[threadIdx.x - off] : 0;
    int64_t vo = threadIdx.x >= off ? s_o[threadIdx.x - off] : 0;
    __syncthreads();
    s_t[threadIdx.x] += vt;
    s_o[threadIdx.x] += vo;
    __syncthreads();
  }
  int64_t rt = threadIdx.x ? s_t[threadIdx.x - 1] : 0;
  int64_t ro = threadIdx.x ? s_o[threadIdx.x - 1] : 0;
  for (int64_t jj = a; jj < e; ++jj) {
    tile_pref[jj] = rt;
    out_pref[jj] = ro;
    int64_t t, o;
    counts(jj, t, o);
    rt += t;
    ro += o;
  }
  if (threadIdx.x == blockDim.x - 1) {
    tile_pref[nJ] = s_t[threadIdx.x];
    out_pref[nJ] = s_o[threadIdx.x];
  }
}

template <typename T, bool RAW>
static cudaError_t czek3_t(const Czek3Box& b, int64_t* work, int64_t n_tiles, cudaStream_t st) {
  using C = typename Prod<T>::C;
  cudaError_t e = cudaFuncSetAttribute(k_czek3<C, RAW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  if (n_tiles <= 0) return cudaSuccess;
  if (n_tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const int64_t nJ = b.j1 - b.j0;
  int64_t* tp = work;
  int64_t* op = work + nJ + 1;
  k_box3_prefix<<<1, 1024, 0, st>>>(b.i0, b.i1, b.j0, b.j1, b.k0, b.k1, C::BM, C::BN, tp, op);
  k_czek3<C, RAW><<<(unsigned)n_tiles, kNT, C::SMEM_BYTES, st>>>(b, tp, op, nJ);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t czek3_from_num_t(const Czek3Box& b, int64_t* work, const void* n3, int64_t e0,
                                    int64_t e1, void* vals, cudaStream_t st) {
  using C = typename Prod<T>::C;
  if (e1 <= e0) return cudaSuccess;
  const int64_t nJ = b.j1 - b.j0;
  int64_t* tp = work;
  int64_t* op = work + nJ + 1;
  k_box3_prefix<<<1, 1024, 0, st>>>(b.i0, b.i1, b.j0, b.j1, b.k0, b.k1, C::BM, C::BN, tp, op);
  int64_t blocks = (e1 - e0 + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_czek3_from_num<T><<<(unsigned)blocks, 256, 0, st>>>(b, op, nJ, static_cast<const T*>(n3), e0,
                                                        e1, static_cast<T*>(vals));
  return cudaGetLastError();
}

cudaError_t czek3_box_numerators(int dtype, const Czek3Box& b, int64_t* d_work, int64_t n_tiles,
                                 cudaStream_t st) {
  return dtype == kF64 ? czek3_t<double, true>(b, d_work, n_tiles, st)
                       : czek3_t<float, true>(b, d_work, n_tiles, st);
}

cudaError_t czek3_from_num(int dtype, const Czek3Box& b, int64_t* d_work, const void* n3,
                           int64_t e0, int64_t e1, void* vals, cudaStream_t st) {
  return dtype == kF64 ? czek3_from_num_t<double>(b, d_work, n3, e0, e1, vals, st)
                       : czek3_from_num_t<float>(b, d_work, n3, e0, e1, vals, st);
}

void tile_shape(int dtype, int* bm, int* bn) {
  if (dtype == kF64) {
    *bm = Prod<double>::C::BM;
    *bn = Prod<double>::C::BN;
  } else {
    *bm = Prod<float>::C::BM;
    *bn = Prod<float>::C::BN;
  }
}

cudaError_t czek3_box(int dtype, const Czek3Box& b, int64_t* d_work, int64_t n_tiles,
                      cudaStream_t st) {
  return dtype == kF64 ? czek3_t<double, false>(b, d_work, n_tiles, st)
                       : czek3_t<float, false>(b, d_work, n_tiles, st);
}

}  // namespace psim
