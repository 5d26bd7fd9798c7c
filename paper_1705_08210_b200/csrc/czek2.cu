// 2-way Czekanowski kernels: min-plus numerators fused with the metric
// epilogue, compaction and the 128-bit checksum.
//
// Reference path replaced (one BlockTask2 of run_2way):
//   numerator  mgemm_blocked          mingemm.py:189-209 / 94-117
//   epilogue   _pair_value_matrix     metrics2.py:85-89   (2*N)/(s_i+s_j), D==0 -> +0
//   compaction _emit_pair_records     metrics2.py:92-105  diagonal keeps li<lj
//   checksum   checksum/add_term      verify.py:74-96
//
// A rank's several tasks (its circulant steps) are launched back to back with
// programmatic dependent launch: every CTA signals launch_dependents on entry,
// so the next task's CTAs fill SMs as the previous grid drains and the tasks
// share one tail. Tasks never read each other's outputs (their checksum terms
// meet only in commutative atomics), so no dependent waits.
#include "minplus.cuh"
#include "psim_internal.h"

namespace psim {

enum Mode2 : int {
  kCzek2 = 0,      // values + checksum (+ degenerate count)
  kRawCol = 1,     // numerators, column-major M[i + j*ldm]; diagonal mirrors to a full square
  kRawPacked = 2,  // numerators in the packed value layout (triangle or row-major rectangle)
};

template <typename T>
struct Args2 {
  const T* W;
  int64_t ldw;
  const T* V;
  int64_t ldv;
  int64_t n_f;
  int64_t m, n;  // rows (W vectors) x cols (V vectors)
  int diagonal;  // W and V are the same block: only i < j is kept
  const T* s_row;
  const T* s_col;
  int64_t g_row, g_col, n_v;  // global id of local row 0 / col 0; global vector count
  T* out;                     // values (kCzek2), numerators (kRaw*)
  int64_t ldm;                // kRawCol leading dimension
  unsigned long long* acc;    // [3]: checksum lo, hi, degenerate count (kCzek2)
  int64_t tiles_m, tiles_n;   // tile grid of this launch
  int64_t row_tile0;          // first row-tile of the launch (row band)
  int64_t m_end;              // rows >= m_end are outside the band
  int64_t band, nbands;       // rasterisation: row-tiles per band, bands in the launch
  const int64_t* row_pref;    // tiles before each band (device), see band_tile
};

// Position of local pair (i, j) in the packed layout shared by values and
// packed numerators: the block triangle in canonical order (diagonal task)
// or the rectangle row-major (off-diagonal task).
__device__ __forceinline__ int64_t packed_pos(int diagonal, int64_t i, int64_t j, int64_t m,
                                              int64_t n) {
  return diagonal ? (int64_t)pair_index(i, j, m) : i * n + j;
}

template <class C, int MODE>
__global__ void __launch_bounds__(kNT, C::MINB) k_minplus2(const Args2<typename C::T> a) {
  using T = typename C::T;
  // let a programmatically dependent next task start filling SMs right away
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  int bi, bj;
  if (!band_tile((int64_t)blockIdx.x, a.row_pref, a.nbands, a.band, a.row_tile0,
                 a.row_tile0 + a.tiles_m, C::BM, C::BN, a.diagonal, bi, bj)) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;  // left of the diagonal inside a diagonal band (uniform per CTA)
  }
  T acc[C::TM][C::TN];
  {
    const int64_t row0 = (int64_t)bi * C::BM, col0 = (int64_t)bj * C::BN;
    minplus_tile<C, false>(a.W + row0 * a.ldw, a.ldw, (int)min64(C::BM, a.m_end - row0),
                           a.V + col0 * a.ldv, a.ldv, (int)min64(C::BN, a.n - col0), nullptr,
                           a.n_f, acc, smem);
  }
  // the tile is decoded again rather than kept live across the mainloop
  band_tile((int64_t)blockIdx.x, a.row_pref, a.nbands, a.band, a.row_tile0,
            a.row_tile0 + a.tiles_m, C::BM, C::BN, a.diagonal, bi, bj);
  const int64_t row0 = (int64_t)bi * C::BM, col0 = (int64_t)bj * C::BN;
  const int rows = (int)min64(C::BM, a.m_end - row0);
  const int cols = (int)min64(C::BN, a.n - col0);

  const int ty = thread_ty(), tx = thread_tx();
  if (MODE == kCzek2) {
    Cks c;
#pragma unroll
    for (int mi = 0; mi < C::TM; ++mi) {
      const int li = ty + 16 * mi;
      if (li >= rows) continue;
      const int64_t i = row0 + li;
      const T si = a.s_row[i];
      const uint64_t gi = (uint64_t)(a.g_row + i);
#pragma unroll
      for (int nj = 0; nj < C::TN; ++nj) {
        const int lj = tx + 16 * nj;
        const int64_t j = col0 + lj;
        if (lj >= cols || (a.diagonal && j <= i)) continue;
        const T d = Traits<T>::add(si, a.s_col[j]);
        const bool zero = (d == T(0));
        const T v = zero ? T(0) : Traits<T>::div(Traits<T>::mul(T(2), acc[mi][nj]), d);
        if (a.out) a.out[packed_pos(a.diagonal, i, j, a.m, a.n)] = v;
        const uint64_t gj = (uint64_t)(a.g_col + j);
        const uint64_t gidx = gi < gj ? pair_index(gi, gj, a.n_v) : pair_index(gj, gi, a.n_v);
        c.term(gidx, Traits<T>::bits(v));
        c.deg += zero ? 1ull : 0ull;
      }
    }
    cks_block_flush<kNT>(a.acc, c);
  } else {
#pragma unroll
    for (int mi = 0; mi < C::TM; ++mi) {
      const int li = ty + 16 * mi;
      if (li >= rows) continue;
      const int64_t i = row0 + li;
#pragma unroll
      for (int nj = 0; nj < C::TN; ++nj) {
        const int lj = tx + 16 * nj;
        const int64_t j = col0 + lj;
        if (lj >= cols) continue;
        if (MODE == kRawCol) {
          if (a.diagonal && j < i) continue;
          a.out[i + j * a.ldm] = acc[mi][nj];
          if (a.diagonal && j != i) a.out[j + i * a.ldm] = acc[mi][nj];
        } else {
          if (a.diagonal && j <= i) continue;
          a.out[packed_pos(a.diagonal, i, j, a.m, a.n)] = acc[mi][nj];
        }
      }
    }
  }
  // A programmatically dependent grid completes only after its predecessor
  // (no-op for a normal launch), so stream order after a task group holds.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Tiles (CTAs) of band b of a launch (see band_tile).
__host__ __device__ __forceinline__ int64_t band_count(int64_t b, int64_t G, int64_t row_tile0,
                                                       int64_t tiles_m, int64_t tiles_n,
                                                       int64_t bm, int64_t bn, int diagonal) {
  const int64_t r0 = row_tile0 + b * G;
  const int64_t rows = min64(G, row_tile0 + tiles_m - r0);
  return rows * max64(0, tiles_n - first_col_tile(r0, bm, bn, diagonal));
}

// Band prefix of a launch's tile grid: one CTA, each thread folds a
// contiguous range of bands, then a block scan.
__global__ void __launch_bounds__(1024) k_band_prefix(int64_t nbands, int64_t G,
                                                      int64_t row_tile0, int64_t tiles_m,
                                                      int64_t tiles_n, int64_t bm, int64_t bn,
                                                      int diagonal, int64_t* __restrict__ pref) {
  __shared__ int64_t s[1024];
  const int64_t per = (nbands + blockDim.x - 1) / blockDim.x;
  const int64_t a = min64(nbands, threadIdx.x * per), e = min64(nbands, a + per);
  int64_t sum = 0;
  for (int64_t b = a; b < e; ++b)
    sum += band_count(b, G, row_tile0, tiles_m, tiles_n, bm, bn, diagonal);
  s[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const int64_t v = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
    __syncthreads();
    s[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? s[threadIdx.x - 1] : 0;
  for (int64_t b = a; b < e; ++b) {
    pref[b] = run;
    run += band_count(b, G, row_tile0, tiles_m, tiles_n, bm, bn, diagonal);
  }
  if (threadIdx.x == blockDim.x - 1) pref[nbands] = s[threadIdx.x];
}

// Band height: about sqrt(resident CTAs) row-tiles, so the resident window
// is roughly square in tiles (fewest distinct panels in flight).
template <class C>
static int64_t band_height() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double resident = (double)sms * C::MINB;
  int64_t g = (int64_t)(sqrt(resident * C::BN / (double)C::BM) + 0.5);
  return g < 1 ? 1 : g;
}

// Tiling of rows [row_begin, row_end) of a task (row_begin % BM == 0);
// returns the CTA count and leaves the band prefix to be built in `pref`.
template <class C>
static int64_t plan2(Args2<typename C::T>& a, int64_t row_begin, int64_t row_end) {
  if (row_end <= 0) row_end = a.m;
  if (a.m <= 0 || a.n <= 0 || row_end <= row_begin) return 0;
  a.row_tile0 = row_begin / C::BM;
  a.m_end = row_end;
  a.tiles_m = (row_end - row_begin + C::BM - 1) / C::BM;
  a.tiles_n = (a.n + C::BN - 1) / C::BN;
  a.band = band_height<C>();
  a.nbands = (a.tiles_m + a.band - 1) / a.band;
  int64_t blocks = 0;
  for (int64_t b = 0; b < a.nbands; ++b)
    blocks += band_count(b, a.band, a.row_tile0, a.tiles_m, a.tiles_n, C::BM, C::BN, a.diagonal);
  return blocks;
}

// Launch a group of tasks (same mode): band prefixes first, then the grids
// back to back, each after the first as a programmatic dependent launch.
template <class C, int MODE>
static cudaError_t launch_group(Args2<typename C::T>* args, const int64_t* row_begin,
                                const int64_t* row_end, int count, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_minplus2<C, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int64_t total_bands = 0;
  int64_t* blocks = new int64_t[count];
  for (int k = 0; k < count; ++k) {
    blocks[k] = plan2<C>(args[k], row_begin ? row_begin[k] : 0, row_end ? row_end[k] : 0);
    if (blocks[k] > 0x7fffffffLL) e = cudaErrorInvalidConfiguration;
    if (blocks[k] > 0) total_bands += args[k].nbands + 1;
  }
  int64_t* pref = nullptr;
  if (e == cudaSuccess && total_bands > 0) e = cudaMallocAsync(&pref, total_bands * 8, st);
  int64_t off = 0;
  for (int k = 0; k < count && e == cudaSuccess; ++k) {
    if (blocks[k] <= 0) continue;
    Args2<typename C::T>& a = args[k];
    a.row_pref = pref + off;
    off += a.nbands + 1;
    k_band_prefix<<<1, 1024, 0, st>>>(a.nbands, a.band, a.row_tile0, a.tiles_m, a.tiles_n,
                                      C::BM, C::BN, a.diagonal, pref + (a.row_pref - pref));
    e = cudaGetLastError();
  }
  bool first = true;
  for (int k = 0; k < count && e == cudaSuccess; ++k) {
    if (blocks[k] <= 0) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks[k]);
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = first ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_minplus2<C, MODE>, args[k]);
    first = false;
  }
  delete[] blocks;
  if (pref) {
    cudaError_t e2 = cudaFreeAsync(pref, st);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}

template <typename T>
static Args2<T> make_args(const void* W, int64_t ldw, const void* V, int64_t ldv, int64_t n_f,
                          int64_t m, int64_t n, int diagonal) {
  Args2<T> a{};
  a.W = static_cast<const T*>(W);
  a.ldw = ldw;
  a.V = static_cast<const T*>(V);
  a.ldv = ldv;
  a.n_f = n_f;
  a.m = m;
  a.n = n;
  a.diagonal = diagonal;
  return a;
}

template <typename T>
cudaError_t czek2_tasks_t(const Czek2Block* tasks, int ntasks, cudaStream_t st) {
  Args2<T>* args = new Args2<T>[ntasks];
  int64_t* rb = new int64_t[ntasks];
  int64_t* re = new int64_t[ntasks];
  for (int k = 0; k < ntasks; ++k) {
    const Czek2Block& t = tasks[k];
    args[k] = make_args<T>(t.W, t.ldw, t.V, t.ldv, t.n_f, t.m, t.n, t.diagonal);
    args[k].s_row = static_cast<const T*>(t.s_row);
    args[k].s_col = static_cast<const T*>(t.s_col);
    args[k].g_row = t.g_row;
    args[k].g_col = t.g_col;
    args[k].n_v = t.n_v;
    args[k].out = static_cast<T*>(t.vals);
    args[k].acc = t.acc;
    rb[k] = t.row_begin;
    re[k] = t.row_end;
  }
  cudaError_t e = launch_group<typename Prod<T>::C, kCzek2>(args, rb, re, ntasks, st);
  delete[] args;
  delete[] rb;
  delete[] re;
  return e;
}

template <typename T>
cudaError_t mgemm_t(const void* W, int64_t ldw, const void* V, int64_t ldv, int64_t n_f,
                    int64_t m, int64_t n, int symmetric, void* M, int64_t ldm, int packed,
                    cudaStream_t st) {
  Args2<T> a = make_args<T>(W, ldw, V, ldv, n_f, m, n, symmetric);
  a.out = static_cast<T*>(M);
  a.ldm = ldm;
  using C = typename Prod<T>::C;
  return packed ? launch_group<C, kRawPacked>(&a, nullptr, nullptr, 1, st)
                : launch_group<C, kRawCol>(&a, nullptr, nullptr, 1, st);
}

// Values + checksum from already-reduced packed numerators (the field-axis
// path: partial N -> ordered fold over p_f -> this epilogue; metrics2.py:156-158).
// One CTA per packed row li in [r0, r1); N and out point at row r0's first entry.
template <typename T>
__global__ void __launch_bounds__(256) k_czek2_from_num(const T* __restrict__ N, int64_t r0,
                                                        int64_t m, int64_t n, int diagonal,
                                                        const T* __restrict__ s_row,
                                                        const T* __restrict__ s_col,
                                                        int64_t g_row, int64_t g_col, int64_t n_v,
                                                        T* __restrict__ out,
                                                        unsigned long long* acc) {
  const int64_t i = r0 + blockIdx.x;
  const int64_t base = packed_pos(diagonal, r0, diagonal ? r0 + 1 : 0, m, n);
  const int64_t jlo = diagonal ? i + 1 : 0;
  const int64_t row_start = (diagonal ? (int64_t)pair_index(i, i + 1, m) : i * n) - base;
  const T si = s_row[i];
  const uint64_t gi = (uint64_t)(g_row + i);
  Cks c;
  for (int64_t j = jlo + threadIdx.x; j < n; j += blockDim.x) {
    const int64_t p = row_start + (j - jlo);
    const T d = Traits<T>::add(si, s_col[j]);
    const bool zero = (d == T(0));
    const T v = zero ? T(0) : Traits<T>::div(Traits<T>::mul(T(2), N[p]), d);
    if (out) out[p] = v;
    const uint64_t gj = (uint64_t)(g_col + j);
    const uint64_t gidx = gi < gj ? pair_index(gi, gj, n_v) : pair_index(gj, gi, n_v);
    c.term(gidx, Traits<T>::bits(v));
    c.deg += zero ? 1ull : 0ull;
  }
  cks_block_flush<256>(acc, c);
}

template <typename T>
cudaError_t czek2_from_num_t(const void* N, int64_t r0, int64_t r1, int64_t m, int64_t n,
                             int diagonal, const void* s_row, const void* s_col, int64_t g_row,
                             int64_t g_col, int64_t n_v, void* vals,
                             unsigned long long* acc, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  if (r1 - r0 > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  k_czek2_from_num<T><<<(unsigned)(r1 - r0), 256, 0, st>>>(
      static_cast<const T*>(N), r0, m, n, diagonal, static_cast<const T*>(s_row),
      static_cast<const T*>(s_col), g_row, g_col, n_v, static_cast<T*>(vals), acc);
  return cudaGetLastError();
}

cudaError_t czek2_block(int dtype, const Czek2Block& t, cudaStream_t st) {
  return czek2_tasks(dtype, &t, 1, st);
}

cudaError_t czek2_tasks(int dtype, const Czek2Block* tasks, int ntasks, cudaStream_t st) {
  if (ntasks <= 0) return cudaSuccess;
  return dtype == kF64 ? czek2_tasks_t<double>(tasks, ntasks, st)
                       : czek2_tasks_t<float>(tasks, ntasks, st);
}

cudaError_t mgemm(int dtype, const void* W, int64_t ldw, const void* V, int64_t ldv, int64_t n_f,
                  int64_t m, int64_t n, int symmetric, void* M, int64_t ldm, int packed,
                  cudaStream_t st) {
  return dtype == kF64 ? mgemm_t<double>(W, ldw, V, ldv, n_f, m, n, symmetric, M, ldm, packed, st)
                       : mgemm_t<float>(W, ldw, V, ldv, n_f, m, n, symmetric, M, ldm, packed, st);
}

cudaError_t czek2_from_num(int dtype, const void* N, int64_t r0, int64_t r1, int64_t m,
                           int64_t n, int diagonal, const void* s_row, const void* s_col,
                           int64_t g_row, int64_t g_col, int64_t n_v, void* vals,
                           unsigned long long* acc, cudaStream_t st) {
  return dtype == kF64 ? czek2_from_num_t<double>(N, r0, r1, m, n, diagonal, s_row, s_col, g_row,
                                                  g_col, n_v, vals, acc, st)
                       : czek2_from_num_t<float>(N, r0, r1, m, n, diagonal, s_row, s_col, g_row,
                                                 g_col, n_v, vals, acc, st);
}

}  // namespace psim
