// 2-way Czekanowski kernels: min-plus numerators fused with the metric
// epilogue, compaction and the 128-bit checksum.
//
// Reference path replaced (one BlockTask2 of run_2way):
//   numerator  mgemm_blocked          mingemm.py:189-209 / 94-117
//   epilogue   _pair_value_matrix     metrics2.py:85-89   (2*N)/(s_i+s_j), D==0 -> +0
//   compaction _emit_pair_records     metrics2.py:92-105  diagonal keeps li<lj
//   checksum   checksum/add_term      verify.py:74-96
//
// One launch can carry up to kMaxTasks block tasks (a rank's whole circulant
// step list): a single grid, no tail between tasks. CTAs map to (task, band,
// column tile, row tile) by scanning per-launch prefix counts held in the
// kernel parameters, so no device-side scratch is needed.
#include "minplus.cuh"
#include "psim_internal.h"

namespace psim {

enum Mode2 : int {
  kCzek2 = 0,      // values + checksum (+ degenerate count)
  kRawCol = 1,     // numerators, column-major M[i + j*ldm]; diagonal mirrors to a full square
  kRawPacked = 2,  // numerators in the packed value layout (triangle or row-major rectangle)
};

constexpr int kMaxTasks = 16;

template <typename T>
struct Task2 {
  const T* W;
  int64_t ldw;
  const T* V;
  int64_t ldv;
  int64_t m, n;  // rows (W vectors) x cols (V vectors)
  int diagonal;  // W and V are the same block: only i < j is kept
  const T* s_row;
  const T* s_col;
  int64_t g_row, g_col;     // global id of local row 0 / col 0
  T* out;                   // values (kCzek2), numerators (kRaw*)
  unsigned long long* acc;  // [3]: checksum lo, hi, degenerate count (kCzek2)
  int64_t row_tile0;        // first row-tile of this launch (row band of the task)
  int64_t m_end;            // rows >= m_end are outside the band
  int64_t tiles_m, tiles_n; // tile grid of the band
  int64_t band, nbands;     // rasterisation: row-tiles per band, bands
};

template <typename T>
struct Launch2 {
  int ntasks;
  int64_t n_f, n_v, ldm;
  int64_t cta_pref[kMaxTasks + 1];  // CTAs before each task
  Task2<T> t[kMaxTasks];
};

// Position of local pair (i, j) in the packed layout shared by values and
// packed numerators: the block triangle in canonical order (diagonal task)
// or the rectangle row-major (off-diagonal task).
__device__ __forceinline__ int64_t packed_pos(int diagonal, int64_t i, int64_t j, int64_t m,
                                              int64_t n) {
  return diagonal ? (int64_t)pair_index(i, j, m) : i * n + j;
}

// CTAs of band b of a task (see band_tile: rows x columns from the band's
// first column tile; diagonal bands include their skipped corner).
__host__ __device__ __forceinline__ int64_t band_count(int64_t b, int64_t G, int64_t row_tile0,
                                                       int64_t tiles_m, int64_t tiles_n,
                                                       int64_t bm, int64_t bn, int diagonal) {
  const int64_t r0 = row_tile0 + b * G;
  const int64_t rows = min64(G, row_tile0 + tiles_m - r0);
  return rows * max64(0, tiles_n - first_col_tile(r0, bm, bn, diagonal));
}

template <class C, int MODE>
__global__ void __launch_bounds__(kNT, C::MINB) k_minplus2(const Launch2<typename C::T> L) {
  using T = typename C::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);

  // task, then band, by linear scans (a handful of tasks, <= ~150 bands)
  int64_t t = blockIdx.x;
  int ti = 0;
  while (ti + 1 < L.ntasks && L.cta_pref[ti + 1] <= t) ++ti;
  const Task2<T>& a = L.t[ti];
  t -= L.cta_pref[ti];
  int64_t b = 0, cnt;
  while ((cnt = band_count(b, a.band, a.row_tile0, a.tiles_m, a.tiles_n, C::BM, C::BN,
                           a.diagonal)) <= t) {
    t -= cnt;
    ++b;
  }
  const int64_t r0t = a.row_tile0 + b * a.band;
  const int64_t rows_b = min64(a.band, a.row_tile0 + a.tiles_m - r0t);
  const int64_t bi = r0t + t % rows_b;
  const int64_t bj = first_col_tile(r0t, C::BM, C::BN, a.diagonal) + t / rows_b;
  if (bj < first_col_tile(bi, C::BM, C::BN, a.diagonal)) return;  // corner of a diagonal band

  const int64_t row0 = bi * C::BM, col0 = bj * C::BN;
  const int rows = (int)min64(C::BM, a.m_end - row0);
  const int cols = (int)min64(C::BN, a.n - col0);

  T acc[C::TM][C::TN];
  minplus_tile<C, false>(a.W + row0 * a.ldw, a.ldw, rows, a.V + col0 * a.ldv, a.ldv, cols,
                         nullptr, L.n_f, acc, smem);

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
        const uint64_t gidx = gi < gj ? pair_index(gi, gj, L.n_v) : pair_index(gj, gi, L.n_v);
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
          a.out[i + j * L.ldm] = acc[mi][nj];
          if (a.diagonal && j != i) a.out[j + i * L.ldm] = acc[mi][nj];
        } else {
          if (a.diagonal && j <= i) continue;
          a.out[packed_pos(a.diagonal, i, j, a.m, a.n)] = acc[mi][nj];
        }
      }
    }
  }
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

// Fill the tiling fields of a task for rows [row_begin, row_end); returns its CTA count.
template <class C>
static int64_t plan_task(Task2<typename C::T>& a, int64_t row_begin, int64_t row_end) {
  if (row_end <= 0) row_end = a.m;
  if (a.m <= 0 || a.n <= 0 || row_end <= row_begin) return 0;
  a.row_tile0 = row_begin / C::BM;
  a.m_end = row_end;
  a.tiles_m = (row_end - row_begin + C::BM - 1) / C::BM;
  a.tiles_n = (a.n + C::BN - 1) / C::BN;
  a.band = band_height<C>();
  a.nbands = (a.tiles_m + a.band - 1) / a.band;
  int64_t ctas = 0;
  for (int64_t b = 0; b < a.nbands; ++b)
    ctas += band_count(b, a.band, a.row_tile0, a.tiles_m, a.tiles_n, C::BM, C::BN, a.diagonal);
  return ctas;
}

template <class C, int MODE>
static cudaError_t launch(Launch2<typename C::T>& L, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_minplus2<C, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int64_t blocks = L.cta_pref[L.ntasks];
  if (blocks <= 0) return cudaSuccess;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  k_minplus2<C, MODE><<<(unsigned)blocks, kNT, C::SMEM_BYTES, st>>>(L);
  return cudaGetLastError();
}

template <typename T>
static Task2<T> make_task(const psim_block2_t& b) {
  Task2<T> a{};
  a.W = static_cast<const T*>(b.W);
  a.ldw = b.ldw;
  a.V = static_cast<const T*>(b.V);
  a.ldv = b.ldv;
  a.m = b.m;
  a.n = b.n;
  a.diagonal = b.diagonal;
  a.s_row = static_cast<const T*>(b.s_row);
  a.s_col = static_cast<const T*>(b.s_col);
  a.g_row = b.g_row;
  a.g_col = b.g_col;
  a.out = static_cast<T*>(b.vals);
  a.acc = b.acc;
  return a;
}

template <typename T>
cudaError_t czek2_tasks_t(const Czek2Block* tasks, int ntasks, cudaStream_t st) {
  using C = typename Prod<T>::C;
  for (int base = 0; base < ntasks; base += kMaxTasks) {
    Launch2<T> L{};
    L.n_f = tasks[base].n_f;
    L.n_v = tasks[base].n_v;
    L.ntasks = ntasks - base < kMaxTasks ? ntasks - base : kMaxTasks;
    L.cta_pref[0] = 0;
    for (int k = 0; k < L.ntasks; ++k) {
      const psim_block2_t& b = tasks[base + k];
      L.t[k] = make_task<T>(b);
      L.cta_pref[k + 1] = L.cta_pref[k] + plan_task<C>(L.t[k], b.row_begin, b.row_end);
    }
    cudaError_t e = launch<C, kCzek2>(L, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
cudaError_t mgemm_t(const void* W, int64_t ldw, const void* V, int64_t ldv, int64_t n_f,
                    int64_t m, int64_t n, int symmetric, void* M, int64_t ldm, int packed,
                    cudaStream_t st) {
  using C = typename Prod<T>::C;
  Launch2<T> L{};
  L.ntasks = 1;
  L.n_f = n_f;
  L.ldm = ldm;
  Task2<T>& a = L.t[0];
  a.W = static_cast<const T*>(W);
  a.ldw = ldw;
  a.V = static_cast<const T*>(V);
  a.ldv = ldv;
  a.m = m;
  a.n = n;
  a.diagonal = symmetric;
  a.out = static_cast<T*>(M);
  L.cta_pref[0] = 0;
  L.cta_pref[1] = plan_task<C>(a, 0, 0);
  return packed ? launch<C, kRawPacked>(L, st) : launch<C, kRawCol>(L, st);
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
