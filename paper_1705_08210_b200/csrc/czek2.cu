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
// meet only in commutative atomics), so no dependent waits. Off-diagonal tasks
// over the same rows run as one column-flattened task (kCzek2Flat), and each
// task's ragged last row tile as a 32-row edge task (czek2_tasks_t).
#include <cstdlib>

#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "minplus.cuh"
#include "psim_tma.h"
#include "psim_internal.h"

namespace psim {

enum Mode2 : int {
  kCzek2 = 0,      // values + checksum (+ degenerate count)
  kRawCol = 1,     // numerators, column-major M[i + j*ldm]; diagonal mirrors to a full square
  kRawPacked = 2,  // numerators in the packed value layout (triangle or row-major rectangle)
  kCzek2Streamed = 3,  // kCzek2 while the block is still arriving: tiles bottom-up, each
                       // waits for its input chunk's ready flag; sums computed in the tile
  kCzek2Flat = 4,  // kCzek2 over several off-diagonal tasks of the same rows laid end to
                   // end along the columns (segments): one ragged column tile per group
                   // instead of one per task; a tile may straddle two segments
};

constexpr int kMaxSeg = 16;  // segments of a kCzek2Flat launch (each >= BN columns)

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
  const unsigned* ready;      // kCzek2Streamed: ready[c] != 0 once vectors of chunk c landed
  int64_t chunk;              // kCzek2Streamed: vectors per chunk
  T* sums;                    // kCzek2Streamed: column sums, published per row tile
  unsigned* sum_ready;        // kCzek2Streamed: sum_ready[r] != 0 once row tile r's are in
  // kCzek2Flat: segment s is flat columns [seg_c0[s], seg_c0[s+1]) = columns of
  // task s, read from seg_V[s] (stride ldv), sums seg_scol[s], global ids from
  // seg_gcol[s], values to seg_out[s] (row-major, seg_c0[s+1]-seg_c0[s] wide)
  int nseg;
  int64_t seg_c0[kMaxSeg + 1];
  const T* seg_V[kMaxSeg];
  const T* seg_scol[kMaxSeg];
  int64_t seg_gcol[kMaxSeg];
  T* seg_out[kMaxSeg];
  // TMA staging (minplus_tile_tma): tensor maps of W (rows) and V (columns;
  // a flattened group whose segments lie back to back is one operand)
  int tma;
  CUtensorMap tmW, tmV;
};

// Segment of flat column c (kCzek2Flat): a short uniform scan.
template <typename T>
__device__ __forceinline__ int seg_of(const Args2<T>& a, int64_t c) {
  int s = 0;
  while (s + 1 < a.nseg && a.seg_c0[s + 1] <= c) ++s;
  return s;
}

// kCzek2Streamed: the host uploads the block in chunks from the LAST vector
// down (copy engine, flag after each chunk), so a tile whose lowest vector is
// v may start once chunk(v)'s flag is set. Bounded spin: a flag that has not
// arrived after kWaitLimitNs sets g_stream_abort and the CTA gives up (its
// tile result is discarded); every other waiter sees the abort flag and
// gives up at once, and the host turns the flag into EngineError
// (psim_stream_error). No __trap(): the CUDA context, torch's and NCCL's
// state survive a stalled upload.
// Wait statistics of streamed runs (psim_stream_stats): total ns spent
// waiting for input chunks / for column sums, count of sum waits, max wait.
__device__ unsigned long long g_stream_wait[4];
__device__ unsigned g_stream_abort;
constexpr uint64_t kWaitLimitNs = 20000000000ull;  // 20 s

__device__ __forceinline__ bool wait_ready(const unsigned* flag, int kind) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint64_t t = t0;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v) {
      if (t > t0) {
        atomicAdd(&g_stream_wait[kind], (unsigned long long)(t - t0));
        if (kind == 1) atomicAdd(&g_stream_wait[2], 1ull);
        atomicMax(&g_stream_wait[3], (unsigned long long)(t - t0));
      }
      return true;
    }
    if (*(volatile unsigned*)&g_stream_abort) return false;
    __nanosleep(512);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > kWaitLimitNs) {
      atomicExch(&g_stream_abort, 1u);
      return false;
    }
  }
}

// One thread waits; the CTA learns the outcome through shared memory.
__device__ __forceinline__ bool cta_wait_ready(const unsigned* flag, int kind) {
  __shared__ int ok;
  if (threadIdx.x == 0) ok = wait_ready(flag, kind);
  __syncthreads();
  const bool r = ok;
  __syncthreads();
  return r;
}

cudaError_t stream_error(unsigned* aborted, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(aborted, g_stream_abort, sizeof(unsigned));
  if (e == cudaSuccess && reset) {
    const unsigned z = 0;
    e = cudaMemcpyToSymbol(g_stream_abort, &z, sizeof(z));
  }
  return e;
}

cudaError_t stream_stats(unsigned long long* out4, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out4, g_stream_wait, sizeof(g_stream_wait));
  if (e == cudaSuccess && reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_stream_wait, z, sizeof(z));
  }
  return e;
}

// kCzek2Streamed CTA order: bands bottom-up; each band starts with one
// column-sum CTA per row tile of the band, then the band's tiles in
// band_tile order. Band b holds launch tiles [pref[b], pref[b+1]) and row
// tiles [b*G, min((b+1)*G, tiles_m)), so with its sum CTAs it spans
// [P(b), P(b+1)) of the extended order, P(b) = pref[b] + b*G (P(nbands) =
// total + tiles_m); bottom-up it sits at [P_end - P(b+1), P_end - P(b)).
// Returns the band_tile index, or -1 - r for the sum CTA of row tile r.
template <typename T>
__device__ __forceinline__ int64_t streamed_tile(const Args2<T>& a) {
  auto P = [&](int64_t b) {
    return ld_pref(a.row_pref + b) + (b == a.nbands ? a.tiles_m : b * a.band);
  };
  const int64_t end = P(a.nbands);
  const int64_t t = blockIdx.x, x = end - 1 - t;
  int64_t lo = 0, hi = a.nbands;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (P(mid) <= x) lo = mid; else hi = mid;
  }
  const int64_t off = t - (end - P(lo + 1));
  const int64_t rows = min64(a.band, a.tiles_m - lo * a.band);
  if (off < rows) return -1 - (lo * a.band + off);
  return ld_pref(a.row_pref + lo) + (off - rows);
}

// Column sums of the 128 (BM) vectors of row tile r, each a sequential
// ascending-q fold from +0 (k_colsum's order), staged kSumQ fields at a time
// through double-buffered shared memory with coalesced loads: the loads of
// the next chunk are in flight (registers) while the current one is folded,
// one barrier per chunk. Published with sum_ready[r].
template <class C>
__device__ void streamed_row_sums(const Args2<typename C::T>& a, int64_t r,
                                  typename C::T* smem) {
  using T = typename C::T;
  constexpr int kSumQ = 64;                 // fields per chunk
  constexpr int kPitch = kSumQ + 1;         // conflict-free column reads
  constexpr int kRows = C::BM / (kNT / 32);  // rows each warp stages
  constexpr int kPer = kSumQ / 32;          // fields per lane per row
  static_assert(2 * C::BM * kPitch * (int)sizeof(T) <= C::SMEM_BYTES, "sum staging");
  const int64_t v0 = r * C::BM;
  const int nv = (int)min64(C::BM, a.n - v0);
  if (!cta_wait_ready(a.ready + v0 / a.chunk, 0)) return;  // aborted: sums never published
  T (*tile)[C::BM][kPitch] = reinterpret_cast<T (*)[C::BM][kPitch]>(smem);  // [2][BM][pitch]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T nxt[kRows][kPer];
  auto load = [&](int64_t q0) {
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
      const int lv = warp + j * (kNT / 32);
#pragma unroll
      for (int h = 0; h < kPer; ++h) {
        const int64_t q = q0 + h * 32 + lane;
        nxt[j][h] = (lv < nv && q < a.n_f) ? __ldcg(a.W + (v0 + lv) * a.ldw + q) : T(0);
      }
    }
  };
  T acc = T(0);
  load(0);
  int buf = 0;
  for (int64_t q0 = 0; q0 < a.n_f; q0 += kSumQ, buf ^= 1) {
#pragma unroll
    for (int j = 0; j < kRows; ++j)
#pragma unroll
      for (int h = 0; h < kPer; ++h) tile[buf][warp + j * (kNT / 32)][h * 32 + lane] = nxt[j][h];
    // (this chunk's buffer was last read two chunks ago, before the previous barrier)
    __syncthreads();
    if (q0 + kSumQ < a.n_f) load(q0 + kSumQ);
    if (threadIdx.x < C::BM) {
      const int cnt = (int)min64(kSumQ, a.n_f - q0);
      for (int k = 0; k < cnt; ++k) acc = Traits<T>::add(acc, tile[buf][threadIdx.x][k]);
    }
  }
  if (threadIdx.x < nv) a.sums[v0 + threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.sum_ready + r), "r"(1u)
                 : "memory");
  }
}

// Position of local pair (i, j) in the packed layout shared by values and
// packed numerators: the block triangle in canonical order (diagonal task)
// or the rectangle row-major (off-diagonal task).
__device__ __forceinline__ int64_t packed_pos(int diagonal, int64_t i, int64_t j, int64_t m,
                                              int64_t n) {
  return diagonal ? (int64_t)pair_index(i, j, m) : i * n + j;
}

template <class C, int MODE>
__global__ void __launch_bounds__(kNT, C::MINB)
    k_minplus2(const __grid_constant__ Args2<typename C::T> a) {
  using T = typename C::T;
  // let a programmatically dependent next task start filling SMs right away
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) unsigned char smem_raw[];  // TMA destinations: 128 B
  T* smem = reinterpret_cast<T*>(smem_raw);
  constexpr bool STREAMED = MODE == kCzek2Streamed;
  // streamed: bands bottom-up (their input arrives first), each led by the
  // CTAs that publish its row tiles' column sums
  int64_t tb = blockIdx.x;
  if constexpr (STREAMED) {
    tb = streamed_tile(a);
    if (tb < 0) {
      streamed_row_sums<C>(a, -1 - tb, smem);
      // keep the PDL invariant of every exit path (see the end of the kernel),
      // although a streamed launch is never programmatically dependent
      asm volatile("griddepcontrol.wait;" ::: "memory");
      return;
    }
  }
  int bi, bj;
  if (!band_tile(tb, a.row_pref, a.nbands, a.band, a.row_tile0, a.row_tile0 + a.tiles_m, C::BM,
                 C::BN, a.diagonal, bi, bj)) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;  // left of the diagonal inside a diagonal band (uniform per CTA)
  }
  T acc[C::TM][C::TN];
  {
    const int64_t row0 = (int64_t)bi * C::BM, col0 = (int64_t)bj * C::BN;
    if (STREAMED) {
      if (!cta_wait_ready(a.ready + min64(row0, col0) / a.chunk, 0)) return;
      // the chunk was written by the copy engine: order the flag's acquire
      // before the async-proxy (TMA) reads of it
      if (a.tma) asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (a.tma) {  // launch-uniform
      minplus_tile_tma<C>(&a.tmW, (int)row0, &a.tmV, (int)col0, a.n_f, acc, smem);
    } else if constexpr (MODE == kCzek2Flat) {
      // columns [col0, split) from segment s, the rest from segment s + 1
      const int s = seg_of(a, col0);
      const int cols = (int)min64(C::BN, a.n - col0);
      const int split = (int)min64(cols, a.seg_c0[s + 1] - col0);
      const T* V1 = a.seg_V[s] + (col0 - a.seg_c0[s]) * a.ldv;
      const T* V2b = split < cols ? a.seg_V[s + 1] - (int64_t)split * a.ldv : V1;
      minplus_tile<C, false, false, true>(a.W + row0 * a.ldw, a.ldw,
                                          (int)min64(C::BM, a.m_end - row0), V1, a.ldv, cols,
                                          nullptr, a.n_f, acc, smem, nullptr, V2b, split);
    } else {
      minplus_tile<C, false>(a.W + row0 * a.ldw, a.ldw, (int)min64(C::BM, a.m_end - row0),
                             a.V + col0 * a.ldv, a.ldv, (int)min64(C::BN, a.n - col0), nullptr,
                             a.n_f, acc, smem);
    }
  }
  // the tile is decoded again rather than kept live across the mainloop
  band_tile(tb, a.row_pref, a.nbands, a.band, a.row_tile0, a.row_tile0 + a.tiles_m, C::BM, C::BN,
            a.diagonal, bi, bj);
  const int64_t row0 = (int64_t)bi * C::BM, col0 = (int64_t)bj * C::BN;
  const int rows = (int)min64(C::BM, a.m_end - row0);
  const int cols = (int)min64(C::BN, a.n - col0);
  if (STREAMED) {
    // the sums of this tile's rows and columns: published by the owners of
    // row tiles bi .. (col0 + cols - 1) / BM (columns lie at or right of the rows)
    __shared__ int sums_ok;
    if (threadIdx.x == 0) {
      bool ok = wait_ready(a.sum_ready + bi, 1);
      for (int64_t r = col0 / C::BM; ok && r <= (col0 + cols - 1) / C::BM; ++r)
        if (r != bi) ok = wait_ready(a.sum_ready + r, 1);
      sums_ok = ok;
    }
    __syncthreads();
    if (!sums_ok) return;
  }
  const int ty = thread_ty<C::MAP>(), tx = thread_tx<C::MAP>();
  if constexpr (MODE == kCzek2Flat) {
    const int s1 = seg_of(a, col0);
    const int64_t cb = a.seg_c0[s1 + 1];  // first flat column of segment s1 + 1
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
        if (lj >= cols) continue;
        const int64_t jf = col0 + lj;
        const int s = jf >= cb ? s1 + 1 : s1;
        const int64_t j = jf - a.seg_c0[s];
        const T d = Traits<T>::add(si, a.seg_scol[s][j]);
        const bool zero = (d == T(0));
        const T v = zero ? T(0) : Traits<T>::div(Traits<T>::mul(T(2), acc[mi][nj]), d);
        T* out = a.seg_out[s];
        if (out) out[i * (a.seg_c0[s + 1] - a.seg_c0[s]) + j] = v;
        const uint64_t gj = (uint64_t)(a.seg_gcol[s] + j);
        const uint64_t gidx = gi < gj ? pair_index(gi, gj, a.n_v) : pair_index(gj, gi, a.n_v);
        c.term(gidx, Traits<T>::bits(v));
        c.deg += zero ? 1ull : 0ull;
      }
    }
    cks_block_flush<kNT>(a.acc, c);
  } else if (MODE == kCzek2 || STREAMED) {
    Cks c;
#pragma unroll
    for (int mi = 0; mi < C::TM; ++mi) {
      const int li = ty + 16 * mi;
      if (li >= rows) continue;
      const int64_t i = row0 + li;
      const T si = STREAMED ? __ldcg(a.sums + i) : a.s_row[i];  // (L2: written this launch)
      const uint64_t gi = (uint64_t)(a.g_row + i);
#pragma unroll
      for (int nj = 0; nj < C::TN; ++nj) {
        const int lj = tx + 16 * nj;
        const int64_t j = col0 + lj;
        if (lj >= cols || (a.diagonal && j <= i)) continue;
        const T d = Traits<T>::add(si, STREAMED ? __ldcg(a.sums + j) : a.s_col[j]);
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

// Tensor maps for TMA staging (minplus_tile_tma): psim_tma.h. A flattened
// group uses TMA only when its segments lie back to back in memory (one V
// operand); otherwise the two-pointer cp.async loader runs.
template <class C>
static void setup_tma(Args2<typename C::T>& a, int mode) {
  using T = typename C::T;
  a.tma = 0;
  if (!tma_enabled() || !(mode == kCzek2 || mode == kCzek2Flat || mode == kCzek2Streamed ||
               mode == kRawCol || mode == kRawPacked))
    return;
  const T* vbase = a.V;
  if (a.nseg > 0) {
    for (int s = 0; s + 1 < a.nseg; ++s)
      if (a.seg_V[s] + (a.seg_c0[s + 1] - a.seg_c0[s]) * a.ldv != a.seg_V[s + 1]) return;
    vbase = a.seg_V[0];
  }
  if (encode_operand<T>(&a.tmW, a.W, a.n_f, a.m, a.ldw, C::BM, C::PITCH) &&
      encode_operand<T>(&a.tmV, vbase, a.n_f, a.n, a.ldv, C::BN, C::PITCH))
    a.tma = 1;
}

// Launch a group of tasks (same mode): band prefixes first, then the grids
// back to back, each after the first as a programmatic dependent launch.
// Tasks with edge[k] run the 32-row edge configuration CE.
template <class C, int MODE, class CE = C>
static cudaError_t launch_group(Args2<typename C::T>* args, const int64_t* row_begin,
                                const int64_t* row_end, int count, cudaStream_t st,
                                const bool* edge = nullptr) {
  // a kCzek2 group may hold flattened tasks (nseg > 0): those run k_minplus2<C, kCzek2Flat>
  constexpr int FLAT_MODE = MODE == kCzek2 ? kCzek2Flat : MODE;
  cudaError_t e = cudaSuccess;
  {
    static_assert(std::is_same<typename C::T, typename CE::T>::value, "one element type");
    void* const kerns[4] = {(void*)k_minplus2<C, MODE>, (void*)k_minplus2<C, FLAT_MODE>,
                            (void*)k_minplus2<CE, MODE>, (void*)k_minplus2<CE, FLAT_MODE>};
    const int smem[4] = {C::SMEM_BYTES, C::SMEM_BYTES, CE::SMEM_BYTES, CE::SMEM_BYTES};
    for (int q = 0; q < 4 && e == cudaSuccess; ++q)
      e = cudaFuncSetAttribute(kerns[q], cudaFuncAttributeMaxDynamicSharedMemorySize, smem[q]);
  }
  if (e != cudaSuccess) return e;
  auto is_edge = [&](int k) { return edge != nullptr && edge[k]; };
  int64_t total_bands = 0;
  int64_t* blocks = new int64_t[count];
  for (int k = 0; k < count; ++k) {
    const int64_t rb = row_begin ? row_begin[k] : 0, re = row_end ? row_end[k] : 0;
    blocks[k] = is_edge(k) ? plan2<CE>(args[k], rb, re) : plan2<C>(args[k], rb, re);
    if (MODE == kCzek2Streamed && blocks[k] > 0) blocks[k] += args[k].tiles_m;  // sum CTAs
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
    const int64_t bm = is_edge(k) ? CE::BM : C::BM, bn = is_edge(k) ? CE::BN : C::BN;
    note_launch();
    k_band_prefix<<<1, 1024, 0, st>>>(a.nbands, a.band, a.row_tile0, a.tiles_m, a.tiles_n, bm,
                                      bn, a.diagonal, pref + (a.row_pref - pref));
    e = cudaGetLastError();
  }
  bool first = true;
  for (int k = 0; k < count && e == cudaSuccess; ++k) {
    if (blocks[k] <= 0) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks[k]);
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = is_edge(k) ? CE::SMEM_BYTES : C::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = first ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool flat = args[k].nseg > 0;
    if (is_edge(k))
      setup_tma<CE>(args[k], flat ? FLAT_MODE : MODE);
    else
      setup_tma<C>(args[k], flat ? FLAT_MODE : MODE);
    note_launch();
    if (is_edge(k))
      e = flat ? cudaLaunchKernelEx(&cfg, k_minplus2<CE, FLAT_MODE>, args[k])
               : cudaLaunchKernelEx(&cfg, k_minplus2<CE, MODE>, args[k]);
    else
      e = flat ? cudaLaunchKernelEx(&cfg, k_minplus2<C, FLAT_MODE>, args[k])
               : cudaLaunchKernelEx(&cfg, k_minplus2<C, MODE>, args[k]);
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

// Off-diagonal tasks over the same rows (same W, sums, global row ids, whole
// row range) and field layout are merged, in order, into one kCzek2Flat task
// whose columns are theirs laid end to end: the group has one ragged column
// tile instead of one per task (a task of 5000 vectors fills 39 of its 40
// column tiles with 8/128 of the last). Each segment must be >= BN wide, so a
// tile touches at most two. Values, record layout and checksum terms are those
// of the separate tasks. PSIM_NO_FLAT=1 disables it (A/B).
template <class C>
static int flatten_tasks(Args2<typename C::T>* args, int64_t* rb, int64_t* re, int ntasks) {
  static const bool off = [] {
    const char* v = getenv("PSIM_NO_FLAT");
    return v && v[0] == '1';
  }();
  if (off) return ntasks;
  auto eligible = [&](int k) {
    const auto& a = args[k];
    return !a.diagonal && rb[k] == 0 && re[k] == 0 && a.n >= C::BN && a.m > 0;
  };
  const bool tma = tma_enabled();
  auto same_rows = [&](int k, int l) {
    const auto& a = args[k];
    const auto& b = args[l];
    // with TMA staging a group is one V operand: its columns must lie back to
    // back in memory (the runtime receives blocks into one contiguous ring)
    const bool adjacent = !tma || args[l - 1].V + args[l - 1].n * args[l - 1].ldv == b.V;
    return a.W == b.W && a.ldw == b.ldw && a.m == b.m && a.n_f == b.n_f && a.ldv == b.ldv &&
           a.s_row == b.s_row && a.g_row == b.g_row && a.n_v == b.n_v && a.acc == b.acc &&
           adjacent;
  };
  int out = 0;
  for (int k = 0; k < ntasks;) {
    int l = k + 1;
    if (eligible(k))
      while (l < ntasks && l - k < kMaxSeg && eligible(l) && same_rows(k, l)) ++l;
    Args2<typename C::T> a = args[k];
    if (l - k > 1) {
      a.nseg = l - k;
      int64_t c = 0;
      for (int s = 0; s < a.nseg; ++s) {
        const auto& t = args[k + s];
        a.seg_c0[s] = c;
        a.seg_V[s] = t.V;
        a.seg_scol[s] = t.s_col;
        a.seg_gcol[s] = t.g_col;
        a.seg_out[s] = t.out;
        c += t.n;
      }
      a.seg_c0[a.nseg] = c;
      a.n = c;
    }
    rb[out] = rb[k];
    re[out] = re[k];
    args[out++] = a;
    k = l;
  }
  return out;
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
  using C = typename Prod<T>::C;
  using CE = typename Edge<T>::C;
  const int count = flatten_tasks<C>(args, rb, re, ntasks);
  // The ragged last row tile of each task (rows past the last multiple of BM)
  // runs as an edge task with 32-row tiles at the end of the chain, where its
  // small CTAs also fill the tail -- when it has at most 3 * 32 rows: a 32-row
  // tile issues at ~85% of the full tile's rate, so 4 of them cost more than
  // one 128-row tile. PSIM_NO_EDGE=1 disables it (A/B).
  static const bool no_edge = [] {
    const char* v = getenv("PSIM_NO_EDGE");
    return v && v[0] == '1';
  }();
  Args2<T>* all = new Args2<T>[2 * count];
  int64_t* arb = new int64_t[2 * count];
  int64_t* are = new int64_t[2 * count];
  bool* edge = new bool[2 * count];
  int n_all = 0;
  for (int k = 0; k < count; ++k) {
    const int64_t m_end = re[k] > 0 ? re[k] : args[k].m;
    const int64_t full = rb[k] + (m_end - rb[k]) / C::BM * C::BM;
    const bool split = !no_edge && full < m_end && m_end - full <= 3 * CE::BM;
    if (!split || full > rb[k]) {
      all[n_all] = args[k];
      arb[n_all] = rb[k];
      are[n_all] = split ? full : re[k];
      edge[n_all++] = false;
    }
  }
  for (int k = 0; k < count; ++k) {
    const int64_t m_end = re[k] > 0 ? re[k] : args[k].m;
    const int64_t full = rb[k] + (m_end - rb[k]) / C::BM * C::BM;
    if (no_edge || full >= m_end || m_end - full > 3 * CE::BM) continue;
    all[n_all] = args[k];
    arb[n_all] = full;
    are[n_all] = m_end;
    edge[n_all++] = true;
  }
  cudaError_t e = launch_group<C, kCzek2, CE>(all, arb, are, n_all, st, edge);
  delete[] all;
  delete[] arb;
  delete[] are;
  delete[] edge;
  delete[] args;
  delete[] rb;
  delete[] re;
  return e;
}

// Single diagonal task over a block that is still on the host: the block is
// uploaded by the copy engine in chunks from the last vector down (2-D copies
// into the padded layout, each followed by its ready flag), while the kernel
// (tiles bottom-up) starts on the first chunk. See kCzek2Streamed.
constexpr int64_t kMaxChunks = kStreamMaxFlags;

static cudaError_t flag_sources(const unsigned** zeros, const unsigned** one) {
  static unsigned* buf = nullptr;  // pinned [0] * kMaxChunks + [1]; never freed
  static cudaError_t st = [] {
    cudaError_t e = cudaHostAlloc(&buf, (kMaxChunks + 1) * sizeof(unsigned), cudaHostAllocDefault);
    if (e == cudaSuccess) {
      for (int64_t c = 0; c < kMaxChunks; ++c) buf[c] = 0;
      buf[kMaxChunks] = 1;
    }
    return e;
  }();
  *zeros = buf;
  *one = buf ? buf + kMaxChunks : nullptr;
  return st;
}

// Pageable host input of a streamed run: each chunk (last first) is copied
// by host threads into a slot of a pinned ring, then uploaded from there by
// the copy engine (one cudaMemcpyAsync per chunk) and flagged; a slot is
// reused once its upload has completed. The host thread returns when the last
// chunk is enqueued -- the kernel, launched before, computes meanwhile.
namespace {
constexpr int kRing = 4;
struct PinnedRing {
  std::mutex mu;
  char* buf[kRing] = {};
  cudaEvent_t done[kRing] = {};
  size_t cap = 0;
};
PinnedRing& ring() {
  static PinnedRing r;  // grown on demand, kept for the process (pinning is slow)
  return r;
}

cudaError_t spin_event(cudaEvent_t ev) {  // (blocking waits wake late on these boxes)
  for (;;) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e != cudaErrorNotReady) return e;
  }
}

void copy_rows(char* dst, int64_t dst_ld, const char* src, int64_t src_ld, int64_t row_bytes,
               int64_t rows) {
  const int64_t total = rows * row_bytes;
  const int nt = total > (16 << 20) ? 4 : 1;
  auto part = [&](int k) {
    for (int64_t r = rows * k / nt; r < rows * (k + 1) / nt; ++r)
      std::memcpy(dst + r * dst_ld, src + r * src_ld, row_bytes);
  };
  std::vector<std::thread> th;
  for (int k = 1; k < nt; ++k) th.emplace_back(part, k);
  part(0);
  for (auto& x : th) x.join();
}
}  // namespace

// Grow the ring to `need` bytes per slot. Called BEFORE the streamed kernel
// is launched: cudaFreeHost / cudaHostAlloc synchronize with the device, and a
// launched kernel waiting for chunks would deadlock against them.
static cudaError_t prepare_ring(size_t need) {
  PinnedRing& R = ring();
  std::lock_guard<std::mutex> lock(R.mu);
  cudaError_t e = cudaSuccess;
  if (R.cap < need) {
    for (int k = 0; k < kRing; ++k) {
      if (R.buf[k]) cudaFreeHost(R.buf[k]);
      R.buf[k] = nullptr;
    }
    R.cap = 0;
    for (int k = 0; k < kRing && e == cudaSuccess; ++k) {
      e = cudaHostAlloc(&R.buf[k], need, cudaHostAllocDefault);
      if (e == cudaSuccess && !R.done[k])
        e = cudaEventCreateWithFlags(&R.done[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) R.cap = need;
  }
  return e;
}

static cudaError_t stage_pageable(void* dst_, int64_t ldw, const void* src_, int64_t host_ld,
                                  int64_t n_f, int64_t n, int64_t chunk, size_t sz,
                                  unsigned* ready, const unsigned* one, int64_t nflags,
                                  cudaStream_t copy) {
  PinnedRing& R = ring();
  std::lock_guard<std::mutex> lock(R.mu);
  cudaError_t e = R.cap >= (size_t)chunk * ldw * sz ? cudaSuccess : cudaErrorInvalidValue;
  char* dst = static_cast<char*>(dst_);
  const char* src = static_cast<const char*>(src_);
  const int64_t nchunks = (n + chunk - 1) / chunk;
  int64_t i = 0;
  for (int64_t c = nchunks - 1; c >= 0 && e == cudaSuccess; --c, ++i) {
    const int slot = (int)(i % kRing);
    if (i >= kRing) e = spin_event(R.done[slot]);  // its previous upload is done
    if (e != cudaSuccess) break;
    const int64_t lo = c * chunk, rows = min64(n, lo + chunk) - lo;
    copy_rows(R.buf[slot], ldw * sz, src + lo * host_ld * sz, host_ld * sz, n_f * sz, rows);
    e = cudaMemcpyAsync(dst + lo * ldw * sz, R.buf[slot], rows * ldw * sz,
                        cudaMemcpyHostToDevice, copy);
    if (e == cudaSuccess) e = cudaEventRecord(R.done[slot], copy);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ready + c, one, sizeof(unsigned), cudaMemcpyHostToDevice, copy);
  }
  if (e != cudaSuccess)  // release every flag: the kernel finishes, the error discards it
    for (int64_t k = 0; k < nflags; ++k)
      cudaMemcpyAsync(ready + k, one, sizeof(unsigned), cudaMemcpyHostToDevice, copy);
  // the ring must not be refilled before this run's last uploads are done
  for (int k = 0; k < kRing && e == cudaSuccess; ++k)
    if (R.done[k]) e = spin_event(R.done[k]);
  return e;
}

template <typename T>
cudaError_t czek2_streamed_t(const Czek2Block& t, const void* host, int64_t host_ld,
                             int64_t chunk, unsigned* ready, cudaStream_t compute,
                             cudaStream_t copy) {
  using C = typename Prod<T>::C;
  const int64_t n = t.n, nchunks = (n + chunk - 1) / chunk;
  const int64_t nflags = nchunks + (n + C::BM - 1) / C::BM;  // data flags, then sum flags
  const unsigned *zeros = nullptr, *one = nullptr;
  cudaError_t e = flag_sources(&zeros, &one);
  if (e != cudaSuccess) return e;
  cudaEvent_t cleared;
  if ((e = cudaEventCreateWithFlags(&cleared, cudaEventDisableTiming)) != cudaSuccess) return e;
  const size_t sz = sizeof(T);
  // flags cleared by the copy engine first; the kernel may only start polling
  // after that. The kernel is launched BEFORE the chunk copies are enqueued
  // (enqueueing ~100 copies takes host time that must not delay the compute).
  e = cudaMemcpyAsync(ready, zeros, nflags * sizeof(unsigned), cudaMemcpyHostToDevice, copy);
  if (e == cudaSuccess) e = cudaEventRecord(cleared, copy);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(compute, cleared, 0);
  cudaEventDestroy(cleared);
  if (e != cudaSuccess) return e;
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, host) == cudaSuccess &&
                      pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (!pinned && (e = prepare_ring((size_t)chunk * t.ldw * sizeof(T))) != cudaSuccess) return e;
  void* abort_flag = nullptr;  // cleared before every streamed launch
  if ((e = cudaGetSymbolAddress(&abort_flag, g_stream_abort)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(abort_flag, 0, sizeof(unsigned), compute)) != cudaSuccess) return e;
  Args2<T> a = make_args<T>(t.W, t.ldw, t.V, t.ldv, t.n_f, t.m, t.n, 1);
  a.g_row = t.g_row;
  a.g_col = t.g_col;
  a.n_v = t.n_v;
  a.out = static_cast<T*>(t.vals);
  a.acc = t.acc;
  a.ready = ready;
  a.chunk = chunk;
  a.sums = static_cast<T*>(const_cast<void*>(t.s_row));
  a.sum_ready = ready + nchunks;
  if ((e = launch_group<C, kCzek2Streamed>(&a, nullptr, nullptr, 1, compute)) != cudaSuccess)
    return e;
  T* dst = static_cast<T*>(const_cast<void*>(t.W));
  const T* src = static_cast<const T*>(host);
  if (!pinned)  // pageable: staged through a pinned ring, chunk by chunk
    return stage_pageable(dst, t.ldw, src, host_ld, t.n_f, n, chunk, sz, ready, one, nflags, copy);
  for (int64_t c = nchunks - 1; c >= 0; --c) {
    const int64_t lo = c * chunk, hi = min64(n, lo + chunk);
    e = host_ld == t.ldw  // same pitch: the chunk is one contiguous span
            ? cudaMemcpyAsync(dst + lo * t.ldw, src + lo * host_ld, (hi - lo) * t.ldw * sz,
                              cudaMemcpyHostToDevice, copy)
            : cudaMemcpy2DAsync(dst + lo * t.ldw, t.ldw * sz, src + lo * host_ld, host_ld * sz,
                                t.n_f * sz, hi - lo, cudaMemcpyHostToDevice, copy);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ready + c, one, sizeof(unsigned), cudaMemcpyHostToDevice, copy);
    if (e != cudaSuccess) {
      // the launched kernel would wait for chunks that never come: release all
      // flags so it finishes (its results are discarded by the error)
      for (int64_t k = 0; k < nflags; ++k)
        cudaMemcpyAsync(ready + k, one, sizeof(unsigned), cudaMemcpyHostToDevice, copy);
      return e;
    }
  }
  return cudaSuccess;
}

cudaError_t czek2_streamed(int dtype, const Czek2Block& t, const void* host, int64_t host_ld,
                           int64_t chunk, unsigned* ready, cudaStream_t compute,
                           cudaStream_t copy) {
  return dtype == kF64
             ? czek2_streamed_t<double>(t, host, host_ld, chunk, ready, compute, copy)
             : czek2_streamed_t<float>(t, host, host_ld, chunk, ready, compute, copy);
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
  note_launch();
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
