/*
 * psim_oracle.c -- C restatement of the reference's CPU hot path.
 * TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py): used by the
 * tests as a checker and by bench.py as the CPU baseline ("port"); never by
 * the product package.
 *
 * Restates (paths relative to /root/reference/pkg/src/propsim):
 *   oracle_mgemm_*   _blocked_kernel      mingemm.py:94-117  (tile over outputs only,
 *                    q ascending per element from +0, `w if w < v else v`)
 *   oracle_colsum_*  _colsum_kernel       mingemm.py:120-127
 *   oracle_czek2_*   one full single-rank run_2way: numerators, sums,
 *                    (2*N)/(s_i+s_j) with D==0 -> 0 (metrics2.py:77-89),
 *                    canonical compaction (metrics2.py:92-105) and the 128-bit
 *                    checksum (verify.py:36-96).
 * Threads split output tiles (the reference's thread transport runs its
 * numba kernels concurrently with nogil=True, mingemm.py:94).
 * Compile WITHOUT -ffast-math (IEEE adds / division, no contraction).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE_I 64  /* DEFAULT_TILE, mingemm.py:18 */
#define TILE_J 128

static uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

/* ---- blocked min-plus kernel, templated by macro over the element type ---- */
#define DEFINE_MGEMM(T, SUFFIX)                                                          \
  typedef struct {                                                                       \
    const T* W; int64_t ldw; const T* V; int64_t ldv; int64_t n_f, m, n;                 \
    T* M; int64_t ldm; int64_t next_tile; int64_t n_tiles; pthread_mutex_t* lock;         \
  } mg_job_##SUFFIX;                                                                     \
  static void* mg_worker_##SUFFIX(void* arg) {                                           \
    mg_job_##SUFFIX* jb = (mg_job_##SUFFIX*)arg;                                         \
    T* Vp = (T*)malloc(sizeof(T) * (size_t)TILE_J * (size_t)(jb->n_f > 0 ? jb->n_f : 1)); \
    T acc[TILE_J];                                                                       \
    const int64_t tj_count = (jb->n + TILE_J - 1) / TILE_J;                              \
    for (;;) {                                                                           \
      pthread_mutex_lock(jb->lock);                                                      \
      int64_t t = jb->next_tile++;                                                       \
      pthread_mutex_unlock(jb->lock);                                                    \
      if (t >= jb->n_tiles) break;                                                       \
      const int64_t tj = t % tj_count, ti = t / tj_count;                                \
      const int64_t j0 = tj * TILE_J, j1 = j0 + TILE_J < jb->n ? j0 + TILE_J : jb->n;    \
      const int64_t bw = j1 - j0;                                                        \
      /* contiguous copy of the V tile, rows = q (mingemm.py:106) */                     \
      for (int64_t q = 0; q < jb->n_f; ++q)                                              \
        for (int64_t jj = 0; jj < bw; ++jj) Vp[q * TILE_J + jj] = jb->V[(j0 + jj) * jb->ldv + q]; \
      const int64_t i0 = ti * TILE_I, i1 = i0 + TILE_I < jb->m ? i0 + TILE_I : jb->m;    \
      for (int64_t i = i0; i < i1; ++i) {                                                \
        for (int64_t jj = 0; jj < bw; ++jj) acc[jj] = (T)0;                              \
        const T* wcol = jb->W + i * jb->ldw;                                             \
        for (int64_t q = 0; q < jb->n_f; ++q) {                                          \
          const T w = wcol[q];                                                           \
          const T* row = Vp + q * TILE_J;                                                \
          for (int64_t jj = 0; jj < bw; ++jj) {                                          \
            const T v = row[jj];                                                         \
            acc[jj] = acc[jj] + (w < v ? w : v);                                         \
          }                                                                              \
        }                                                                                \
        for (int64_t jj = 0; jj < bw; ++jj) jb->M[i + (j0 + jj) * jb->ldm] = acc[jj];    \
      }                                                                                  \
    }                                                                                    \
    free(Vp);                                                                            \
    return NULL;                                                                         \
  }                                                                                      \
  void oracle_mgemm_##SUFFIX(const T* W, int64_t ldw, const T* V, int64_t ldv,           \
                             int64_t n_f, int64_t m, int64_t n, T* M, int64_t ldm,        \
                             int nthreads) {                                             \
    pthread_mutex_t lock = PTHREAD_MUTEX_INITIALIZER;                                    \
    mg_job_##SUFFIX jb = {W, ldw, V, ldv, n_f, m, n, M, ldm, 0,                          \
                          ((m + TILE_I - 1) / TILE_I) * ((n + TILE_J - 1) / TILE_J), &lock}; \
    if (nthreads < 1) nthreads = 1;                                                      \
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);            \
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, mg_worker_##SUFFIX, &jb); \
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);                        \
    free(th);                                                                            \
  }                                                                                      \
  void oracle_colsum_##SUFFIX(const T* V, int64_t ld, int64_t n_f, int64_t n, T* out) {  \
    for (int64_t i = 0; i < n; ++i) {                                                    \
      T acc = (T)0;                                                                      \
      for (int64_t q = 0; q < n_f; ++q) acc = acc + V[i * ld + q];                       \
      out[i] = acc;                                                                      \
    }                                                                                    \
  }

DEFINE_MGEMM(double, f64)
DEFINE_MGEMM(float, f32)

/* 128-bit checksum accumulation of one term. */
static void cks_add(uint64_t* lo, uint64_t* hi, uint64_t idx, uint64_t bits) {
  unsigned __int128 t = (unsigned __int128)mix64(idx) * (unsigned __int128)(mix64(bits) | 1ull);
  unsigned __int128 s = ((unsigned __int128)*hi << 64 | *lo) + t;
  *lo = (uint64_t)s;
  *hi = (uint64_t)(s >> 64);
}

/* Full single-rank 2-way run: vals[pair_index(i,j)] for all i<j, checksum
 * into cks[0..1] (lo, hi), returns the degenerate count. */
#define DEFINE_CZEK2(T, SUFFIX, BITS)                                                     \
  int64_t oracle_czek2_##SUFFIX(const T* V, int64_t ld, int64_t n_f, int64_t n_v, T* vals, \
                                uint64_t* cks, int nthreads) {                            \
    T* M = (T*)malloc(sizeof(T) * (size_t)n_v * (size_t)n_v);                            \
    T* s = (T*)malloc(sizeof(T) * (size_t)n_v);                                          \
    oracle_mgemm_##SUFFIX(V, ld, V, ld, n_f, n_v, n_v, M, n_v, nthreads);                \
    oracle_colsum_##SUFFIX(V, ld, n_f, n_v, s);                                          \
    uint64_t lo = 0, hi = 0;                                                             \
    int64_t deg = 0, p = 0;                                                              \
    for (int64_t i = 0; i < n_v; ++i)                                                    \
      for (int64_t j = i + 1; j < n_v; ++j, ++p) {                                       \
        const T d = s[i] + s[j];                                                         \
        T v;                                                                             \
        if (d == (T)0) { v = (T)0; ++deg; } else v = ((T)2 * M[i + j * n_v]) / d;       \
        vals[p] = v;                                                                     \
        cks_add(&lo, &hi, (uint64_t)p, BITS(v));                                         \
      }                                                                                  \
    cks[0] = lo;                                                                         \
    cks[1] = hi;                                                                         \
    free(M);                                                                             \
    free(s);                                                                             \
    return deg;                                                                          \
  }

static uint64_t bits_f64(double v) { uint64_t b; memcpy(&b, &v, 8); return b; }
static uint64_t bits_f32(float v) { uint32_t b; memcpy(&b, &v, 4); return (uint64_t)b; }

DEFINE_CZEK2(double, f64, bits_f64)
DEFINE_CZEK2(float, f32, bits_f32)

/* mix64 exported for the known-answer tests. */
uint64_t oracle_mix64(uint64_t x) { return mix64(x); }
