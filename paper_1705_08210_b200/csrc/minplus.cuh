// The min-plus ("mGEMM") CTA mainloop on CUDA cores for sm_100a.
//
//   acc[i][j] = sum_q min(W[q, i], V[q, j])      (mingemm.py:94-117)
//
// Each output element is accumulated by exactly one thread, sequentially in
// ascending q, starting from +0 in the run dtype (mingemm.py:86, 110-116;
// SURVEY Appendix C rules 1-4). There is no split-K and no partial
// accumulator, so the sum order -- and hence every bit -- matches the
// reference's naive/blocked kernels on any NaN-free input.
//
// Layout: vectors are columns with q contiguous (element (q, i) at i*ld + q,
// core.py:235-236), so both operands are "K-major". A 128-byte field chunk of
// the tile's vectors is staged into shared memory with 16-byte cp.async
// copies (zero-filled past n_f / past the last vector: min(0, x) adds +0,
// which leaves every nonnegative sum bit-identical), STAGES deep. Shared rows
// are padded to a 144-byte pitch so the LDS.128 operand fetches of a warp
// (4 distinct A rows, 8 distinct B rows) hit distinct bank groups.
//
// Register micro-tile: 256 threads as a 16 x 16 grid, TM x TN outputs each,
// CTA tile (16 TM) x (16 TN). Thread (ty, tx) owns rows ty + 16m and columns
// tx + 16n. One LDS.128 brings 2 (FP64) or 4 (FP32) consecutive q of one
// vector; for each q in order every accumulator is updated.
//
// Instruction mix per comparison (sm_100a SASS):
//   FP64: DSETP + FSEL + FSEL + DADD      (no DMNMX exists; `w < v ? w : v`)
//   FP32: FMNMX + half an FADD2 (packed f32x2 add over two accumulators)
#pragma once

#include <type_traits>

#include "psim_common.cuh"
#include "psim_internal.h"

namespace psim {

constexpr int kNT = 256;  // threads per CTA (16 x 16)

// Unroll factor of the per-stage micro-step loop: measured (exp_minplus,
// profiles/r01_unroll_sweep.jsonl) FP64 best rolled (1: the 8.5 KB body stays
// in the instruction cache; +0.9% vs full), FP32 best at 4 (+0.7%).
// -DPSIM_KK_UNROLL=u overrides it for experiments.

constexpr int kPitchBytes = 144;

// Tile configuration: TM x TN per thread, STAGES-deep cp.async pipeline,
// MINB CTAs per SM requested from ptxas (__launch_bounds__).
template <typename T_, int TM_, int TN_, int STAGES_, int MINB_, int VAR_ = 0, int MAP_ = 0>
struct Cfg {
  using T = T_;
  static constexpr int TM = TM_, TN = TN_, STAGES = STAGES_, MINB = MINB_;
  // FP32 inner-op variant: 0 FMNMX + FADD2, 1 FMNMX + FADD, 2 IMNMX + FADD2,
  // 3 IMNMX + FADD (integer min on the bits: exact for nonnegative floats)
  static constexpr int VAR = VAR_;
  // thread grid of a warp (thread_ty / thread_tx): 0 = 4 rows x 8 columns
  // (a warp pair shares its A rows), 1 = 2 rows x 16 columns (measured 0.6%
  // slower on cfg2, profiles/r02_final/map_ab/; kept for A/B builds)
  static constexpr int MAP = MAP_;
  static constexpr int BM = 16 * TM;                 // CTA tile rows (W vectors)
  static constexpr int BN = 16 * TN;                 // CTA tile cols (V vectors)
  static constexpr int BK = 128 / (int)sizeof(T);    // q per stage (one 128-B chunk)
  static constexpr int VEC = 16 / (int)sizeof(T);    // q per LDS.128
  static constexpr int PITCH = kPitchBytes / (int)sizeof(T);
  static constexpr int STAGE_ELEMS = (BM + BN) * PITCH + 2 * BK;  // A, B, 2 pivot chunks
#ifdef PSIM_KK_UNROLL
  static constexpr int KKU = PSIM_KK_UNROLL;
#else
  static constexpr int KKU = std::is_same<T_, double>::value ? 1
                             : std::is_same<T_, float>::value ? 4 : BK / VEC;
#endif
  static constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * (int)sizeof(T);
  static_assert((BM * 8) % kNT == 0 && (BN * 8) % kNT == 0, "tile / thread mismatch");
  static_assert(sizeof(T) == 8 || TN % 2 == 0, "FP32 pairs columns for FADD2");
};

// Production configurations (tile shape of the 2-way and 3-way kernels).
template <typename T>
struct Prod;
// (-DPSIM_F64_TN= / _STAGES= / _MINB= / _MAP= override it for A/B builds,
// tools/build_variant.sh)
#ifndef PSIM_F64_TN
#define PSIM_F64_TN 8
#endif
#ifndef PSIM_F64_STAGES
#define PSIM_F64_STAGES 4
#endif
#ifndef PSIM_F64_MINB
#define PSIM_F64_MINB 1
#endif
#ifndef PSIM_F64_MAP
#define PSIM_F64_MAP 0
#endif
template <>
struct Prod<double> {  // 128 x 128, 1 CTA/SM, 4 stages
  using C = Cfg<double, 8, PSIM_F64_TN, PSIM_F64_STAGES, PSIM_F64_MINB, 0, PSIM_F64_MAP>;
};

// 3-way tiles (k_czek3; psim_tile_shape reports their shape): 128 x 128 FP64
// / 128 x 64 FP32 on the 4 x 8 warp grid, which the per-warp pivot rewrite
// (minplus_tile_pivot_ilv) is written for. Fixed, so 2-way A/B builds leave
// the 3-way kernels alone.
template <typename T>
struct Tile3Cfg;
template <>
struct Tile3Cfg<double> {
  using C = Cfg<double, 8, 8, 4, 1, 0, 0>;
};
template <>
struct Tile3Cfg<float> {
  using C = Cfg<float, 8, 4, 3, 2, 1, 0>;
};
// (-DPSIM_F32_TN= / _STAGES= / _MINB= / _VAR= override it for A/B builds,
// tools/build_variant.sh)
#ifndef PSIM_F32_TN
#define PSIM_F32_TN 4
#endif
#ifndef PSIM_F32_STAGES
#define PSIM_F32_STAGES 3
#endif
#ifndef PSIM_F32_MINB
#define PSIM_F32_MINB 2
#endif
#ifndef PSIM_F32_VAR
#define PSIM_F32_VAR 1
#endif
template <>
struct Prod<float> {  // 128 x 64, 2 CTAs/SM, 3 stages, scalar FADD
  using C = Cfg<float, 8, PSIM_F32_TN, PSIM_F32_STAGES, PSIM_F32_MINB, PSIM_F32_VAR>;
};

// Edge configurations: 32-row tiles for the last, ragged row tile of a 2-way
// task (a 5000-vector block leaves 8 rows in its 40th 128-row tile).
template <typename T>
struct Edge;
template <>
struct Edge<double> {
  using C = Cfg<double, 2, 8, 4, 2, 0>;  // 32 x 128
};
template <>
struct Edge<float> {
  using C = Cfg<float, 2, 4, 3, 4, 1>;  // 32 x 64
};

// FP32 packed add: two independent accumulators, each rounded exactly as a
// scalar __fadd_rn (add.rn.f32x2 keeps subnormals; no .ftz).
__device__ __forceinline__ void fadd2(float& a0, float& a1, float x0, float x1) {
  asm("{\n\t.reg .b64 t, s;\n\t"
      "mov.b64 t, {%0, %1};\n\t"
      "mov.b64 s, {%2, %3};\n\t"
      "add.rn.f32x2 t, t, s;\n\t"
      "mov.b64 {%0, %1}, t;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(x0), "f"(x1));
}

// One LDS.128 step (VEC consecutive q) of the register micro-kernel.
template <class C>
__device__ __forceinline__ void micro_step(double (&acc)[C::TM][C::TN], const double* As,
                                           const double* Bs, int ty, int tx, int kk) {
  constexpr int P = C::PITCH;
  // (measured alternatives, profiles/r01_tile_sweep.jsonl: B-stationary
  // register tiles and per-element q pairs are no faster; the FP64 mix tops
  // out near 21.3 cmp/clk/SM for every tile shape)
  double2 a[C::TM];
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
    a[m] = *reinterpret_cast<const double2*>(As + (ty + 16 * m) * P + kk);
#pragma unroll
  for (int n = 0; n < C::TN; ++n) {
    const double2 b = *reinterpret_cast<const double2*>(Bs + (tx + 16 * n) * P + kk);
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
      acc[m][n] = __dadd_rn(acc[m][n], Traits<double>::min(a[m].x, b.x));
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
      acc[m][n] = __dadd_rn(acc[m][n], Traits<double>::min(a[m].y, b.y));
  }
}

// min of two nonnegative floats; VAR 2/3 compare the bit patterns as signed
// ints (the order of nonnegative IEEE floats; -0 sorts below +0, harmless
// because the sums start at +0).
template <int VAR>
__device__ __forceinline__ float fmin_v(float a, float b) {
  if (VAR >= 2) return __int_as_float(min(__float_as_int(a), __float_as_int(b)));
  return fminf(a, b);
}

template <class C>
__device__ __forceinline__ void micro_step(float (&acc)[C::TM][C::TN], const float* As,
                                           const float* Bs, int ty, int tx, int kk) {
  constexpr int P = C::PITCH;
  float4 a[C::TM];
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
    a[m] = *reinterpret_cast<const float4*>(As + (ty + 16 * m) * P + kk);
  if constexpr (C::VAR % 2 == 1) {  // scalar adds
#pragma unroll
    for (int n = 0; n < C::TN; ++n) {
      const float4 b = *reinterpret_cast<const float4*>(Bs + (tx + 16 * n) * P + kk);
#pragma unroll
      for (int m = 0; m < C::TM; ++m) acc[m][n] = __fadd_rn(acc[m][n], fmin_v<C::VAR>(a[m].x, b.x));
#pragma unroll
      for (int m = 0; m < C::TM; ++m) acc[m][n] = __fadd_rn(acc[m][n], fmin_v<C::VAR>(a[m].y, b.y));
#pragma unroll
      for (int m = 0; m < C::TM; ++m) acc[m][n] = __fadd_rn(acc[m][n], fmin_v<C::VAR>(a[m].z, b.z));
#pragma unroll
      for (int m = 0; m < C::TM; ++m) acc[m][n] = __fadd_rn(acc[m][n], fmin_v<C::VAR>(a[m].w, b.w));
    }
  } else {
#pragma unroll
  for (int n = 0; n < C::TN; n += 2) {
    const float4 b0 = *reinterpret_cast<const float4*>(Bs + (tx + 16 * n) * P + kk);
    const float4 b1 = *reinterpret_cast<const float4*>(Bs + (tx + 16 * (n + 1)) * P + kk);
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
      fadd2(acc[m][n], acc[m][n + 1], fmin_v<C::VAR>(a[m].x, b0.x), fmin_v<C::VAR>(a[m].x, b1.x));
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
      fadd2(acc[m][n], acc[m][n + 1], fmin_v<C::VAR>(a[m].y, b0.y), fmin_v<C::VAR>(a[m].y, b1.y));
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
      fadd2(acc[m][n], acc[m][n + 1], fmin_v<C::VAR>(a[m].z, b0.z), fmin_v<C::VAR>(a[m].z, b1.z));
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
      fadd2(acc[m][n], acc[m][n + 1], fmin_v<C::VAR>(a[m].w, b0.w), fmin_v<C::VAR>(a[m].w, b1.w));
  }
  }
}

// Bit-packed 0/1 operands (Sorenson, sorenson.cu): 4 uint32 words = 128 fields
// per LDS.128; the count of a pair is popc(a & b) summed over words
// (mgemm_bitpacked, mingemm.py:294-312). Integer adds: any order is exact.
template <class C>
__device__ __forceinline__ void micro_step(uint32_t (&acc)[C::TM][C::TN], const uint32_t* As,
                                           const uint32_t* Bs, int ty, int tx, int kk) {
  constexpr int P = C::PITCH;
  uint4 a[C::TM];
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
    a[m] = *reinterpret_cast<const uint4*>(As + (ty + 16 * m) * P + kk);
#pragma unroll
  for (int n = 0; n < C::TN; ++n) {
    const uint4 b = *reinterpret_cast<const uint4*>(Bs + (tx + 16 * n) * P + kk);
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
      acc[m][n] += (__popc(a[m].x & b.x) + __popc(a[m].y & b.y)) +
                   (__popc(a[m].z & b.z) + __popc(a[m].w & b.w));
  }
}

// Stage field chunk kt of `rows` W vectors and `cols` V vectors (and, with
// PIVOT, of the pivot column) into stage buffer `st`. TWO: the tile's columns
// come from two blocks -- columns >= split are read from V2b + col * ldv
// (V2b = the second block's first vector minus split vectors).
template <class C, bool PIVOT, bool TWO = false>
__device__ __forceinline__ void stage_load(typename C::T* st, const typename C::T* __restrict__ W,
                                           int64_t ldw, int rows,
                                           const typename C::T* __restrict__ V, int64_t ldv,
                                           int cols, const typename C::T* __restrict__ xj,
                                           int64_t n_f, int kt,
                                           const typename C::T* V2b = nullptr, int split = 0) {
  using T = typename C::T;
  const int tid = threadIdx.x;
  const int64_t q_base = (int64_t)kt * C::BK;
#pragma unroll
  for (int r = 0; r < (C::BM * 8) / kNT; ++r) {
    const int c = tid + r * kNT;
    const int row = c >> 3, ch = c & 7;
    const int64_t q0 = q_base + ch * C::VEC;
    const int64_t rem = (n_f - q0) * (int64_t)sizeof(T);
    int bytes = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
    const T* src = W;
    if (row < rows && bytes) src = W + row * ldw + q0; else bytes = 0;
    cp_async16(st + row * C::PITCH + ch * C::VEC, src, bytes);
  }
#pragma unroll
  for (int r = 0; r < (C::BN * 8) / kNT; ++r) {
    const int c = tid + r * kNT;
    const int row = c >> 3, ch = c & 7;
    const int64_t q0 = q_base + ch * C::VEC;
    const int64_t rem = (n_f - q0) * (int64_t)sizeof(T);
    int bytes = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
    const T* src = V;
    const T* vb = V;
    if constexpr (TWO) vb = row < split ? V : V2b;
    if (row < cols && bytes) src = vb + row * ldv + q0; else bytes = 0;
    cp_async16(st + (C::BM + row) * C::PITCH + ch * C::VEC, src, bytes);
  }
}

// Pivot chunk kt (3-way) into the pivot slot of stage buffer `st`.
template <class C>
__device__ __forceinline__ void pivot_load(typename C::T* st, const typename C::T* __restrict__ xj,
                                           int64_t n_f, int kt) {
  using T = typename C::T;
  const int tid = threadIdx.x;
  if (tid < 8) {
    const int64_t q0 = (int64_t)kt * C::BK + tid * C::VEC;
    const int64_t rem = (n_f - q0) * (int64_t)sizeof(T);
    const int bytes = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
    cp_async16(st + (C::BM + C::BN) * C::PITCH + tid * C::VEC, bytes ? xj + q0 : xj, bytes);
  }
}

// 3-way prologue on a landed stage: A[r][q] <- min(x_j[q], A[r][q])
// (xj_columns, mingemm.py:225-234). min is exact, so the later sum of
// min(X, V_k) equals sum_q min(min(x_j, v_i), v_k) bit for bit (Appendix C r8).
// Runs after the stage's barrier; each thread rewrites the A chunks its own
// cp.asyncs brought in, with the stage's pivot chunk `xs`.
template <class C>
__device__ __forceinline__ void stage_pivot_min(typename C::T* st, const typename C::T* xs) {
  // 16-byte vector accesses: a warp's 8 consecutive lanes cover one row's
  // 128 B (distinct banks), so the rewrite is conflict-free.
  using V4 = typename std::conditional<sizeof(typename C::T) == 8, double2, float4>::type;
  const int tid = threadIdx.x;
  const int ch = tid & 7;  // the same chunk column for all of this thread's rows
  const V4 x = *reinterpret_cast<const V4*>(xs + ch * C::VEC);
#pragma unroll
  for (int r = 0; r < (C::BM * 8) / kNT; ++r) {
    const int row = (tid + r * kNT) >> 3;
    V4* p = reinterpret_cast<V4*>(st + row * C::PITCH + ch * C::VEC);
    V4 a = *p;
    if constexpr (sizeof(typename C::T) == 8) {
      a.x = Traits<double>::min(x.x, a.x);
      a.y = Traits<double>::min(x.y, a.y);
    } else {
      a.x = Traits<float>::min(x.x, a.x);
      a.y = Traits<float>::min(x.y, a.y);
      a.z = Traits<float>::min(x.z, a.z);
      a.w = Traits<float>::min(x.w, a.w);
    }
    *p = a;
  }
}

// Thread (ty, tx) of the 16 x 16 grid: MAP 0 gives each warp 4 rows x 8
// columns (warps 2p, 2p + 1 share rows), MAP 1 2 rows x 16 columns (every A
// row read by one warp; a B fetch covers 256 contiguous-pitch bytes).
template <int MAP = 0>
__device__ __forceinline__ int thread_ty() {
  if constexpr (MAP == 1) return (threadIdx.x >> 5) * 2 + ((threadIdx.x & 31) >> 4);
  return ((threadIdx.x >> 5) >> 1) * 4 + ((threadIdx.x & 31) >> 3);
}
template <int MAP = 0>
__device__ __forceinline__ int thread_tx() {
  if constexpr (MAP == 1) return threadIdx.x & 15;
  return ((threadIdx.x >> 5) & 1) * 8 + (threadIdx.x & 7);
}

// Full-depth mainloop for one tile. `W` / `V` point at the first vector of
// the tile's rows / columns. All threads of the CTA must call it.
// SUMS: thread t < BM + BN also folds the column sum of tile vector t (rows,
// then columns) from the staged chunks -- sequential ascending q from +0,
// the order of k_colsum, so the sum is bit-identical -- into *vsum.
template <class C, bool PIVOT, bool SUMS = false, bool TWO = false>
__device__ __forceinline__ void minplus_tile(const typename C::T* __restrict__ W, int64_t ldw,
                                             int rows, const typename C::T* __restrict__ V,
                                             int64_t ldv, int cols,
                                             const typename C::T* __restrict__ xj, int64_t n_f,
                                             typename C::T (&acc)[C::TM][C::TN],
                                             typename C::T* smem,
                                             typename C::T* vsum = nullptr,
                                             const typename C::T* V2b = nullptr, int split = 0) {
  using T = typename C::T;
  using V4 = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  constexpr int S = C::STAGES;
  const int ty = thread_ty<C::MAP>(), tx = thread_tx<C::MAP>();
  T vs = T();
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = T(0);

  const int KT = (int)((n_f + C::BK - 1) / C::BK);
  constexpr int XS = (C::BM + C::BN) * C::PITCH;  // pivot slot offset inside a stage
  // PIVOT with >= 4 stages: the pivot min of stage kt+1 is applied in
  // iteration kt, right after the one barrier that also publishes stage kt,
  // so a 3-way tile needs no second barrier per stage (one stage less of
  // prefetch depth). Each thread rewrites exactly the chunks its own
  // cp.asyncs brought in; the barrier publishes the pivot chunk.
  constexpr bool AHEAD = PIVOT && S >= 4;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < KT) {
      stage_load<C, PIVOT, TWO>(smem + s * C::STAGE_ELEMS, W, ldw, rows, V, ldv, cols, xj, n_f,
                                s, V2b, split);
      if (PIVOT) pivot_load<C>(smem + s * C::STAGE_ELEMS, xj, n_f, s);
    }
    cp_async_commit();
  }
  if (AHEAD && KT > 0) {
    cp_async_wait<S - 2>();
    __syncthreads();
    stage_pivot_min<C>(smem, smem + XS);
  }
  for (int kt = 0; kt < KT; ++kt) {
    if constexpr (AHEAD) {
      cp_async_wait<(AHEAD ? S - 3 : 0)>();
    } else {
      cp_async_wait<S - 2>();
    }
    __syncthreads();
    T* st = smem + (kt % S) * C::STAGE_ELEMS;
    if constexpr (AHEAD) {
      if (kt + 1 < KT) {
        T* nx = smem + ((kt + 1) % S) * C::STAGE_ELEMS;
        stage_pivot_min<C>(nx, nx + XS);
      }
    } else if (PIVOT) {
      // (measured: transforming own chunks before the barrier with the pivot
      // staged one group early was 3% slower than this extra barrier)
      stage_pivot_min<C>(st, st + XS);
      __syncthreads();
    }
    const int nk = kt + S - 1;
    if (nk < KT) {
      stage_load<C, PIVOT, TWO>(smem + (nk % S) * C::STAGE_ELEMS, W, ldw, rows, V, ldv, cols,
                                xj, n_f, nk, V2b, split);
      if (PIVOT) pivot_load<C>(smem + (nk % S) * C::STAGE_ELEMS, xj, n_f, nk);
    }
    cp_async_commit();
    if constexpr (SUMS) {
      if (threadIdx.x < C::BM + C::BN) {
        // LDS.128: 8 consecutive threads read 8 rows' 16 B at a 144-B pitch = distinct banks
        const V4* p = reinterpret_cast<const V4*>(st + threadIdx.x * C::PITCH);
#pragma unroll
        for (int h = 0; h < C::BK / C::VEC; ++h) {
          const V4 x = p[h];
          if constexpr (sizeof(T) == 8) {
            vs = Traits<T>::add(Traits<T>::add(vs, x.x), x.y);
          } else {
            vs = Traits<T>::add(
                Traits<T>::add(Traits<T>::add(Traits<T>::add(vs, x.x), x.y), x.z), x.w);
          }
        }
      }
    }
    const T* As = st;
    const T* Bs = st + C::BM * C::PITCH;
    // (the 3-way pivot loop keeps the full unroll: rolled it measured 2% slower)
#ifdef PSIM_PIVOT_KKU
    constexpr int U = PIVOT ? PSIM_PIVOT_KKU : C::KKU;
#else
    constexpr int U = PIVOT ? C::BK / C::VEC : C::KKU;
#endif
#pragma unroll U
    for (int kk = 0; kk < C::BK; kk += C::VEC) micro_step<C>(acc, As, Bs, ty, tx, kk);
  }
  cp_async_wait<0>();
  if constexpr (SUMS) *vsum = vs;
}

// ---------------------------------------------------------------------------
// TMA staging (sm_100a): the same stage layout -- (BM + BN) rows at the
// 144-byte pitch -- filled by two cp.async.bulk.tensor 2-D box loads per stage
// (box = PITCH fields x BM or BN vectors; the PITCH - BK fields past the chunk
// belong to the next one and are never read; fields past n_f and vectors past
// the operand's end arrive as zeros, as with cp.async), issued by one thread
// and signalled on a per-stage "full" mbarrier with the transaction byte
// count. Each warp releases a stage on its "empty" mbarrier when it is done
// with it; the issuing thread refills the slot once all eight warps have.
// No CTA-wide barrier per stage and no per-thread copy instructions: warps
// drift up to STAGES - 1 stages apart. Measured (tools/exp_tma.cu,
// profiles/r02_tma_ab.jsonl): 22.64 vs 21.54 cmp/clk/SM for the FP64 tile,
// i.e. the rate of the mainloop on operands already in shared memory.

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// Box (PITCH fields from field q0) x (rows from vector v0) of the tensor map.
__device__ __forceinline__ void tma_box(void* dst, const void* map, int q0, int v0,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(q0), "r"(v0), "r"(smem_u32(bar))
      : "memory");
}

// Mainloop of one tile with TMA staging: mapW / mapV are __grid_constant__
// tensor maps of the W and V operands (dims {n_f, vectors}, stride ld),
// w_row0 / v_row0 the tile's first vector in each. All threads must call it.
template <class C>
__device__ __forceinline__ void minplus_tile_tma(const void* mapW, int w_row0, const void* mapV,
                                                 int v_row0, int64_t n_f,
                                                 typename C::T (&acc)[C::TM][C::TN],
                                                 typename C::T* smem) {
  using T = typename C::T;
  constexpr int S = C::STAGES;
  constexpr unsigned kBytes = (C::BM + C::BN) * C::PITCH * sizeof(T);
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = T(0);
  __syncthreads();
  const int KT = (int)((n_f + C::BK - 1) / C::BK);
  auto issue = [&](int kt) {
    const int s = kt % S;
    T* st = smem + s * C::STAGE_ELEMS;
    mbar_expect_tx(&full[s], kBytes);
    tma_box(st, mapW, kt * C::BK, w_row0, &full[s]);
    tma_box(st + C::BM * C::PITCH, mapV, kt * C::BK, v_row0, &full[s]);
  };
  if (tid == 0)
    for (int kt = 0; kt < S && kt < KT; ++kt) issue(kt);
  const int ty = thread_ty<C::MAP>(), tx = thread_tx<C::MAP>();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % S;
    const unsigned ph = (unsigned)(kt / S) & 1u;
    mbar_wait(&full[s], ph);
    const T* st = smem + s * C::STAGE_ELEMS;
#pragma unroll C::KKU
    for (int kk = 0; kk < C::BK; kk += C::VEC)
      micro_step<C>(acc, st, st + C::BM * C::PITCH, ty, tx, kk);
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && kt + S < KT) {
      mbar_wait(&empty[s], ph);  // all warps are done with this slot
      issue(kt + S);
    }
  }
}

// 3-way single-pivot tile with TMA staging, per-warp interleaved pivot min:
// the A rows a warp reads in micro_step are ty + 16 m with ty in
// {4 (w/2) .. 4 (w/2) + 3}, so each warp rewrites exactly those 32 rows,
// A[r][q] <- min(x_j[q], A[r][q]) (xj_columns, mingemm.py:225-234), and needs
// no other warp's work: no "ready" barrier, only full / empty as in the 2-way
// loop. The two warps of a pair read (and so rewrite) the same rows; min is
// idempotent, so the second rewrite stores the values already there. The
// rewrite of stage kt + A is spread over the micro-steps of stage kt:
// micro-step u loads chunk u (row ty0 + 16u, this lane's 16 bytes) at its top
// and stores min(x, chunk) at its bottom, so the load latency hides behind
// the micro-step's FP instructions. Measured (tools/exp_pivot_tma.cu,
// profiles/r02_3way_pivot/, FP64 128 x 128 tiles, cmp/clk/SM): 2-way loop
// 22.26 / 22.68 (n_f = 20000 / 10000), the earlier "ready"-barrier loop (now
// tools/exp_pivot_tma.cu: minplus_tile_pivot_tma) 18.25 /
// 20.41 (the barrier alone costs 2-4%, and it bounds warp skew to D stages),
// this loop with A = 1 21.38 / 21.81 (96% of the 2-way loop), bitwise equal.
template <class C, int A>
__device__ __forceinline__ void minplus_tile_pivot_ilv(const void* mapA, int a_row0,
                                                       const void* mapC, int c_row0,
                                                       const void* mapB, int p_row, int64_t n_f,
                                                       typename C::T (&acc)[C::TM][C::TN],
                                                       typename C::T* smem) {
  using T = typename C::T;
  using V4 = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  static_assert(C::BK / C::VEC == C::TM, "one chunk of the warp's rows per micro-step");
  static_assert(A >= 1 && A < C::STAGES, "transform distance");
  static_assert(C::MAP == 0, "the per-warp rewrite follows the 4 x 8 warp grid");
  constexpr int S = C::STAGES;
  constexpr int XS = (C::BM + C::BN) * C::PITCH;  // pivot slot inside a stage
  constexpr unsigned kBytes = (C::BM + C::BN + 1) * C::PITCH * sizeof(T);
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = T(0);
  __syncthreads();
  const int KT = (int)((n_f + C::BK - 1) / C::BK);
  auto issue = [&](int kt) {
    const int s = kt % S;
    T* st = smem + s * C::STAGE_ELEMS;
    mbar_expect_tx(&full[s], kBytes);
    tma_box(st, mapA, kt * C::BK, a_row0, &full[s]);
    tma_box(st + C::BM * C::PITCH, mapC, kt * C::BK, c_row0, &full[s]);
    tma_box(st + XS, mapB, kt * C::BK, p_row, &full[s]);
  };
  auto vmin = [](const V4& x, V4 a) {
    if constexpr (sizeof(T) == 8) {
      a.x = Traits<double>::min(x.x, a.x);
      a.y = Traits<double>::min(x.y, a.y);
    } else {
      a.x = Traits<float>::min(x.x, a.x);
      a.y = Traits<float>::min(x.y, a.y);
      a.z = Traits<float>::min(x.z, a.z);
      a.w = Traits<float>::min(x.w, a.w);
    }
    return a;
  };
  // this lane's chunk u: row (w/2)*4 + lane/8 + 16u, 16-byte column lane%8
  const int xoff = (lane & 7) * C::VEC;
  const int roff = ((w >> 1) * 4 + (lane >> 3)) * C::PITCH + xoff;
  if (tid == 0)
    for (int kt = 0; kt < S && kt < KT; ++kt) issue(kt);
  for (int kt = 0; kt < A && kt < KT; ++kt) {  // the first A stages up front
    T* st = smem + (kt % S) * C::STAGE_ELEMS;
    mbar_wait(&full[kt % S], (unsigned)(kt / S) & 1u);
    const V4 x = *reinterpret_cast<const V4*>(st + XS + xoff);
#pragma unroll
    for (int u = 0; u < C::TM; ++u) {
      V4* p = reinterpret_cast<V4*>(st + roff + 16 * u * C::PITCH);
      *p = vmin(x, *p);
    }
  }
  __syncwarp();
  const int ty = thread_ty(), tx = thread_tx();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % S;
    const unsigned ph = (unsigned)(kt / S) & 1u;
    const bool xf = kt + A < KT;
    T* nx = smem + ((kt + A) % S) * C::STAGE_ELEMS;
    V4 x{};
    if (xf) {
      mbar_wait(&full[(kt + A) % S], (unsigned)((kt + A) / S) & 1u);
      x = *reinterpret_cast<const V4*>(nx + XS + xoff);
    }
    const T* st = smem + s * C::STAGE_ELEMS;
#pragma unroll 1
    for (int u = 0; u < C::TM; ++u) {
      V4* pa = reinterpret_cast<V4*>(nx + roff + 16 * u * C::PITCH);
      V4 a{};
      if (xf) a = *pa;
      micro_step<C>(acc, st, st + C::BM * C::PITCH, ty, tx, u * C::VEC);
      if (xf) *pa = vmin(x, a);
    }
    // this warp's generic-proxy writes (stage kt + A) before the async-proxy
    // refill of that slot, which follows every warp's release of it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && kt + S < KT) {
      mbar_wait(&empty[s], ph);
      issue(kt + S);
    }
  }
}

// First column tile of row-tile b in a diagonal task (the tile holding
// column b*BM + 1: every tile with some i < j); 0 for rectangles.
__host__ __device__ __forceinline__ int64_t first_col_tile(int64_t b, int64_t bm, int64_t bn,
                                                           int diagonal) {
  return diagonal ? (b * bm + 1) / bn : 0;
}

// Banded rasterisation (2-way kernels, czek2.cu): row-tiles are grouped in
// bands of G ~ sqrt(resident CTAs); inside a band tiles run column-major (all
// G rows of one column tile, then the next), so the CTAs resident at the same
// time share ~G row panels and ~W/G column panels in L2 instead of one row
// panel and W column panels (W = resident CTAs). band_pref[b] = tiles before
// band b (device); in a diagonal band the tiles left of a row's first column
// are enumerated too and skipped (returns false) -- at most G(G-1)/2 empty
// CTAs per band.
__device__ __forceinline__ bool band_tile(int64_t t, const int64_t* __restrict__ band_pref,
                                          int64_t nbands, int64_t G, int64_t row_tile0,
                                          int64_t row_tile_end, int64_t bm, int64_t bn,
                                          int diagonal, int& bi, int& bj) {
  int64_t lo = 0, hi = nbands;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (ld_pref(band_pref + mid) <= t) lo = mid; else hi = mid;
  }
  const int64_t r0 = row_tile0 + lo * G;
  const int64_t rows = min64(G, row_tile_end - r0);
  const int64_t u = t - ld_pref(band_pref + lo);
  const int64_t b = r0 + u % rows;
  const int64_t c = first_col_tile(r0, bm, bn, diagonal) + u / rows;
  bi = (int)b;
  bj = (int)c;
  return c >= first_col_tile(b, bm, bn, diagonal);
}

}  // namespace psim
