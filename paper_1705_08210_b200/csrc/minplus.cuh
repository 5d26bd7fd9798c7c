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
// 128 vectors per operand is staged into shared memory with 16-byte
// cp.async copies (zero-filled past n_f / past the last vector: min(0, x)
// adds +0, which leaves every nonnegative sum bit-identical). Shared rows
// are padded to a 144-byte pitch so that the LDS.128 operand fetches of a
// warp (4 distinct A rows, 8 distinct B rows) hit distinct bank groups.
//
// Register micro-tile: 256 threads, 8x8 outputs each, CTA tile 128x128.
// Thread (ty, tx) owns rows ty + 16m and columns tx + 16n. One LDS.128
// brings 2 (FP64) or 4 (FP32) consecutive q of one vector; for each q in
// order every accumulator is updated, keeping each element's q order.
//
// Instruction mix per comparison (sm_100a SASS):
//   FP64: DSETP.MIN + SEL + FSEL + DADD          (no DMNMX exists)
//   FP32: FMNMX + half of an FADD2 (packed f32x2 add, two accumulators)
#pragma once

#include "psim_common.cuh"
#include "psim_internal.h"

namespace psim {

constexpr int kBM = 128;        // CTA tile rows (W vectors)
constexpr int kBN = 128;        // CTA tile cols (V vectors)
constexpr int kTM = 8;          // per-thread rows
constexpr int kTN = 8;          // per-thread cols
constexpr int kNT = 256;        // threads per CTA
constexpr int kPitchBytes = 144;
static_assert(kBM == kTileM && kBN == kTileN, "tile constants out of sync");

template <typename T>
struct Tile {
  static constexpr int BK = 128 / (int)sizeof(T);          // q per stage (one 128-B chunk)
  static constexpr int VEC = 16 / (int)sizeof(T);          // q per LDS.128
  static constexpr int PITCH = kPitchBytes / (int)sizeof(T);
  static constexpr int STAGE_ELEMS = (kBM + kBN) * PITCH + BK;  // A, B, pivot chunk
  static constexpr int STAGES = sizeof(T) == 8 ? 4 : 4;
  static constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * (int)sizeof(T);
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

template <typename T>
struct Micro;

template <>
struct Micro<double> {
  // One LDS.128 step: 2 consecutive q for every (m, n).
  __device__ __forceinline__ static void step(double (&acc)[kTM][kTN], const double* As,
                                              const double* Bs, int ty, int tx, int kk) {
    constexpr int P = Tile<double>::PITCH;
    double2 a[kTM];
#pragma unroll
    for (int m = 0; m < kTM; ++m)
      a[m] = *reinterpret_cast<const double2*>(As + (ty + 16 * m) * P + kk);
#pragma unroll
    for (int n = 0; n < kTN; ++n) {
      const double2 b = *reinterpret_cast<const double2*>(Bs + (tx + 16 * n) * P + kk);
#pragma unroll
      for (int m = 0; m < kTM; ++m) acc[m][n] = __dadd_rn(acc[m][n], Traits<double>::min(a[m].x, b.x));
#pragma unroll
      for (int m = 0; m < kTM; ++m) acc[m][n] = __dadd_rn(acc[m][n], Traits<double>::min(a[m].y, b.y));
    }
  }
};

template <>
struct Micro<float> {
  // One LDS.128 step: 4 consecutive q; columns n, n+1 share an FADD2.
  __device__ __forceinline__ static void step(float (&acc)[kTM][kTN], const float* As,
                                              const float* Bs, int ty, int tx, int kk) {
    constexpr int P = Tile<float>::PITCH;
    float4 a[kTM];
#pragma unroll
    for (int m = 0; m < kTM; ++m)
      a[m] = *reinterpret_cast<const float4*>(As + (ty + 16 * m) * P + kk);
#pragma unroll
    for (int n = 0; n < kTN; n += 2) {
      const float4 b0 = *reinterpret_cast<const float4*>(Bs + (tx + 16 * n) * P + kk);
      const float4 b1 = *reinterpret_cast<const float4*>(Bs + (tx + 16 * (n + 1)) * P + kk);
#pragma unroll
      for (int m = 0; m < kTM; ++m)
        fadd2(acc[m][n], acc[m][n + 1], fminf(a[m].x, b0.x), fminf(a[m].x, b1.x));
#pragma unroll
      for (int m = 0; m < kTM; ++m)
        fadd2(acc[m][n], acc[m][n + 1], fminf(a[m].y, b0.y), fminf(a[m].y, b1.y));
#pragma unroll
      for (int m = 0; m < kTM; ++m)
        fadd2(acc[m][n], acc[m][n + 1], fminf(a[m].z, b0.z), fminf(a[m].z, b1.z));
#pragma unroll
      for (int m = 0; m < kTM; ++m)
        fadd2(acc[m][n], acc[m][n + 1], fminf(a[m].w, b0.w), fminf(a[m].w, b1.w));
    }
  }
};

// Stage one 128-byte field chunk kt of `rows` W vectors and `cols` V vectors
// (and, with PIVOT, of the pivot column) into stage buffer `st`.
template <typename T, bool PIVOT>
__device__ __forceinline__ void stage_load(T* st, const T* __restrict__ W, int64_t ldw, int rows,
                                           const T* __restrict__ V, int64_t ldv, int cols,
                                           const T* __restrict__ xj, int64_t n_f, int kt) {
  using TL = Tile<T>;
  const int tid = threadIdx.x;
  const int64_t q_base = (int64_t)kt * TL::BK;
#pragma unroll
  for (int r = 0; r < (kBM * 8) / kNT; ++r) {
    const int c = tid + r * kNT;
    const int row = c >> 3, ch = c & 7;
    const int64_t q0 = q_base + ch * TL::VEC;
    int64_t rem = (n_f - q0) * (int64_t)sizeof(T);
    int bytes = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
    const T* srcA = W;
    if (row < rows && bytes) srcA = W + row * ldw + q0; else bytes = 0;
    cp_async16(st + row * TL::PITCH + ch * TL::VEC, srcA, bytes);
  }
#pragma unroll
  for (int r = 0; r < (kBN * 8) / kNT; ++r) {
    const int c = tid + r * kNT;
    const int row = c >> 3, ch = c & 7;
    const int64_t q0 = q_base + ch * TL::VEC;
    int64_t rem = (n_f - q0) * (int64_t)sizeof(T);
    int bytes = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
    const T* srcB = V;
    if (row < cols && bytes) srcB = V + row * ldv + q0; else bytes = 0;
    cp_async16(st + (kBM + row) * TL::PITCH + ch * TL::VEC, srcB, bytes);
  }
  if (PIVOT && tid < 8) {
    const int64_t q0 = q_base + tid * TL::VEC;
    int64_t rem = (n_f - q0) * (int64_t)sizeof(T);
    int bytes = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
    cp_async16(st + (kBM + kBN) * TL::PITCH + tid * TL::VEC, bytes ? xj + q0 : xj, bytes);
  }
}

// 3-way prologue on a landed stage: A[r][q] <- min(A[r][q], x_j[q])
// (xj_columns, mingemm.py:225-234). min is exact, so the later sum of
// min(X, V_k) equals sum_q min(min(x_j, v_i), v_k) bit for bit (Appendix C r8).
template <typename T>
__device__ __forceinline__ void stage_pivot_min(T* st) {
  using TL = Tile<T>;
  const T* xs = st + (kBM + kBN) * TL::PITCH;
  const int tid = threadIdx.x;
#pragma unroll
  for (int r = 0; r < (kBM * 8) / kNT; ++r) {
    const int c = tid + r * kNT;
    const int row = c >> 3, ch = c & 7;
    T* p = st + row * TL::PITCH + ch * TL::VEC;
#pragma unroll
    for (int v = 0; v < TL::VEC; ++v) p[v] = Traits<T>::min(xs[ch * TL::VEC + v], p[v]);
  }
}

// Full-depth mainloop for one 128x128 tile. `W` / `V` point at the first
// vector of the tile's rows / columns. All threads of the CTA must call it.
template <typename T, bool PIVOT>
__device__ __forceinline__ void minplus_tile(const T* __restrict__ W, int64_t ldw, int rows,
                                             const T* __restrict__ V, int64_t ldv, int cols,
                                             const T* __restrict__ xj, int64_t n_f,
                                             T (&acc)[kTM][kTN], T* smem) {
  using TL = Tile<T>;
  constexpr int S = TL::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);
  const int tx = (warp & 1) * 8 + (lane & 7);
#pragma unroll
  for (int m = 0; m < kTM; ++m)
#pragma unroll
    for (int n = 0; n < kTN; ++n) acc[m][n] = T(0);

  const int KT = (int)((n_f + TL::BK - 1) / TL::BK);
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < KT) stage_load<T, PIVOT>(smem + s * TL::STAGE_ELEMS, W, ldw, rows, V, ldv, cols, xj, n_f, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<S - 2>();
    __syncthreads();
    T* st = smem + (kt % S) * TL::STAGE_ELEMS;
    if (PIVOT) {
      stage_pivot_min<T>(st);
      __syncthreads();
    }
    const int nk = kt + S - 1;
    if (nk < KT)
      stage_load<T, PIVOT>(smem + (nk % S) * TL::STAGE_ELEMS, W, ldw, rows, V, ldv, cols, xj, n_f, nk);
    cp_async_commit();
    const T* As = st;
    const T* Bs = st + kBM * TL::PITCH;
#pragma unroll
    for (int kk = 0; kk < TL::BK; kk += TL::VEC) Micro<T>::step(acc, As, Bs, ty, tx, kk);
  }
  cp_async_wait<0>();
}

__device__ __forceinline__ int thread_ty() {
  return ((threadIdx.x >> 5) >> 1) * 4 + ((threadIdx.x & 31) >> 3);
}
__device__ __forceinline__ int thread_tx() {
  return ((threadIdx.x >> 5) & 1) * 8 + (threadIdx.x & 7);
}

// Upper-triangular tile enumeration (bi <= bj) of a T x T tile grid, row
// major; the same arithmetic as pair_unindex (core.py:133-148) with the
// diagonal included.
__device__ __forceinline__ void tri_tile(int64_t t, int64_t T_, int& bi, int& bj) {
  // start(b) = b*T - b(b-1)/2 ; find largest b with start(b) <= t
  double b2 = 2.0 * (double)T_ + 1.0;
  int64_t b = (int64_t)((b2 - sqrt(b2 * b2 - 8.0 * (double)t)) * 0.5);
  if (b < 0) b = 0;
  while (b > 0 && b * T_ - (b * (b - 1)) / 2 > t) --b;
  while ((b + 1) * T_ - ((b + 1) * b) / 2 <= t) ++b;
  bi = (int)b;
  bj = (int)(b + (t - (b * T_ - (b * (b - 1)) / 2)));
}

}  // namespace psim
