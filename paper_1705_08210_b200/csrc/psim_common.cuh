// Shared device helpers for libpsim: the 64-bit mix, the 128-bit checksum
// accumulator, canonical tuple indexing and the run-dtype traits.
//
// Every helper restates one piece of the reference's arithmetic so that the
// kernels reproduce its bits:
//   mix64                 verify.py:36-44 (wrapping 64-bit avalanche)
//   term / fold           verify.py:74-76 (mix64(idx) * (mix64(bits) | 1) mod 2^128)
//   value bits            verify.py:58-65 (FP32 zero-extended to 64 bits)
//   pair_index            core.py:122-130
//   triple_index          core.py:151-156
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace psim {

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr uint64_t kMixC1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMixC2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= kMixC1;
  x ^= x >> 27;
  x *= kMixC2;
  x ^= x >> 31;
  return x;
}

// Number of unordered pairs / triples among m items (core.py:114-119).
__host__ __device__ __forceinline__ uint64_t choose2(uint64_t m) {
  return m < 2 ? 0 : (m * (m - 1)) / 2;
}
__host__ __device__ __forceinline__ uint64_t choose3(uint64_t m) {
  // (m(m-1)/2) * (m-2) is divisible by 3; stays < 2^64 for m < 2.6e6.
  return m < 3 ? 0 : (choose2(m) * (m - 2)) / 3;
}

// Lexicographic index of (i, j), i < j < n (core.py:122-130).
__host__ __device__ __forceinline__ uint64_t pair_index(uint64_t i, uint64_t j, uint64_t n) {
  return i * n - (i * (i + 1)) / 2 + (j - i - 1);
}

// Lexicographic index of (i, j, k), i < j < k < n (core.py:151-156).
__host__ __device__ __forceinline__ uint64_t triple_index(uint64_t i, uint64_t j, uint64_t k,
                                                          uint64_t n) {
  return choose3(n) - choose3(n - i) + pair_index(j - i - 1, k - i - 1, n - i - 1);
}

template <typename T>
struct Traits;

template <>
struct Traits<double> {
  static constexpr int kVec = 2;  // elements per 16-byte chunk
  __device__ __forceinline__ static uint64_t bits(double v) {
    return (uint64_t)__double_as_longlong(v);
  }
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
  // `w if w < v else v` (mingemm.py:90): DSETP + 2 FSEL, no NaN fix-up
  // (fmin would add a predicated LOP3 per comparison; inputs are NaN-free).
  __device__ __forceinline__ static double min(double a, double b) { return a < b ? a : b; }
};

template <>
struct Traits<float> {
  static constexpr int kVec = 4;
  __device__ __forceinline__ static uint64_t bits(float v) {
    return (uint64_t)(uint32_t)__float_as_uint(v);
  }
  __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static float div(float a, float b) { return __fdiv_rn(a, b); }
  __device__ __forceinline__ static float min(float a, float b) { return fminf(a, b); }
};

// ---------------------------------------------------------------------------
// 128-bit wrapping checksum (verify.py:68-96) kept as (lo, hi) u64 pairs.

struct Cks {
  uint64_t lo = 0, hi = 0;
  unsigned long long deg = 0;  // degenerate-record count (metrics2.py:200)

  __device__ __forceinline__ void add128(uint64_t l, uint64_t h) {
    uint64_t n = lo + l;
    hi += h + (n < lo ? 1ull : 0ull);
    lo = n;
  }
  __device__ __forceinline__ void term(uint64_t canonical_index, uint64_t value_bits) {
    uint64_t a = mix64(canonical_index);
    uint64_t b = mix64(value_bits) | 1ull;
    add128(a * b, __umul64hi(a, b));
  }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      uint64_t l = __shfl_down_sync(0xffffffffu, lo, o);
      uint64_t h = __shfl_down_sync(0xffffffffu, hi, o);
      unsigned long long d = __shfl_down_sync(0xffffffffu, deg, o);
      add128(l, h);
      deg += d;
    }
  }
};

// acc[0..1] = 128-bit sum (lo, hi), acc[2] = degenerate count.
// Wrapping adds commute, so atomics in any order give the same total; the
// carry out of the low word is detected from the value each atomic saw.
__device__ __forceinline__ void cks_atomic_flush(unsigned long long* acc, const Cks& c) {
  unsigned long long old = atomicAdd(acc, (unsigned long long)c.lo);
  unsigned long long carry = (old + c.lo) < old ? 1ull : 0ull;
  unsigned long long h = c.hi + carry;
  if (h) atomicAdd(acc + 1, h);
  if (c.deg) atomicAdd(acc + 2, c.deg);
}

// Block-wide reduction then one atomic triple per CTA. Must be called by
// every thread of the block (contains __syncthreads).
template <int NT>
__device__ __forceinline__ void cks_block_flush(unsigned long long* acc, Cks c) {
  __shared__ uint64_t s_lo[NT / 32], s_hi[NT / 32];
  __shared__ unsigned long long s_deg[NT / 32];
  c.warp_reduce();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_lo[warp] = c.lo;
    s_hi[warp] = c.hi;
    s_deg[warp] = c.deg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Cks t;
    for (int w = 0; w < NT / 32; ++w) {
      t.add128(s_lo[w], s_hi[w]);
      t.deg += s_deg[w];
    }
    if (t.lo | t.hi | t.deg) cks_atomic_flush(acc, t);
  }
}

// ---------------------------------------------------------------------------
// cp.async helpers (16-byte global->shared copies with zero fill).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Volatile read-only load: never CSE'd or hoisted, so tile decodes repeated
// after a mainloop are recomputed instead of held live in registers.
__device__ __forceinline__ int64_t ld_pref(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

}  // namespace psim
