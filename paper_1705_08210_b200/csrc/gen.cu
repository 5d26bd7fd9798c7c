// Element-wise device kernels around the min-plus core: synthetic input
// generators, input validation, column sums and the ordered field fold.
//
//   gen_random_exact  SyntheticSpec.local_block, kind random-exact  verify.py:126-147
//   gen_analytic      SyntheticSpec.local_block, kind analytic      verify.py:126-147
//   gen_uniform       general-FP inputs: (mix64(seed ^ (q*n_v+i)) >> 11) * 2^-53
//   check_block       VectorBlock.__post_init__ finite / >= 0       core.py:231-242
//   column_sums       _colsum_kernel, ascending q from +0            mingemm.py:120-127
//   fold_add          reduce_field_axis ascending-p_f fold step      engine.py:197-216
#include "psim_common.cuh"
#include "psim_internal.h"

namespace psim {

static inline unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 64) b = 148 * 64;
  return (unsigned)(b < 1 ? 1 : b);
}

template <typename T, int KIND>
__global__ void k_gen(uint64_t seed, uint64_t mask, int64_t n_v_total, int64_t f0, int64_t v0,
                      int64_t n_fp, int64_t n_vp, T* __restrict__ out, int64_t ld) {
  const int64_t total = n_fp * n_vp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lv = e / n_fp, lq = e - lv * n_fp;
    const uint64_t q = (uint64_t)(f0 + lq), i = (uint64_t)(v0 + lv);
    T val;
    if (KIND == 0) {  // random-exact: integers in [0, 2^bits)
      val = (T)(mix64((q * (uint64_t)n_v_total + i) ^ seed) & mask);
    } else if (KIND == 1) {  // analytic: 1 + [q mod n_v == i]
      val = (T)(1 + ((q % (uint64_t)n_v_total) == i ? 1 : 0));
    } else {  // uniform [0, 1) with the run dtype's mantissa
      const uint64_t h = mix64((q * (uint64_t)n_v_total + i) ^ seed);
      if (sizeof(T) == 8)
        val = (T)((double)(h >> 11) * 0x1.0p-53);
      else
        val = (T)((float)(uint32_t)(h >> 40) * 0x1.0p-24f);
    }
    out[lv * ld + lq] = val;
  }
}

template <typename T, int KIND>
static cudaError_t gen_t(uint64_t seed, uint64_t mask, int64_t n_v_total, int64_t f0, int64_t v0,
                         int64_t n_fp, int64_t n_vp, void* out, int64_t ld, cudaStream_t st) {
  if (n_fp <= 0 || n_vp <= 0) return cudaSuccess;
  note_launch();
  k_gen<T, KIND><<<grid_for(n_fp * n_vp, 256), 256, 0, st>>>(seed, mask, n_v_total, f0, v0, n_fp,
                                                             n_vp, static_cast<T*>(out), ld);
  return cudaGetLastError();
}

cudaError_t gen_random_exact(int dtype, uint64_t seed, int bits, int64_t n_v_total, int64_t f0,
                             int64_t v0, int64_t n_fp, int64_t n_vp, void* out, int64_t ld,
                             cudaStream_t st) {
  const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
  return dtype == kF64
             ? gen_t<double, 0>(seed, mask, n_v_total, f0, v0, n_fp, n_vp, out, ld, st)
             : gen_t<float, 0>(seed, mask, n_v_total, f0, v0, n_fp, n_vp, out, ld, st);
}

cudaError_t gen_analytic(int dtype, int64_t n_v_total, int64_t f0, int64_t v0, int64_t n_fp,
                         int64_t n_vp, void* out, int64_t ld, cudaStream_t st) {
  return dtype == kF64 ? gen_t<double, 1>(0, 0, n_v_total, f0, v0, n_fp, n_vp, out, ld, st)
                       : gen_t<float, 1>(0, 0, n_v_total, f0, v0, n_fp, n_vp, out, ld, st);
}

cudaError_t gen_uniform(int dtype, uint64_t seed, int64_t n_v_total, int64_t f0, int64_t v0,
                        int64_t n_fp, int64_t n_vp, void* out, int64_t ld, cudaStream_t st) {
  return dtype == kF64 ? gen_t<double, 2>(seed, 0, n_v_total, f0, v0, n_fp, n_vp, out, ld, st)
                       : gen_t<float, 2>(seed, 0, n_v_total, f0, v0, n_fp, n_vp, out, ld, st);
}

// flags[0] += non-finite count, flags[1] += negative count.
template <typename T>
__global__ void k_check(const T* __restrict__ V, int64_t n_fp, int64_t n_vp, int64_t ld,
                        unsigned long long* flags) {
  unsigned long long bad = 0, neg = 0;
  const int64_t total = n_fp * n_vp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lv = e / n_fp, lq = e - lv * n_fp;
    const T x = V[lv * ld + lq];
    bad += isfinite(x) ? 0 : 1;
    neg += (x < T(0)) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bad += __shfl_down_sync(0xffffffffu, bad, o);
    neg += __shfl_down_sync(0xffffffffu, neg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(flags, bad);
    if (neg) atomicAdd(flags + 1, neg);
  }
}

cudaError_t check_block(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                        unsigned long long* flags, cudaStream_t st) {
  if (n_fp <= 0 || n_vp <= 0) return cudaSuccess;
  const unsigned g = grid_for(n_fp * n_vp, 256);
  if (dtype == kF64) {
    note_launch();
    k_check<double><<<g, 256, 0, st>>>(static_cast<const double*>(V), n_fp, n_vp, ld, flags);
  } else {
    note_launch();
    k_check<float><<<g, 256, 0, st>>>(static_cast<const float*>(V), n_fp, n_vp, ld, flags);
  }
  return cudaGetLastError();
}

// Column sums, each a sequential ascending-q fold from +0 (bit-identical to
// the min-plus diagonal M[i, i], test_mingemm.py:75-78). A CTA stages a
// 32-vector x 32-field tile through shared memory with coalesced loads; one
// thread per vector then folds its 32 values in order.
template <typename T>
__global__ void __launch_bounds__(256) k_colsum(const T* __restrict__ V, int64_t n_fp,
                                                int64_t n_vp, int64_t ld, T* __restrict__ out) {
  __shared__ T tile[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v_base = (int64_t)blockIdx.x * 32;
  T acc = T(0);
  for (int64_t q0 = 0; q0 < n_fp; q0 += 32) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int lv = warp + 8 * r;
      const int64_t v = v_base + lv, q = q0 + lane;
      tile[lv][lane] = (v < n_vp && q < n_fp) ? V[v * ld + q] : T(0);
    }
    __syncthreads();
    if (warp == 0) {
      const int cnt = (int)min64(32, n_fp - q0);
      for (int t = 0; t < cnt; ++t) acc = Traits<T>::add(acc, tile[lane][t]);
    }
    __syncthreads();
  }
  if (warp == 0 && v_base + lane < n_vp) out[v_base + lane] = acc;
}

cudaError_t column_sums(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                        void* out, cudaStream_t st) {
  if (n_vp <= 0) return cudaSuccess;
  const unsigned g = (unsigned)((n_vp + 31) / 32);
  if (dtype == kF64) {
    note_launch();
    k_colsum<double><<<g, 256, 0, st>>>(static_cast<const double*>(V), n_fp, n_vp, ld,
                                        static_cast<double*>(out));
  } else {
    note_launch();
    k_colsum<float><<<g, 256, 0, st>>>(static_cast<const float*>(V), n_fp, n_vp, ld,
                                       static_cast<float*>(out));
  }
  return cudaGetLastError();
}

template <typename T>
__global__ void k_fold(T* __restrict__ dst, const T* __restrict__ src, int64_t count) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = Traits<T>::add(dst[e], src[e]);
}

cudaError_t fold_add(int dtype, void* dst, const void* src, int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const unsigned g = grid_for(count, 256);
  if (dtype == kF64) {
    note_launch();
    k_fold<double><<<g, 256, 0, st>>>(static_cast<double*>(dst), static_cast<const double*>(src),
                                      count);
  } else {
    note_launch();
    k_fold<float><<<g, 256, 0, st>>>(static_cast<float*>(dst), static_cast<const float*>(src),
                                     count);
  }
  return cudaGetLastError();
}

// xj_columns (mingemm.py:225-234): out[:, k] = np.minimum(v_j, V[:, k]),
// numpy's rule (x < y || x is NaN) ? x : y, so signed zeros and NaNs match.
template <typename T>
__global__ void k_min_columns(const T* __restrict__ V, int64_t n_fp, int64_t n_vp, int64_t ld,
                              const T* __restrict__ vj, T* __restrict__ out, int64_t ldo) {
  const int64_t total = n_fp * n_vp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / n_fp, q = e - k * n_fp;
    const T x = vj[q], y = V[k * ld + q];
    out[k * ldo + q] = (x < y || x != x) ? x : y;
  }
}

cudaError_t min_columns(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                        const void* vj, void* out, int64_t ldo, cudaStream_t st) {
  if (n_fp <= 0 || n_vp <= 0) return cudaSuccess;
  const unsigned g = grid_for(n_fp * n_vp, 256);
  if (dtype == kF64) {
    note_launch();
    k_min_columns<double><<<g, 256, 0, st>>>(static_cast<const double*>(V), n_fp, n_vp, ld,
                                             static_cast<const double*>(vj),
                                             static_cast<double*>(out), ldo);
  } else {
    note_launch();
    k_min_columns<float><<<g, 256, 0, st>>>(static_cast<const float*>(V), n_fp, n_vp, ld,
                                            static_cast<const float*>(vj),
                                            static_cast<float*>(out), ldo);
  }
  return cudaGetLastError();
}

// Byte output mode (io.py:122-136): floor(clamp(v, 0, 1) * 255 + 0.5) in
// double, the multiply and add rounded separately (no FMA contraction) so the
// byte equals numpy's. Eight values per thread: one 8-byte store.
__device__ __forceinline__ uint32_t quant1(double v, int& bad) {
  bad |= !isfinite(v);
  const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  return (uint32_t)floor(__dadd_rn(__dmul_rn(c, 255.0), 0.5));
}

template <typename T>
__global__ void k_quantize(const T* __restrict__ vals, int64_t count, uint8_t* __restrict__ out,
                           unsigned long long* __restrict__ flag, int vec) {
  int bad = 0;
  const int64_t groups = count / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += stride) {
    double v[8];
    if (vec && sizeof(T) == 8) {
      const double2* p = reinterpret_cast<const double2*>(vals + g * 8);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 x = __ldcs(p + h);
        v[2 * h] = x.x;
        v[2 * h + 1] = x.y;
      }
    } else if (vec) {
      const float4* p = reinterpret_cast<const float4*>(vals + g * 8);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float4 x = __ldcs(p + h);
        v[4 * h] = x.x; v[4 * h + 1] = x.y; v[4 * h + 2] = x.z; v[4 * h + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int h = 0; h < 8; ++h) v[h] = (double)vals[g * 8 + h];
    }
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      lo |= quant1(v[h], bad) << (8 * h);
      hi |= quant1(v[4 + h], bad) << (8 * h);
    }
    if (vec)
      reinterpret_cast<uint2*>(out)[g] = make_uint2(lo, hi);
    else
      for (int h = 0; h < 8; ++h) out[g * 8 + h] = (uint8_t)(((h < 4 ? lo : hi) >> (8 * (h & 3))) & 255u);
  }
  const int64_t tail = groups * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tail < count && tail < groups * 8 + 8) out[tail] = (uint8_t)quant1((double)vals[tail], bad);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1ull);
}

cudaError_t quantize_bytes(int dtype, const void* vals, int64_t count, void* out, void* flag,
                           cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const unsigned g = grid_for((count + 7) / 8, 256);
  const uintptr_t a = reinterpret_cast<uintptr_t>(vals), b = reinterpret_cast<uintptr_t>(out);
  const int vec = (a % 16 == 0) && (b % 8 == 0);
  auto* f = static_cast<unsigned long long*>(flag);
  if (dtype == kF64) {
    note_launch();
    k_quantize<double><<<g, 256, 0, st>>>(static_cast<const double*>(vals), count,
                                          static_cast<uint8_t*>(out), f, vec);
  } else {
    note_launch();
    k_quantize<float><<<g, 256, 0, st>>>(static_cast<const float*>(vals), count,
                                         static_cast<uint8_t*>(out), f, vec);
  }
  return cudaGetLastError();
}

// checksum (verify.py:86-96) of a value array with canonical indices
// idx[e] (or idx0 + e): grid-stride terms, CTA reduction, one 128-bit atomic
// pair per CTA (psim_common.cuh).
template <typename T>
__global__ void __launch_bounds__(256) k_checksum(const T* __restrict__ vals,
                                                  const int64_t* __restrict__ idx, int64_t idx0,
                                                  int64_t count, unsigned long long* acc) {
  Cks c;
  for (int64_t e = blockIdx.x * 256ll + threadIdx.x; e < count; e += (int64_t)gridDim.x * 256)
    c.term((uint64_t)(idx ? idx[e] : idx0 + e), Traits<T>::bits(vals[e]));
  c.deg = 0;
  cks_block_flush<256>(acc, c);
}

cudaError_t checksum(int dtype, const void* vals, const int64_t* idx, int64_t idx0, int64_t count,
                     unsigned long long* acc, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const unsigned g = grid_for(count, 256);
  note_launch();
  if (dtype == kF64)
    k_checksum<double><<<g, 256, 0, st>>>(static_cast<const double*>(vals), idx, idx0, count, acc);
  else
    k_checksum<float><<<g, 256, 0, st>>>(static_cast<const float*>(vals), idx, idx0, count, acc);
  return cudaGetLastError();
}

}  // namespace psim
