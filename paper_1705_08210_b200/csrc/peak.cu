// Min+add issue-rate microbenchmark: the roofline denominator (SURVEY
// Appendix D). Each thread keeps 16 independent accumulators in registers and
// repeats exactly the mainloop's per-comparison instruction mix:
//   variant 0, FP64: acc += fmin(x, y)            DSETP.MIN + SEL + FSEL + DADD
//   variant 0, FP32: (acc0, acc1) += (fminf, fminf) FMNMX x2 + FADD2
//   variant 1, FP32: acc += fminf(x, y)           FMNMX + FADD (scalar)
//   variant 2: as 0 with one CTA-uniform operand (optimistic)
//   variant 3: the production mainloop (micro_step) over shared-memory operands
//   variant 4: the adds alone (DADD / FADD), per add
// The min operands rotate through the accumulators themselves so nothing can
// be hoisted out of the loop. The grid is one full-occupancy wave; the rate is
// reported per second (CUDA events) and per SM clock (clock64 inside each CTA).
#include "minplus.cuh"
#include "psim_internal.h"

namespace psim {

constexpr int kPeakAcc = 16;

// Two banks of accumulators: each half-iteration updates one bank with min
// operands read from the other bank, so both operands are per-thread vector
// registers that change every iteration (nothing can be hoisted) while every
// dependency is >= 16 instructions away (no latency stall) -- the register
// traffic of the real mainloop, whose operands come from LDS.
// VAR 2 makes one operand CTA-uniform (fewer register-file reads): an
// optimistic bound, reported for reference only.
template <typename T>
__device__ __forceinline__ void peak_bank(T (&dst)[kPeakAcc], const T (&src)[kPeakAcc], T y0,
                                          T y1, bool uniform, bool packed) {
#pragma unroll
  for (int k = 0; k < kPeakAcc; k += 2) {
    const T a0 = src[k], a1 = src[k + 1];
    const T b0 = uniform ? y0 : src[(k + 5) % kPeakAcc];
    const T b1 = uniform ? y1 : src[(k + 11) % kPeakAcc];
    if (sizeof(T) == 4 && packed) {
      fadd2(*reinterpret_cast<float*>(&dst[k]), *reinterpret_cast<float*>(&dst[k + 1]),
            fminf((float)a0, (float)b0), fminf((float)a1, (float)b1));
    } else {
      dst[k] = Traits<T>::add(dst[k], Traits<T>::min(a0, b0));
      dst[k + 1] = Traits<T>::add(dst[k + 1], Traits<T>::min(a1, b1));
    }
  }
}

template <typename T, int VAR>
__global__ void __launch_bounds__(256) k_peak(int64_t iters, T seed, T* sink, long long* cycles) {
  T acc[kPeakAcc], bcc[kPeakAcc];
#pragma unroll
  for (int k = 0; k < kPeakAcc; ++k) {
    acc[k] = seed * T(k + threadIdx.x % 7);
    bcc[k] = seed * T(2 * k + 1 + threadIdx.x % 5);
  }
  const T y0 = seed * T(3), y1 = seed * T(5);
  __syncthreads();
  const long long c0 = clock64();
  for (int64_t it = 0; it < iters; ++it) {
    peak_bank<T>(acc, bcc, y0, y1, VAR == 2, VAR != 1);
    peak_bank<T>(bcc, acc, y0, y1, VAR == 2, VAR != 1);
  }
  __syncthreads();
  const long long c1 = clock64();
  T s = T(0);
#pragma unroll
  for (int k = 0; k < kPeakAcc; ++k) s += acc[k] + bcc[k];
  if (s == T(-1)) sink[threadIdx.x] = s;  // never true; keeps the loop live
  if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
}

// Variant 3: the production mainloop itself (micro_step of Prod<T>::C, the
// same 16 x 16 threads, TM x TN register tile, 144-B pitch shared tiles and
// one barrier per 128-byte field chunk) over operands already resident in
// shared memory -- i.e. the kernel minus global->shared staging, tile setup
// and epilogue. Its rate is the ceiling of the mainloop as compiled.
template <typename T>
__global__ void __launch_bounds__(kNT, sizeof(T) == 8 ? 1 : 2)
    k_peak_smem(int64_t iters, T seed, T* sink, long long* cycles) {
  using C = typename Prod<T>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);
  T* Bs = As + C::BM * C::PITCH;
  for (int e = threadIdx.x; e < (C::BM + C::BN) * C::PITCH; e += kNT)
    As[e] = seed * T((e * 7919) % 1021);
  T acc[C::TM][C::TN];
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = T(0);
  const int ty = thread_ty<C::MAP>(), tx = thread_tx<C::MAP>();
  __syncthreads();
  const long long c0 = clock64();
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll C::KKU
    for (int kk = 0; kk < C::BK; kk += C::VEC) micro_step<C>(acc, As, Bs, ty, tx, kk);
    __syncthreads();  // the kernel's one barrier per stage (keeps the LDS in the loop)
  }
  const long long c1 = clock64();
  T s = T(0);
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) s += acc[m][n];
  if (s == T(-1)) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
}

// Variant 4: FP64 / FP32 adds alone (two-bank accumulators, no min): the
// add pipe's own rate, for reading the mix's pipe balance.
template <typename T>
__global__ void __launch_bounds__(256) k_peak_add(int64_t iters, T seed, T* sink,
                                                  long long* cycles) {
  T acc[kPeakAcc], bcc[kPeakAcc];
#pragma unroll
  for (int k = 0; k < kPeakAcc; ++k) {
    acc[k] = seed * T(k + threadIdx.x % 7);
    bcc[k] = seed * T(2 * k + 1 + threadIdx.x % 5);
  }
  __syncthreads();
  const long long c0 = clock64();
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < kPeakAcc; ++k) acc[k] = Traits<T>::add(acc[k], bcc[(k + 5) % kPeakAcc]);
#pragma unroll
    for (int k = 0; k < kPeakAcc; ++k) bcc[k] = Traits<T>::add(bcc[k], acc[(k + 11) % kPeakAcc]);
  }
  __syncthreads();
  const long long c1 = clock64();
  T s = T(0);
#pragma unroll
  for (int k = 0; k < kPeakAcc; ++k) s += acc[k] + bcc[k];
  if (s == T(-1)) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
}

// Launch one timed variant: cmp_per_iter comparisons (or adds) per thread
// per loop iteration.
template <typename K, typename T>
static cudaError_t time_kernel(K kern, int smem, double cmp_per_iter, int64_t iters,
                               double* cmp_per_s, double* cmp_per_clk_sm, cudaStream_t st) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNT, smem);
  if (per_sm < 1) per_sm = 1;
  const int blocks = sms * per_sm;
  T* sink = nullptr;
  long long* cyc = nullptr;
  if ((e = cudaMallocAsync(&sink, kNT * sizeof(T), st)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&cyc, blocks * sizeof(long long), st)) != cudaSuccess) return e;
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  note_launch();
  kern<<<blocks, kNT, smem, st>>>(iters / 10 + 1, T(1e-3), sink, cyc);  // warm-up
  cudaEventRecord(ev0, st);
  note_launch();
  kern<<<blocks, kNT, smem, st>>>(iters, T(1e-3), sink, cyc);
  cudaEventRecord(ev1, st);
  e = cudaEventSynchronize(ev1);
  float ms = 0;
  cudaEventElapsedTime(&ms, ev0, ev1);
  long long* h = new long long[blocks];
  cudaMemcpyAsync(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  long long cmax = 0;
  for (int b = 0; b < blocks; ++b) cmax = h[b] > cmax ? h[b] : cmax;
  delete[] h;
  const double cmps = (double)blocks * kNT * (double)iters * cmp_per_iter;
  *cmp_per_s = cmps / (ms * 1e-3);
  *cmp_per_clk_sm = cmps / (double)sms / (double)cmax;
  cudaFreeAsync(sink, st);
  cudaFreeAsync(cyc, st);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T>
static cudaError_t peak_smem_t(int64_t iters, double* cps, double* cpc, cudaStream_t st) {
  using C = typename Prod<T>::C;
  const int smem = (C::BM + C::BN) * C::PITCH * (int)sizeof(T);
  return time_kernel<decltype(&k_peak_smem<T>), T>(
      k_peak_smem<T>, smem, (double)C::TM * C::TN * C::BK, iters, cps, cpc, st);
}

template <typename T>
static cudaError_t peak_add_t(int64_t iters, double* cps, double* cpc, cudaStream_t st) {
  return time_kernel<decltype(&k_peak_add<T>), T>(k_peak_add<T>, 0, 2.0 * kPeakAcc, iters, cps,
                                                  cpc, st);
}

template <typename T, int VAR>
static cudaError_t peak_t(int64_t iters, double* cmp_per_s, double* cmp_per_clk_sm,
                          cudaStream_t st) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peak<T, VAR>, 256, 0);
  if (per_sm < 1) per_sm = 1;
  const int blocks = sms * per_sm;
  T* sink = nullptr;
  long long* cyc = nullptr;
  cudaError_t e = cudaMallocAsync(&sink, 256 * sizeof(T), st);
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync(&cyc, blocks * sizeof(long long), st);
  if (e != cudaSuccess) return e;
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  note_launch();
  k_peak<T, VAR><<<blocks, 256, 0, st>>>(iters / 10 + 1, T(1e-3), sink, cyc);  // warm-up
  cudaEventRecord(ev0, st);
  note_launch();
  k_peak<T, VAR><<<blocks, 256, 0, st>>>(iters, T(1e-3), sink, cyc);
  cudaEventRecord(ev1, st);
  e = cudaEventSynchronize(ev1);
  float ms = 0;
  cudaEventElapsedTime(&ms, ev0, ev1);
  long long* h = new long long[blocks];
  cudaMemcpyAsync(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  long long cmax = 0;
  for (int b = 0; b < blocks; ++b) cmax = h[b] > cmax ? h[b] : cmax;
  delete[] h;
  const double cmps = (double)blocks * 256.0 * (double)iters * 2 * kPeakAcc;
  *cmp_per_s = cmps / (ms * 1e-3);
  *cmp_per_clk_sm = cmps / (double)sms / (double)cmax;
  cudaFreeAsync(sink, st);
  cudaFreeAsync(cyc, st);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t peak_minplus(int dtype, int variant, int64_t iters, double* cmp_per_s,
                         double* cmp_per_clk_sm, cudaStream_t st) {
  if (variant == 3)
    return dtype == kF64 ? peak_smem_t<double>(iters / 16 + 1, cmp_per_s, cmp_per_clk_sm, st)
                         : peak_smem_t<float>(iters / 16 + 1, cmp_per_s, cmp_per_clk_sm, st);
  if (variant == 4)
    return dtype == kF64 ? peak_add_t<double>(iters, cmp_per_s, cmp_per_clk_sm, st)
                         : peak_add_t<float>(iters, cmp_per_s, cmp_per_clk_sm, st);
  if (dtype == kF64)
    return variant == 2 ? peak_t<double, 2>(iters, cmp_per_s, cmp_per_clk_sm, st)
                        : peak_t<double, 0>(iters, cmp_per_s, cmp_per_clk_sm, st);
  if (variant == 1) return peak_t<float, 1>(iters, cmp_per_s, cmp_per_clk_sm, st);
  if (variant == 2) return peak_t<float, 2>(iters, cmp_per_s, cmp_per_clk_sm, st);
  return peak_t<float, 0>(iters, cmp_per_s, cmp_per_clk_sm, st);
}

}  // namespace psim
