// FP64 min+add mainloop formulations, measured on operands resident in shared
// memory (experiment, not product; prove or beat the
// FP64 ceiling).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//          -I include -I paper_1705_08210_b200/csrc tools/exp_fp64_mix.cu -o build/exp_fp64_mix
// Run:   build/exp_fp64_mix [iters]   -> one JSON line per variant
// Every variant runs the production thread layout (16 x 16 threads, 8 x 8
// register tile, 144-B pitch tiles, one barrier per 16 fields) and differs
// only in how each acc += min(a, b) is expressed:
//   0 production micro_step (w < v ? w : v: DSETP + FSEL + FSEL + DADD)
//   1 fmin()                            (DSETP.MIN + SEL + FSEL + DADD)
//   2 PTX setp + selp.b64 + add.f64     (what ptxas makes of a 64-bit select)
//   3 PTX setp + selp.b32 lo/hi + add   (two integer selects)
//   4 predicated adds: @p add a; @!p add b      (DSETP + 2 DADD: 3 FP64 ops)
//   5 production, m-major order (x and y of one row pair back to back)
//   6 adds only (acc += a): the DADD pipe alone, per add
//   7 DSETP + selects only, folded into an integer xor (no DADD)
//   8 PTX setp + selp.b32 (lo) + selp.f32 (hi): one SEL + one FSEL
#include <cstdio>
#include <cstdlib>

#include "minplus.cuh"

using namespace psim;
using C = Prod<double>::C;

template <int V>
__device__ __forceinline__ double madd(double acc, double a, double b) {
  if constexpr (V == 0 || V == 5) {
    return __dadd_rn(acc, a < b ? a : b);
  } else if constexpr (V == 1) {
    return __dadd_rn(acc, fmin(a, b));
  } else if constexpr (V == 2) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, %2;\n\tselp.b64 %0, %1, %2, p;\n\t}"
        : "=d"(r) : "d"(a), "d"(b));
    return __dadd_rn(acc, r);
  } else if constexpr (V == 3) {
    double r;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 al, ah, bl, bh, rl, rh;\n\t"
        "setp.lt.f64 p, %1, %2;\n\t"
        "mov.b64 {al, ah}, %1;\n\tmov.b64 {bl, bh}, %2;\n\t"
        "selp.b32 rl, al, bl, p;\n\tselp.b32 rh, ah, bh, p;\n\t"
        "mov.b64 %0, {rl, rh};\n\t}"
        : "=d"(r) : "d"(a), "d"(b));
    return __dadd_rn(acc, r);
  } else if constexpr (V == 8) {
    double r;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 al, bl, rl;\n\t.reg .f32 ah, bh, rh;\n\t"
        "setp.lt.f64 p, %1, %2;\n\t"
        "mov.b64 {al, ah}, %1;\n\tmov.b64 {bl, bh}, %2;\n\t"
        "selp.b32 rl, al, bl, p;\n\tselp.f32 rh, ah, bh, p;\n\t"
        "mov.b64 %0, {rl, rh};\n\t}"
        : "=d"(r) : "d"(a), "d"(b));
    return __dadd_rn(acc, r);
  } else if constexpr (V == 4) {
    double r = acc;
    asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, %2;\n\t"
        "@p add.rn.f64 %0, %0, %1;\n\t@!p add.rn.f64 %0, %0, %2;\n\t}"
        : "+d"(r) : "d"(a), "d"(b));
    return r;
  } else if constexpr (V == 6) {
    return __dadd_rn(acc, a);
  } else {
    const double m = a < b ? a : b;
    return __longlong_as_double(__double_as_longlong(acc) ^ __double_as_longlong(m));
  }
}

template <int V>
__device__ __forceinline__ void step(double (&acc)[C::TM][C::TN], const double* As,
                                     const double* Bs, int ty, int tx, int kk) {
  constexpr int P = C::PITCH;
  double2 a[C::TM];
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
    a[m] = *reinterpret_cast<const double2*>(As + (ty + 16 * m) * P + kk);
  if constexpr (V == 5) {
    double2 b[C::TN];
#pragma unroll
    for (int n = 0; n < C::TN; ++n)
      b[n] = *reinterpret_cast<const double2*>(Bs + (tx + 16 * n) * P + kk);
#pragma unroll
    for (int m = 0; m < C::TM; ++m)
#pragma unroll
      for (int n = 0; n < C::TN; ++n) {
        acc[m][n] = madd<0>(acc[m][n], a[m].x, b[n].x);
        acc[m][n] = madd<0>(acc[m][n], a[m].y, b[n].y);
      }
  } else {
#pragma unroll
    for (int n = 0; n < C::TN; ++n) {
      const double2 b = *reinterpret_cast<const double2*>(Bs + (tx + 16 * n) * P + kk);
#pragma unroll
      for (int m = 0; m < C::TM; ++m) acc[m][n] = madd<V>(acc[m][n], a[m].x, b.x);
#pragma unroll
      for (int m = 0; m < C::TM; ++m) acc[m][n] = madd<V>(acc[m][n], a[m].y, b.y);
    }
  }
}

template <int V>
__global__ void __launch_bounds__(kNT, 1) k_mix(int64_t iters, double seed, double* sink,
                                                long long* cycles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + C::BM * C::PITCH;
  for (int e = threadIdx.x; e < (C::BM + C::BN) * C::PITCH; e += kNT)
    As[e] = seed * double((e * 7919) % 1021);
  double acc[C::TM][C::TN];
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = 0.0;
  const int ty = thread_ty(), tx = thread_tx();
  __syncthreads();
  const long long c0 = clock64();
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int kk = 0; kk < C::BK; kk += C::VEC) step<V>(acc, As, Bs, ty, tx, kk);
    __syncthreads();
  }
  const long long c1 = clock64();
  double s = 0;
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) s += acc[m][n];
  if (s == -1.0) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
}

template <int V>
void run(int64_t iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = (C::BM + C::BN) * C::PITCH * 8;
  cudaFuncSetAttribute(k_mix<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mix<V>, kNT, smem);
  const int blocks = sms * (per_sm > 0 ? per_sm : 1);
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, kNT * 8);
  cudaMalloc(&cyc, blocks * 8);
  k_mix<V><<<blocks, kNT, smem>>>(iters / 10 + 1, 1e-3, sink, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mix<V><<<blocks, kNT, smem>>>(iters, 1e-3, sink, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  long long cmax = 0;
  for (int b = 0; b < blocks; ++b) cmax = h[b] > cmax ? h[b] : cmax;
  const double cmp = (double)blocks * kNT * iters * C::TM * C::TN * C::BK;
  printf("{\"variant\": %d, \"ctas_per_sm\": %d, \"cmp_per_clk_sm\": %.3f, \"cmp_per_s\": %.4e, "
         "\"mhz\": %.0f, \"err\": \"%s\"}\n",
         V, per_sm, cmp / sms / (double)cmax, cmp / (ms * 1e-3), (double)cmax / (ms * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  delete[] h;
  cudaFree(sink);
  cudaFree(cyc);
}

int main(int argc, char** argv) {
  const int64_t iters = argc > 1 ? atoll(argv[1]) : 20000;
  run<0>(iters);
  run<1>(iters);
  run<2>(iters);
  run<3>(iters);
  run<4>(iters);
  run<5>(iters);
  run<6>(iters);
  run<7>(iters);
  run<8>(iters);
  return 0;
}
