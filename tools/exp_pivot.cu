// 3-way pivot-prologue experiment (not product): mainloop rate of
//   v0  no pivot (the 2-way mainloop)
//   v1  pivot min on the landed stage by the whole CTA + a second barrier (production)
//   v2  each warp rewrites only the A rows it reads (idempotent; warp pairs that
//       share rows both do it), __syncwarp instead of the second CTA barrier
//   v3  product minplus_tile with the in-mainloop column sums (SUMS)
//   v4  product minplus_tile without them
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//          -I include -I paper_1705_08210_b200/csrc tools/exp_pivot.cu -o build/exp_pivot
// Run:   build/exp_pivot [n] [n_f]
#include <cstdio>
#include <cstdlib>

#include "minplus.cuh"

using namespace psim;

// v2: the rows warp w reads are ty + 16 m, ty in {4 (w>>1) .. 4 (w>>1) + 3}.
template <class C>
__device__ __forceinline__ void warp_pivot_min(typename C::T* st, const typename C::T* xs) {
  using T = typename C::T;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ch = lane & 7;
  const double2 x = *reinterpret_cast<const double2*>(xs + ch * C::VEC);
#pragma unroll
  for (int r = 0; r < C::TM; ++r) {
    const int row = (w >> 1) * 4 + (lane >> 3) + 16 * r;
    double2* p = reinterpret_cast<double2*>(st + row * C::PITCH + ch * C::VEC);
    double2 a = *p;
    a.x = Traits<T>::min(x.x, a.x);
    a.y = Traits<T>::min(x.y, a.y);
    *p = a;
  }
}

template <class C, int VARIANT>
__device__ __forceinline__ void tile_v(const double* __restrict__ W, int64_t ldw, int rows,
                                       const double* __restrict__ V, int64_t ldv, int cols,
                                       const double* __restrict__ xj, int64_t n_f,
                                       double (&acc)[C::TM][C::TN], double* smem) {
  constexpr int S = C::STAGES;
  constexpr int XS = (C::BM + C::BN) * C::PITCH;
  constexpr bool PIVOT = VARIANT > 0;
  const int KT = (int)((n_f + C::BK - 1) / C::BK);
  const int ty = thread_ty(), tx = thread_tx();
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = 0.0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < KT) {
      stage_load<C, PIVOT>(smem + s * C::STAGE_ELEMS, W, ldw, rows, V, ldv, cols, xj, n_f, s);
      if (PIVOT) pivot_load<C>(smem + s * C::STAGE_ELEMS, xj, n_f, s);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<S - 2>();
    __syncthreads();
    double* st = smem + (kt % S) * C::STAGE_ELEMS;
    if (VARIANT == 1) {
      stage_pivot_min<C>(st, st + XS);
      __syncthreads();
    } else if (VARIANT == 2) {
      warp_pivot_min<C>(st, st + XS);
      __syncwarp();
    }
    const int nk = kt + S - 1;
    if (nk < KT) {
      stage_load<C, PIVOT>(smem + (nk % S) * C::STAGE_ELEMS, W, ldw, rows, V, ldv, cols, xj,
                           n_f, nk);
      if (PIVOT) pivot_load<C>(smem + (nk % S) * C::STAGE_ELEMS, xj, n_f, nk);
    }
    cp_async_commit();
    const double* As = st;
    const double* Bs = st + C::BM * C::PITCH;
#pragma unroll
    for (int kk = 0; kk < C::BK; kk += C::VEC) micro_step<C>(acc, As, Bs, ty, tx, kk);
  }
  cp_async_wait<0>();
}

template <class C, int VARIANT>
__global__ void __launch_bounds__(kNT, C::MINB)
    k_exp(const double* W, int64_t ld, int64_t n, int64_t n_f, double* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const int64_t tiles_n = (n + C::BN - 1) / C::BN;
  const int64_t bi = blockIdx.x / tiles_n, bj = blockIdx.x % tiles_n;
  const int64_t row0 = bi * C::BM, col0 = bj * C::BN;
  const int rows = (int)min64(C::BM, n - row0), cols = (int)min64(C::BN, n - col0);
  double acc[C::TM][C::TN];
  const double* xj = W + ((bi * 7 + bj) % n) * ld;  // some pivot vector
  double s = 0;
  if (VARIANT == 3) {
    double vs;
    minplus_tile<C, false, true>(W + row0 * ld, ld, rows, W + col0 * ld, ld, cols, nullptr, n_f,
                                 acc, smem, &vs);
    s = vs;
  } else if (VARIANT == 4) {
    minplus_tile<C, false>(W + row0 * ld, ld, rows, W + col0 * ld, ld, cols, nullptr, n_f, acc,
                           smem);
  } else {
    tile_v<C, VARIANT>(W + row0 * ld, ld, rows, W + col0 * ld, ld, cols, xj, n_f, acc, smem);
  }
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int k = 0; k < C::TN; ++k) s += acc[m][k];
  out[blockIdx.x * kNT + threadIdx.x] = s;
}

__global__ void k_fill(double* p, int64_t cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x)
    p[e] = (double)(mix64((uint64_t)e) & 0xFFFFF);
}

template <int VARIANT>
double run(const double* W, int64_t ld, int64_t n, int64_t n_f, double* out) {
  using C = Prod<double>::C;
  const int64_t tiles = ((n + C::BM - 1) / C::BM) * ((n + C::BN - 1) / C::BN);
  cudaFuncSetAttribute(k_exp<C, VARIANT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::SMEM_BYTES);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_exp<C, VARIANT><<<(unsigned)tiles, kNT, C::SMEM_BYTES>>>(W, ld, n, n_f, out);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int r = 0; r < reps; ++r)
    k_exp<C, VARIANT><<<(unsigned)tiles, kNT, C::SMEM_BYTES>>>(W, ld, n, n_f, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double cmp = (double)tiles * C::BM * C::BN * (double)n_f;
  double chk = 0;
  {
    static double h[4096];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    for (double v : h) chk += v;
  }
  printf("{\"variant\": %d, \"ms\": %.3f, \"cmp_per_clk_sm_1965\": %.3f, \"chk\": %.6e, "
         "\"err\": \"%s\"}\n",
         VARIANT, ms, cmp / (ms * 1e-3) / sms / 1.965e9, chk,
         cudaGetErrorString(cudaGetLastError()));
  return chk;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8192;
  const int64_t nf = argc > 2 ? atoll(argv[2]) : 10000;
  const int64_t ld = (nf + 31) / 32 * 32;
  double *W, *out;
  cudaMalloc(&W, sizeof(double) * ld * n);
  k_fill<<<1184, 256>>>(W, ld * n);
  const int64_t tiles = ((n + 127) / 128) * ((n + 127) / 128);
  cudaMalloc(&out, sizeof(double) * tiles * kNT);
  run<0>(W, ld, n, nf, out);
  const double c1 = run<1>(W, ld, n, nf, out);
  const double c2 = run<2>(W, ld, n, nf, out);
  printf("{\"v1_equals_v2\": %s}\n", c1 == c2 ? "true" : "false");
  run<0>(W, ld, n, nf, out);
  run<1>(W, ld, n, nf, out);
  run<2>(W, ld, n, nf, out);
  run<3>(W, ld, n, nf, out);
  run<4>(W, ld, n, nf, out);
  run<3>(W, ld, n, nf, out);
  run<4>(W, ld, n, nf, out);
  return 0;
}
