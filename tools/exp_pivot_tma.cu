// 3-way single-pivot tile with TMA staging: where does it lose against the 2-way
// TMA mainloop? Experiment, not product. Every variant computes, per 128 x 128
// tile (bi, bj) with its own pivot p(bi, bj),
//   acc[i][k] = sum_q min(min(x_p[q], w_i[q]), w_k[q])
// and the outputs are compared bit for bit with variant "prod".
//   tma2      minplus_tile_tma, no pivot (the 2-way ceiling; outputs differ)
//   prod      minplus_tile_pivot_tma (production: every thread transforms its
//             share of the stage D ahead, published on per-stage "ready" mbarriers)
//   warp_own  each warp rewrites exactly the A rows it reads (its warp-pair
//             partner writes the same values: min is idempotent), one stage ahead;
//             no cross-warp synchronisation beyond full / empty
//   ws        warp-specialised: 256 math threads + one producer warp that issues
//             the TMA boxes and applies the pivot min to the whole A stage
//             (9 warps: the per-SMSP register file caps every thread at 168 regs)
//   ws_wg     warp-specialised with a producer warpgroup (384 threads):
//             setmaxnreg gives the producers 40 registers and the math warps 232;
//             each producer warp transforms 32 rows, warp 8 issues the boxes
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xptxas -v \
//          -I include -I paper_1705_08210_b200/csrc tools/exp_pivot_tma.cu -o build/exp_pivot_tma
// Run:   build/exp_pivot_tma [n] [n_f]  -> one JSON line per variant
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "minplus.cuh"
#include "psim_tma.h"

using namespace psim;
using C = Prod<double>::C;
using T = double;

__device__ __forceinline__ int64_t pivot_of(int64_t bi, int64_t bj, int64_t n) {
  return (bi * 131 + bj * 17) % n;
}

template <class Cc>
__device__ __forceinline__ void store_tile(double (&acc)[Cc::TM][Cc::TN], double* out, int64_t n,
                                           int64_t row0, int64_t col0) {
  const int ty = thread_ty(), tx = thread_tx();
#pragma unroll
  for (int m = 0; m < Cc::TM; ++m)
#pragma unroll
    for (int q = 0; q < Cc::TN; ++q) {
      const int64_t i = row0 + ty + 16 * m, j = col0 + tx + 16 * q;
      if (i < n && j < n) out[i + j * n] = acc[m][q];
    }
}

// ---- warp_own: each warp transforms the 32 A rows it reads
__device__ __forceinline__ void warp_rows_min(double* st, const double* xs) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ch = lane & 7;
  const double2 x = *reinterpret_cast<const double2*>(xs + ch * C::VEC);
  double2 a[C::TM];
#pragma unroll
  for (int m = 0; m < C::TM; ++m) {
    const int row = (w >> 1) * 4 + (lane >> 3) + 16 * m;
    a[m] = *reinterpret_cast<const double2*>(st + row * C::PITCH + ch * C::VEC);
  }
#pragma unroll
  for (int m = 0; m < C::TM; ++m) {
    const int row = (w >> 1) * 4 + (lane >> 3) + 16 * m;
    double2 v;
    v.x = Traits<double>::min(x.x, a[m].x);
    v.y = Traits<double>::min(x.y, a[m].y);
    *reinterpret_cast<double2*>(st + row * C::PITCH + ch * C::VEC) = v;
  }
}

__device__ __forceinline__ void tile_warp_own(const void* mapA, int a_row0, const void* mapC,
                                              int c_row0, const void* mapB, int p_row, int64_t n_f,
                                              double (&acc)[C::TM][C::TN], double* smem) {
  constexpr int S = C::STAGES;
  constexpr int XS = (C::BM + C::BN) * C::PITCH;
  constexpr unsigned kBytes = (C::BM + C::BN + 1) * C::PITCH * sizeof(T);
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31;
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
    for (int n = 0; n < C::TN; ++n) acc[m][n] = 0.0;
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
  auto transform = [&](int kt) {
    const int s = kt % S;
    mbar_wait(&full[s], (unsigned)(kt / S) & 1u);
    T* st = smem + s * C::STAGE_ELEMS;
    warp_rows_min(st, st + XS);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
  };
  if (tid == 0)
    for (int kt = 0; kt < S && kt < KT; ++kt) issue(kt);
  if (KT > 0) transform(0);
  const int ty = thread_ty(), tx = thread_tx();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % S;
    const unsigned ph = (unsigned)(kt / S) & 1u;
    if (kt + 1 < KT) transform(kt + 1);
    const T* st = smem + s * C::STAGE_ELEMS;
#pragma unroll 1
    for (int kk = 0; kk < C::BK; kk += C::VEC)
      micro_step<C>(acc, st, st + C::BM * C::PITCH, ty, tx, kk);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && kt + S < KT) {
      mbar_wait(&empty[s], ph);
      issue(kt + S);
    }
  }
}

// ---- ws: warp-specialised producer (warp 8) + 8 math warps
constexpr int kNTW = kNT + 32;

__device__ __forceinline__ bool tile_ws(const void* mapA, int a_row0, const void* mapC, int c_row0,
                                        const void* mapB, int p_row, int64_t n_f,
                                        double (&acc)[C::TM][C::TN], double* smem) {
  constexpr int S = C::STAGES;
  constexpr int XS = (C::BM + C::BN) * C::PITCH;
  constexpr unsigned kBytes = (C::BM + C::BN + 1) * C::PITCH * sizeof(T);
  __shared__ __align__(8) uint64_t full[S], ready[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 1);
      mbar_init(&empty[s], kNT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int KT = (int)((n_f + C::BK - 1) / C::BK);
  if (tid >= kNT) {  // producer warp
    auto issue = [&](int kt) {
      const int s = kt % S;
      T* st = smem + s * C::STAGE_ELEMS;
      mbar_expect_tx(&full[s], kBytes);
      tma_box(st, mapA, kt * C::BK, a_row0, &full[s]);
      tma_box(st + C::BM * C::PITCH, mapC, kt * C::BK, c_row0, &full[s]);
      tma_box(st + XS, mapB, kt * C::BK, p_row, &full[s]);
    };
    if (lane == 0)
      for (int kt = 0; kt < S && kt < KT; ++kt) issue(kt);
    const int ch = lane & 7;
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % S;
      mbar_wait(&full[s], (unsigned)(kt / S) & 1u);
      T* st = smem + s * C::STAGE_ELEMS;
      const double2 x = *reinterpret_cast<const double2*>(st + XS + ch * C::VEC);
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // 4 x 8 chunks per lane (128 rows x 8 chunks / 32 lanes)
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int row = (lane >> 3) + 4 * (r + 8 * h);
          a[r] = *reinterpret_cast<const double2*>(st + row * C::PITCH + ch * C::VEC);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int row = (lane >> 3) + 4 * (r + 8 * h);
          double2 v;
          v.x = Traits<double>::min(x.x, a[r].x);
          v.y = Traits<double>::min(x.y, a[r].y);
          *reinterpret_cast<double2*>(st + row * C::PITCH + ch * C::VEC) = v;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&ready[s]);
        // slot of stage kt - 1 -> stage kt - 1 + S once the math warps are done with it
        const int kp = kt - 1;
        if (kp >= 0 && kp + S < KT) {
          mbar_wait(&empty[kp % S], (unsigned)(kp / S) & 1u);
          issue(kp + S);
        }
      }
      __syncwarp();
    }
    return false;
  }
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = 0.0;
  const int ty = thread_ty(), tx = thread_tx();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % S;
    mbar_wait(&ready[s], (unsigned)(kt / S) & 1u);
    const T* st = smem + s * C::STAGE_ELEMS;
#pragma unroll 1
    for (int kk = 0; kk < C::BK; kk += C::VEC)
      micro_step<C>(acc, st, st + C::BM * C::PITCH, ty, tx, kk);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  return true;
}

// ---- ws_wg: producer warpgroup (warps 8-11) + 8 math warps, setmaxnreg
constexpr int kNTG = kNT + 128;

__device__ __forceinline__ bool tile_ws_wg(const void* mapA, int a_row0, const void* mapC,
                                           int c_row0, const void* mapB, int p_row, int64_t n_f,
                                           double (&acc)[C::TM][C::TN], double* smem) {
  constexpr int S = C::STAGES;
  constexpr int XS = (C::BM + C::BN) * C::PITCH;
  constexpr unsigned kBytes = (C::BM + C::BN + 1) * C::PITCH * sizeof(T);
  __shared__ __align__(8) uint64_t full[S], ready[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 4);
      mbar_init(&empty[s], kNT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int KT = (int)((n_f + C::BK - 1) / C::BK);
  if (tid >= kNT) {  // producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    const int pw = (tid - kNT) >> 5;  // 0..3
    auto issue = [&](int kt) {
      const int s = kt % S;
      T* st = smem + s * C::STAGE_ELEMS;
      mbar_expect_tx(&full[s], kBytes);
      tma_box(st, mapA, kt * C::BK, a_row0, &full[s]);
      tma_box(st + C::BM * C::PITCH, mapC, kt * C::BK, c_row0, &full[s]);
      tma_box(st + XS, mapB, kt * C::BK, p_row, &full[s]);
    };
    if (pw == 0 && lane == 0)
      for (int kt = 0; kt < S && kt < KT; ++kt) issue(kt);
    const int ch = lane & 7;
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % S;
      mbar_wait(&full[s], (unsigned)(kt / S) & 1u);
      T* st = smem + s * C::STAGE_ELEMS;
      const double2 x = *reinterpret_cast<const double2*>(st + XS + ch * C::VEC);
      double2 a[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int row = (lane >> 3) + 4 * (r + 8 * pw);
        a[r] = *reinterpret_cast<const double2*>(st + row * C::PITCH + ch * C::VEC);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int row = (lane >> 3) + 4 * (r + 8 * pw);
        double2 v;
        v.x = Traits<double>::min(x.x, a[r].x);
        v.y = Traits<double>::min(x.y, a[r].y);
        *reinterpret_cast<double2*>(st + row * C::PITCH + ch * C::VEC) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
      if (pw == 0 && lane == 0) {
        const int kp = kt - 1;
        if (kp >= 0 && kp + S < KT) {
          mbar_wait(&empty[kp % S], (unsigned)(kp / S) & 1u);
          issue(kp + S);
        }
      }
      __syncwarp();
    }
    return false;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int n = 0; n < C::TN; ++n) acc[m][n] = 0.0;
  const int ty = thread_ty(), tx = thread_tx();
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % S;
    mbar_wait(&ready[s], (unsigned)(kt / S) & 1u);
    const T* st = smem + s * C::STAGE_ELEMS;
#pragma unroll 1
    for (int kk = 0; kk < C::BK; kk += C::VEC)
      micro_step<C>(acc, st, st + C::BM * C::PITCH, ty, tx, kk);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  return true;
}

struct Maps {
  CUtensorMap a, p;  // rows / cols (same matrix, box 128 vectors) and pivot (box 1)
};

template <int V>
__global__ void __launch_bounds__(V == 3 ? kNTW : V == 4 ? kNTG : kNT, 1)
    k_var(const __grid_constant__ Maps mp, int64_t n, int64_t n_f, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const int64_t tiles_n = (n + C::BN - 1) / C::BN;
  const int64_t bi = blockIdx.x / tiles_n, bj = blockIdx.x % tiles_n;
  const int64_t row0 = bi * C::BM, col0 = bj * C::BN;
  const int p = (int)pivot_of(bi, bj, n);
  double acc[C::TM][C::TN];
  if (V == 0) {
    minplus_tile_tma<C>(&mp.a, (int)row0, &mp.a, (int)col0, n_f, acc, smem);
  } else if (V == 1) {
    minplus_tile_pivot_tma<C>(&mp.a, (int)row0, &mp.a, (int)col0, &mp.p, p, n_f, acc, smem);
  } else if (V == 2) {
    tile_warp_own(&mp.a, (int)row0, &mp.a, (int)col0, &mp.p, p, n_f, acc, smem);
  } else if (V == 4) {
    if (!tile_ws_wg(&mp.a, (int)row0, &mp.a, (int)col0, &mp.p, p, n_f, acc, smem)) return;
  } else {
    if (!tile_ws(&mp.a, (int)row0, &mp.a, (int)col0, &mp.p, p, n_f, acc, smem)) return;
  }
  store_tile<C>(acc, out, n, row0, col0);
}

__global__ void k_fill(double* p, int64_t cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x)
    p[e] = (double)(mix64((uint64_t)e) & 0xFFFFF);
}

template <typename F>
float timed(F&& launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8192;
  const int64_t n_f = argc > 2 ? atoll(argv[2]) : 10000;
  const int64_t ld = (n_f + 31) / 32 * 32;
  double *W, *o1, *o2;
  cudaMalloc(&W, sizeof(double) * ld * n);
  cudaMalloc(&o1, sizeof(double) * n * n);
  cudaMalloc(&o2, sizeof(double) * n * n);
  cudaMemset(W, 0, sizeof(double) * ld * n);
  k_fill<<<1184, 256>>>(W, ld * n);
  Maps mp;
  if (!encode_operand<double>(&mp.a, W, n_f, n, ld, C::BM, C::PITCH) ||
      !encode_operand<double>(&mp.p, W, n_f, n, ld, 1, C::PITCH)) {
    printf("{\"error\": \"tensor map encode failed\"}\n");
    return 1;
  }
  const int smem = C::SMEM_BYTES;
  cudaFuncSetAttribute(k_var<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_var<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_var<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_var<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_var<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int64_t tiles = ((n + 127) / 128) * ((n + 127) / 128);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double useful = (double)n * n * n_f;
  std::vector<double> h1(n * n), h2(n * n);
  const char* names[5] = {"tma2", "prod", "warp_own", "ws", "ws_wg"};
  const void* fns[5] = {(const void*)k_var<0>, (const void*)k_var<1>, (const void*)k_var<2>,
                        (const void*)k_var<3>, (const void*)k_var<4>};
  auto run = [&](int v, double* o) {
    switch (v) {
      case 0: k_var<0><<<(unsigned)tiles, kNT, smem>>>(mp, n, n_f, o); break;
      case 1: k_var<1><<<(unsigned)tiles, kNT, smem>>>(mp, n, n_f, o); break;
      case 2: k_var<2><<<(unsigned)tiles, kNT, smem>>>(mp, n, n_f, o); break;
      case 3: k_var<3><<<(unsigned)tiles, kNTW, smem>>>(mp, n, n_f, o); break;
      default: k_var<4><<<(unsigned)tiles, kNTG, smem>>>(mp, n, n_f, o); break;
    }
  };
  run(1, o1);
  cudaDeviceSynchronize();
  cudaMemcpy(h1.data(), o1, 8 * n * n, cudaMemcpyDeviceToHost);
  for (int round = 0; round < 2; ++round)
    for (int v = 0; v < 5; ++v) {
      cudaMemset(o2, 0xff, 8 * n * n);
      const float ms = timed([&] { run(v, o2); }, 3);
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, fns[v]);
      cudaMemcpy(h2.data(), o2, 8 * n * n, cudaMemcpyDeviceToHost);
      const bool same = std::memcmp(h1.data(), h2.data(), 8 * n * n) == 0;
      printf("{\"variant\": \"%s\", \"n\": %lld, \"n_f\": %lld, \"ms\": %.3f, "
             "\"cmp_per_clk_sm_1965\": %.3f, \"regs\": %d, \"bitwise_equal_prod\": %s, "
             "\"err\": \"%s\"}\n",
             names[v], (long long)n, (long long)n_f, ms, useful / (ms * 1e-3) / sms / 1.965e9,
             fa.numRegs, same ? "true" : "false", cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  return 0;
}
