// Tile-configuration sweep for the min-plus mainloop (experiment, not product).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I include -I paper_1705_08210_b200/csrc tools/exp_minplus.cu -o build/exp_minplus
// Run:   build/exp_minplus [n_v] [n_f]
// Times a raw rectangular n_v x n_v min-plus (numerators written out) per
// configuration and prints cmp/s and cmp/clk/SM (clock from cudaDeviceProp
// is not used: SM clock is read with clock64 inside CTA 0).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "minplus.cuh"

using namespace psim;

template <class C>
__global__ void __launch_bounds__(kNT, C::MINB)
    k_exp(const typename C::T* W, int64_t ld, int64_t n, int64_t n_f, typename C::T* out,
          long long* clk) {
  using T = typename C::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const int64_t tiles_n = (n + C::BN - 1) / C::BN;
  const int64_t bi = blockIdx.x / tiles_n, bj = blockIdx.x % tiles_n;
  const int64_t row0 = bi * C::BM, col0 = bj * C::BN;
  const int rows = (int)min64(C::BM, n - row0), cols = (int)min64(C::BN, n - col0);
  long long c0 = clock64();
  T acc[C::TM][C::TN];
  minplus_tile<C, false>(W + row0 * ld, ld, rows, W + col0 * ld, ld, cols, nullptr, n_f, acc,
                         smem);
  T s = 0;
#pragma unroll
  for (int m = 0; m < C::TM; ++m)
#pragma unroll
    for (int k = 0; k < C::TN; ++k) s += acc[m][k];
  out[blockIdx.x * kNT + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) clk[0] = clock64() - c0;
}

template <typename T>
__global__ void k_fill(T* p, int64_t cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x)
    p[e] = (T)(mix64((uint64_t)e) & 0xFFFFF);
}

template <class C>
void run(const char* name, int64_t n, int64_t n_f) {
  using T = typename C::T;
  int64_t ld = (n_f + 31) / 32 * 32;
  T *W, *out;
  long long* clk;
  cudaMalloc(&W, sizeof(T) * ld * n);
  k_fill<T><<<1184, 256>>>(W, ld * n);
  const int64_t tiles = ((n + C::BM - 1) / C::BM) * ((n + C::BN - 1) / C::BN);
  cudaMalloc(&out, sizeof(T) * tiles * kNT);
  cudaMalloc(&clk, sizeof(long long));
  cudaFuncSetAttribute(k_exp<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_exp<C><<<(unsigned)tiles, kNT, C::SMEM_BYTES>>>(W, ld, n, n_f, out, clk);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) k_exp<C><<<(unsigned)tiles, kNT, C::SMEM_BYTES>>>(W, ld, n, n_f, out, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  cudaError_t err = cudaGetLastError();
  int dev, sms, occ = 0, clock_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_exp<C>, kNT, C::SMEM_BYTES);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_exp<C>);
  const double cmp = (double)tiles * C::BM * C::BN * (double)n_f;  // padded tiles
  const double useful = (double)n * n * n_f;
  printf("{\"cfg\": \"%s\", \"TM\": %d, \"TN\": %d, \"stages\": %d, \"minb\": %d, \"regs\": %d, "
         "\"occ\": %d, \"ms\": %.3f, \"cmp_per_s\": %.4e, \"cmp_per_clk_sm_1965\": %.2f, "
         "\"err\": \"%s\"}\n",
         name, C::TM, C::TN, C::STAGES, C::MINB, fa.numRegs, occ, ms, useful / (ms * 1e-3),
         useful / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(err));
  (void)cmp;
  cudaFree(W);
  cudaFree(out);
  cudaFree(clk);
}

int main(int argc, char** argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 8192;
  int64_t nf = argc > 2 ? atoll(argv[2]) : 20000;
  char name[64];
  snprintf(name, sizeof name, "f64_8x8_s4_u%d", PSIM_KK_UNROLL);
  run<Cfg<double, 8, 8, 4, 1, 0>>(name, n, nf);
  snprintf(name, sizeof name, "f32_8x4_s3_b2_v1_u%d", PSIM_KK_UNROLL);
  run<Cfg<float, 8, 4, 3, 2, 1>>(name, n, (nf * 5) / 2);
  return 0;
}
