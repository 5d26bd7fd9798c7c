// Host wake-up latency after a multi-second kernel (experiment, not product).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          tools/exp_sync.cu -o build/exp_sync -Lpaper_1705_08210_b200/_lib -lpsim \
//          -Xlinker -rpath,'$ORIGIN/../paper_1705_08210_b200/_lib'
// Run:   build/exp_sync [reps] [mode: 0 blocking event sync, 1 spin on cudaEventQuery,
//                                    2 cudaDeviceScheduleBlockingSync, 3 cudaDeviceScheduleSpin]
// Times the cfg2 fused 2-way task through the C ABI with no Python or torch in
// the process; prints host wall time minus the GPU event time per rep.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#include "psim.h"

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 8;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  if (mode == 2) cudaSetDeviceFlags(cudaDeviceScheduleBlockingSync);
  if (mode == 3) cudaSetDeviceFlags(cudaDeviceScheduleSpin);
  const int64_t n_f = 20000, n = 40000, ld = 20000;
  double *V, *sums, *vals;
  unsigned long long* acc;
  cudaMalloc(&V, sizeof(double) * ld * n);
  cudaMalloc(&sums, sizeof(double) * n);
  cudaMalloc(&vals, sizeof(double) * (n * (n - 1) / 2));
  cudaMalloc(&acc, 3 * sizeof(unsigned long long));
  psim_gen_random_exact(1, 2026, 20, n, 0, 0, n_f, n, V, ld, nullptr);
  psim_column_sums(1, V, n_f, n, ld, sums, nullptr);
  psim_block2_t t{};
  t.W = V; t.ldw = ld; t.V = V; t.ldv = ld; t.n_f = n_f; t.m = n; t.n = n; t.diagonal = 1;
  t.s_row = sums; t.s_col = sums; t.n_v = n; t.vals = vals; t.acc = acc;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < reps; ++r) {
    auto h0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0, nullptr);
    int st = psim_czek2_block(1, &t, nullptr);
    cudaEventRecord(e1, nullptr);
    if (mode == 1) {
      while (cudaEventQuery(e1) == cudaErrorNotReady) {
      }
    } else {
      cudaEventSynchronize(e1);
    }
    auto h1 = std::chrono::steady_clock::now();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double host_ms = std::chrono::duration<double, std::milli>(h1 - h0).count();
    printf("{\"mode\": %d, \"rep\": %d, \"status\": %d, \"gpu_ms\": %.3f, \"host_ms\": %.3f, "
           "\"late_ms\": %.3f}\n", mode, r, st, ms, host_ms, host_ms - ms);
    fflush(stdout);
  }
  return 0;
}
