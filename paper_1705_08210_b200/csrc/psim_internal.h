// Internal (C++) launch interface between the C-ABI layer (capi.cu) and the
// kernel translation units. Not part of the public ABI; see include/psim.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "psim.h"

namespace psim {

// Process-wide count of kernel launches issued by libpsim (psim_launch_count):
// every launch site calls note_launch() right before it launches.
void note_launch(int n = 1);

constexpr int kF32 = 0;
constexpr int kF64 = 1;

// CTA output tile (rows x cols) of the production min-plus kernels per dtype
// (defined from the tile configurations in minplus.cuh).
void tile_shape(int dtype, int* bm, int* bn);

// The public task descriptors double as the internal ones.
using Czek2Block = psim_block2_t;
using Czek3Box = psim_box3_t;

cudaError_t gen_random_exact(int dtype, uint64_t seed, int bits, int64_t n_v_total, int64_t f0,
                             int64_t v0, int64_t n_fp, int64_t n_vp, void* out, int64_t ld,
                             cudaStream_t st);
cudaError_t gen_analytic(int dtype, int64_t n_v_total, int64_t f0, int64_t v0, int64_t n_fp,
                         int64_t n_vp, void* out, int64_t ld, cudaStream_t st);
cudaError_t gen_uniform(int dtype, uint64_t seed, int64_t n_v_total, int64_t f0, int64_t v0,
                        int64_t n_fp, int64_t n_vp, void* out, int64_t ld, cudaStream_t st);
cudaError_t check_block(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                        unsigned long long* flags, cudaStream_t st);
cudaError_t column_sums(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                        void* out, cudaStream_t st);
cudaError_t fold_add(int dtype, void* dst, const void* src, int64_t count, cudaStream_t st);
cudaError_t quantize_bytes(int dtype, const void* vals, int64_t count, void* out, void* flag,
                           cudaStream_t st);

cudaError_t czek2_block(int dtype, const Czek2Block& t, cudaStream_t st);
cudaError_t czek2_streamed(int dtype, const Czek2Block& t, const void* host, int64_t host_ld,
                           int64_t chunk, unsigned* ready, cudaStream_t compute,
                           cudaStream_t copy);
cudaError_t stream_stats(unsigned long long* out4, int reset);
cudaError_t stream_error(unsigned* aborted, int reset);
constexpr int64_t kStreamMaxFlags = 65536;  // data + sum flags of a streamed run
// Sorenson (0/1) path: bit packing and the AND+POPC 2-way task (sorenson.cu).
cudaError_t pack_bits(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                      uint32_t* words, int64_t ldw, unsigned long long* flags, cudaStream_t st);
cudaError_t sorenson2_block(int dtype, const psim_block2_t& t, cudaStream_t st);
cudaError_t mgemm_bits(const uint32_t* W, int64_t ldw, const uint32_t* V, int64_t ldv,
                       int64_t n_rows, int64_t m, int64_t n, long long* M, int64_t ldm,
                       cudaStream_t st);
cudaError_t min_columns(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                        const void* vj, void* out, int64_t ldo, cudaStream_t st);
// Several 2-way tasks (same n_f, n_v, dtype) in one grid (<= 16 per launch).
cudaError_t czek2_tasks(int dtype, const Czek2Block* tasks, int ntasks, cudaStream_t st);
cudaError_t mgemm(int dtype, const void* W, int64_t ldw, const void* V, int64_t ldv, int64_t n_f,
                  int64_t m, int64_t n, int symmetric, void* M, int64_t ldm, int packed,
                  cudaStream_t st);
cudaError_t czek2_from_num(int dtype, const void* N, int64_t r0, int64_t r1, int64_t m,
                           int64_t n, int diagonal, const void* s_row, const void* s_col,
                           int64_t g_row, int64_t g_col, int64_t n_v, void* vals,
                           unsigned long long* acc, cudaStream_t st);

// Launches the box kernels (single-pivot grid, then the packed-pair grid,
// box3_plan.cuh); the per-pivot prefix sums are built on the device in
// `d_work` (3 * (j1 - j0 + 1) int64).
cudaError_t czek3_box(int dtype, const Czek3Box& b, int64_t* d_work, int64_t n_single,
                      int64_t n_packed, cudaStream_t st);
// Same box, writing the n_ijk partial sums to b.vals instead of values.
cudaError_t czek3_box_numerators(int dtype, const Czek3Box& b, int64_t* d_work, int64_t n_single,
                                 int64_t n_packed, cudaStream_t st);
// Values + checksum of elements [e0, e1) of the box from folded n_ijk.
cudaError_t czek3_from_num(int dtype, const Czek3Box& b, int64_t* d_work, const void* n3,
                           int64_t e0, int64_t e1, void* vals, cudaStream_t st);

cudaError_t peak_minplus(int dtype, int variant, int64_t iters, double* cmp_per_s,
                         double* cmp_per_clk_sm, cudaStream_t st);

}  // namespace psim
