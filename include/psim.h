/*
 * libpsim — B200-native Proportional Similarity (Czekanowski) metric engine.
 *
 * C ABI of the hot path of propsim (reference: /root/reference/pkg/src/propsim).
 * Every entry point names the reference function it replaces (file:line).
 * Plain pointers and sizes only: device buffers are allocated by the caller
 * (the Python host layer uses torch for that), `stream` is a cudaStream_t
 * (NULL = legacy default stream). Calls are stream-ordered and asynchronous
 * unless stated otherwise; the library never frees caller memory.
 *
 * Data layout in device memory (the reference's, core.py:235-236): a vector
 * block is column-major, element (q, i) at V[i * ld + q]. `ld` must be a
 * multiple of 16 bytes / sizeof(element) (2 for FP64, 4 for FP32) and V must
 * be 16-byte aligned; rows q >= n_f of the padding are never read.
 *
 * Every function returns a status: 0 ok, 1 configuration error (propsim
 * ConfigError / ValueError, core.py:20-25), 2 data error (DataError,
 * core.py:24-25), 3 runtime error (EngineError, core.py:28-29; CUDA
 * failures). psim_last_error() describes the last failure of the calling
 * thread.
 */
#ifndef PSIM_H
#define PSIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSIM_OK 0
#define PSIM_ECONFIG 1
#define PSIM_EDATA 2
#define PSIM_ERUNTIME 3

/* run precision (core.py:16 PRECISIONS) */
#define PSIM_F32 0 /* "single" */
#define PSIM_F64 1 /* "double" */

#define PSIM_VERSION 1

/* One 2-way block task: rows = m vectors of W, cols = n vectors of V.
 * Replaces one BlockTask2 of run_2way (metrics2.py:149-158): numerator
 * (mgemm_blocked, mingemm.py:189-209), value matrix (metrics2.py:85-89),
 * compaction (_emit_pair_records, metrics2.py:92-105) and checksum terms
 * (verify.py:74-96).
 * Output `vals` (may be NULL for checksum-only): diagonal task (W == V,
 * m == n): the block triangle li < lj at pair_index(li, lj, m); otherwise
 * the rectangle row-major at li * n + lj. acc[0..1] += 128-bit checksum of
 * the task (global canonical indices), acc[2] += degenerate count.
 * row_begin / row_end (row_end == 0: all rows) restrict one launch to a band
 * of local rows (row_begin a multiple of the CTA tile height, see
 * psim_tile_shape); positions stay those of the whole task, so consecutive
 * bands fill consecutive segments of `vals` (used to overlap D2H with compute). */
typedef struct psim_block2 {
  const void* W;
  int64_t ldw;
  const void* V;
  int64_t ldv;
  int64_t n_f;
  int64_t m, n;
  int32_t diagonal;
  int64_t row_begin, row_end;
  const void* s_row; /* column sums of W's vectors (m) */
  const void* s_col; /* column sums of V's vectors (n) */
  int64_t g_row;     /* global vector id of W column 0 */
  int64_t g_col;     /* global vector id of V column 0 */
  int64_t n_v;       /* total vector count (canonical indexing) */
  void* vals;
  unsigned long long* acc; /* device, 3 x u64 */
} psim_block2_t;

/* One 3-way interval box: every (i, j, k) in [i0,i1) x [j0,j1) x [k0,k1),
 * i < j < k, global ids. Replaces one SliceTask3 of run_3way
 * (_execute_slice, metrics3.py:131-192; regions schedule.py:231-254).
 * Block A holds I (column 0 = global a0), B holds J, C holds K (may alias).
 * N_XY are 2-way numerator tables, column-major N_XY[x + y * ld_XY], x local
 * in X, y local in Y. Output `vals` (may be NULL): pivot-major — for each j
 * in J ascending, rows i, columns k row-major; psim_box3_plan gives the size. */
typedef struct psim_box3 {
  int64_t n_f, n_v;
  const void* VA;
  int64_t ldA, a0;
  const void* VB;
  int64_t ldB, b0;
  const void* VC;
  int64_t ldC, c0;
  const void* SA;
  const void* SB;
  const void* SC;
  const void* NAB;
  int64_t ldAB;
  const void* NAC;
  int64_t ldAC;
  const void* NBC;
  int64_t ldBC;
  int64_t i0, i1, j0, j1, k0, k1;
  void* vals;
  unsigned long long* acc; /* device, 3 x u64 */
} psim_box3_t;

/* --- library / device ----------------------------------------------------- */
int psim_version(void);
const char* psim_last_error(void);
/* Layout of the public structs, for bindings that restate them (ctypes,
 * cgo, ...): out[2k] = sizeof, out[2k + 1] = offsetof its last member, for
 * k = psim_block2_t, psim_box3_t, psim_problem_t, psim_grid_t, psim_piece_t,
 * psim_traffic_t, psim_out_t, psim_plan_t, psim_msg_t (in that order).
 * Writes min(n, 9) pairs; returns 9. */
int psim_abi_layout(int64_t* out, int n);
/* SM count and compute capability of the current device. */
int psim_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* CTA output tile (rows x cols) of the min-plus kernels for a dtype. */
int psim_tile_shape(int dtype, int* rows, int* cols);
/* Kernel launches libpsim has issued in this process (all threads, all
 * devices) since the last reset; reset != 0 returns the count and zeroes it.
 * The benchmark's gpu_launches is this counter over the timed region. */
int psim_launch_count(unsigned long long* out, int reset);

/* --- inputs ---------------------------------------------------------------- */
/* SyntheticSpec.local_block, kind "random-exact" (verify.py:126-147):
 * V[q, i] = mix64((q * n_v_total + i) ^ seed) mod 2^bits for global
 * q in [f0, f0 + n_fp), i in [v0, v0 + n_vp). */
int psim_gen_random_exact(int dtype, uint64_t seed, int bits, int64_t n_v_total, int64_t f0,
                          int64_t v0, int64_t n_fp, int64_t n_vp, void* V, int64_t ld,
                          void* stream);
/* SyntheticSpec.local_block, kind "analytic" (verify.py:126-129): 1 + [q mod n_v == i]. */
int psim_gen_analytic(int dtype, int64_t n_v_total, int64_t f0, int64_t v0, int64_t n_fp,
                      int64_t n_vp, void* V, int64_t ld, void* stream);
/* General-FP test input: uniform [0,1) from the same hash. */
int psim_gen_uniform(int dtype, uint64_t seed, int64_t n_v_total, int64_t f0, int64_t v0,
                     int64_t n_fp, int64_t n_vp, void* V, int64_t ld, void* stream);
/* VectorBlock.__post_init__ (core.py:231-242): flags[0] += #non-finite,
 * flags[1] += #negative (device u64[2]). */
int psim_check_block(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                     unsigned long long* flags, void* stream);

/* --- kernels --------------------------------------------------------------- */
/* column_sums (mingemm.py:212-222): out[i] = sum_q V[q, i], ascending q from +0. */
int psim_column_sums(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                     void* out, void* stream);
/* mgemm_blocked (mingemm.py:189-209): M[i, j] = sum_q min(W[q, i], V[q, j]).
 * packed == 0: M column-major (ldm >= m); symmetric != 0 requires W == V,
 * m == n, computes the upper triangle once and mirrors it.
 * packed != 0: M in the psim_block2_t value layout (triangle if symmetric). */
int psim_mgemm(int dtype, const void* W, int64_t ldw, const void* V, int64_t ldv, int64_t n_f,
               int64_t m, int64_t n, int symmetric, void* M, int64_t ldm, int packed,
               void* stream);
/* Fused 2-way block task (see psim_block2_t). */
int psim_czek2_block(int dtype, const psim_block2_t* task, void* stream);
/* Several tasks of one rank (same dtype, n_f, n_v) in a single grid, so the
 * circulant steps of a slab share one launch and one tail (metrics2.py:148-158
 * over the plan of schedule.py:116-142). Consecutive off-diagonal tasks over
 * the same rows (same W, s_row, g_row, whole row range, each >= one column
 * tile wide) are computed as one task with their columns end to end, and each
 * task's rows past its last multiple of 128 as a 32-row-tile edge task; the
 * values each task writes and its checksum terms do not change. */
int psim_czek2_tasks(int dtype, const psim_block2_t* tasks, int ntasks, void* stream);
/* pack_bits (mingemm.py:279-291): 32 fields per uint32 word, bit q%32 of
 * word q/32 of vector i at words[i * ldw + q/32] (ldw % 4 == 0, padding
 * bits zero); flags[0] += #entries outside {0, 1} (DataError). */
int psim_pack_bits(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                   uint32_t* words, int64_t ldw, unsigned long long* flags, void* stream);
/* mgemm_bitpacked (mingemm.py:294-312): raw counts M[i + j * ldm] = popcount
 * of W_i & V_j over n_rows bits, int64, column-major (ldm >= m). W / V as for
 * psim_pack_bits (16-byte aligned, ld in words, a multiple of 4). */
int psim_mgemm_bits(const uint32_t* W, int64_t ldw, const uint32_t* V, int64_t ldv,
                    int64_t n_rows, int64_t m, int64_t n, int64_t* M, int64_t ldm, void* stream);
/* xj_columns (mingemm.py:225-234): out[k * ldo + q] = min(vj[q], V[k * ld + q])
 * for the n_vp columns of V (the 3-way pivot columns; fused into the 3-way
 * mainloop elsewhere). */
int psim_min_columns(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                     const void* vj, void* out, int64_t ldo, void* stream);
/* Sorenson 2-way task on packed operands (W, V = word arrays, ldw / ldv in
 * words, n_f in fields): counts popcount(a & b) (mgemm_bitpacked,
 * mingemm.py:294-312), converted to the run dtype, then the 2-way value,
 * layout and checksum of psim_czek2_block; s_row / s_col are the dense
 * column sums. No row bands. */
int psim_sorenson2_block(int dtype, const psim_block2_t* task, void* stream);
/* One whole diagonal task (the single-slab run, metrics2.py:149-158) over a
 * block still in host memory (vector i at host + i*host_ld elements): the
 * block is copied into task->W (== task->V, device, padded ld) by the copy
 * engine on copy_stream in chunks of `chunk` vectors from the last one down,
 * each followed by ready[c] = 1 (pageable memory is staged chunk by chunk
 * through a pinned ring by host threads; the call then returns once the last
 * chunk is uploaded); the fused kernel on compute_stream
 * starts at the bottom tiles as soon as their chunk lands. The column sums
 * come from one extra CTA per row tile placed at the head of its bottom-up
 * band: it folds its 128 vectors' sums (k_colsum's sequential order), WRITES
 * them to task->s_row (n entries, device) and sets that row tile's
 * sum-ready flag; the tile CTAs of the band wait on the flags of their rows
 * and columns. task->s_col is not used. vals may be device or pinned host
 * memory. ready: device scratch of ceil(n / chunk) + ceil(n / BM) words (BM
 * from psim_tile_shape). A flag that does not arrive within 20 s makes the
 * kernel give up instead of trapping: psim_stream_error then reports it. The
 * caller validates the block afterwards (psim_check_block) and must keep
 * `host` alive until copy_stream completes. */
int psim_czek2_streamed(int dtype, const psim_block2_t* task, const void* host, int64_t host_ld,
                        int64_t chunk, unsigned* ready, void* compute_stream,
                        void* copy_stream);
/* Wait statistics of streamed runs since the last reset (host, synchronous):
 * out4 = {ns tiles waited for input chunks, ns waited for column sums,
 * number of column-sum waits, longest single wait in ns}. */
int psim_stream_stats(unsigned long long* out4, int reset);
/* *aborted = 1 when the last streamed run gave up waiting for an input chunk
 * or a column-sum flag (its results are invalid: raise EngineError); the
 * flag is cleared by the next psim_czek2_streamed launch. Synchronous. */
int psim_stream_error(unsigned* aborted);
/* 2-way epilogue from reduced packed numerators, rows [r0, r1) of a task's
 * packed layout (field-axis path, metrics2.py:156-158). N and vals point at
 * the first entry of row r0. */
int psim_czek2_from_numerators(int dtype, const void* N, int64_t r0, int64_t r1, int64_t m,
                               int64_t n, int diagonal, const void* s_row, const void* s_col,
                               int64_t g_row, int64_t g_col, int64_t n_v, void* vals,
                               unsigned long long* acc, void* stream);
/* One step of the ordered field-axis fold (RankContext.reduce_field_axis,
 * engine.py:197-216): dst[e] = dst[e] + src[e]. */
int psim_fold_add(int dtype, void* dst, const void* src, int64_t count, void* stream);
/* Byte output mode (io.py:122-136, write_metrics 'byte'): out[e] =
 * floor(clamp(vals[e], 0, 1) * 255 + 0.5) evaluated in double; *flag |= 1 when
 * any value is non-finite (the caller raises DataError, like quantize_values). */
int psim_quantize_bytes(int dtype, const void* vals, int64_t count, uint8_t* out,
                        unsigned long long* flag, void* stream);
/* Output element count and CTA-tile count of a 3-way box (host-only, sync). */
int psim_box3_plan(int dtype, const psim_box3_t* box, int64_t* n_out, int64_t* n_tiles);
/* The tile CTA t of a box's single-pivot grid (packed = 0) or two-segment
 * grid (packed = 1) computes, decoded by the kernels' own code (host-only;
 * the CPU tests check exact coverage with it). out[11] = p0, p1, row0, row1,
 * col0, col1, nr0, nr1, nc0, nc1, side; *n_grid = CTAs of that grid. */
int psim_box3_tile(int dtype, const psim_box3_t* box, int packed, int64_t t, int64_t* out,
                   int64_t* n_grid);
/* Fused 3-way box (see psim_box3_t). */
int psim_czek3_box(int dtype, const psim_box3_t* box, void* stream);
/* Field-axis path of a box (metrics3.py:163-164): n_ijk = sum_q min(min(x_j, v_i), v_k)
 * over this rank's field slab, written to box->vals (pivot-major, no values,
 * no checksum); sums / tables / acc may be NULL. */
int psim_czek3_box_numerators(int dtype, const psim_box3_t* box, void* stream);
/* Values + checksum (into box->acc) of elements [e0, e1) of a box's
 * pivot-major layout from folded n_ijk (n3, vals point at element e0);
 * box->SA..NBC must hold the folded sums and numerator tables. */
int psim_czek3_from_numerators(int dtype, const psim_box3_t* box, const void* n3, int64_t e0,
                               int64_t e1, void* vals, void* stream);

/* --- run-level runtime: the drop-in for run_2way / run_3way ---------------
 * One process per GPU. A context holds the device, this process's rank in the
 * job, the world size and (world > 1) an NCCL communicator plus a comm
 * stream and a copy stream. psim_run2 / psim_run3 run this rank's whole part
 * of a run -- the reference's rank_fn (metrics2.py:131-159,
 * metrics3.py:82-113) and its transport calls (RankContext.send / receive /
 * reduce_field_axis, engine.py:158-216) -- on the device: input block,
 * column sums, the slab plan (circulant 2-way, schedule.py:116-142;
 * tetrahedral 3-way, schedule.py:184-214), NCCL send/recv of blocks, the
 * ordered field-axis fold as a grouped send/recv reduce-scatter, the fused
 * kernels, and the _gather of metrics2.py:174-203 (checksum words, counts,
 * degenerate count, traffic, elapsed: an NCCL all-gather). Synchronous:
 * every rank returns once the global totals are known. Rank r has grid
 * coordinates p_f = r % n_pf, p_v = (r / n_pf) % n_pv, p_r = r / (n_pf
 * n_pv) (core.py:83-97); world must equal n_pf * n_pv * n_pr. */
typedef struct psim_ctx psim_ctx;

#define PSIM_NCCL_ID_BYTES 128

/* input kinds of psim_problem_t (SyntheticSpec kinds, verify.py:126-147, or
 * a caller block: this rank's (n_f / n_pf) x (n_v / n_pv) slab, vector i at
 * block + i * ld elements, in device or host memory) */
#define PSIM_INPUT_RANDOM_EXACT 0
#define PSIM_INPUT_ANALYTIC 1
#define PSIM_INPUT_UNIFORM 2
#define PSIM_INPUT_DEVICE 3
#define PSIM_INPUT_HOST 4

/* psim_run flags */
#define PSIM_RUN_BALANCE_REFERENCE 1 /* 2-way: the reference's unsplit half-offset block */
#define PSIM_RUN_VALUES_SCRATCH 2    /* values stored to a reused workspace buffer (bench) */
#define PSIM_RUN_NO_STREAM 4         /* pinned host input: plain upload, no streamed kernel */

/* Problem (core.py:260-293). */
typedef struct psim_problem {
  int32_t arity; /* 2 or 3 */
  int32_t dtype; /* PSIM_F32 / PSIM_F64 */
  int64_t n_f, n_v;
  int32_t input; /* PSIM_INPUT_* */
  int32_t bits;  /* random-exact */
  uint64_t seed; /* random-exact / uniform */
  const void* block; /* PSIM_INPUT_DEVICE / _HOST */
  int64_t ld;
} psim_problem_t;

/* DecompGrid (core.py:44-80). */
typedef struct psim_grid {
  int32_t n_pf, n_pv, n_pr, n_st;
} psim_grid_t;

/* One value piece of this rank, in canonical ids. kind 2 (PairPiece): v =
 * {g_row, g_col, m, n, diagonal, r0, r1, 0}: rows [r0, r1) of the task's
 * packed layout (psim_block2_t). kind 3 (BoxPiece): v = {i0, i1, j0, j1, k0,
 * k1, e0, e1}: elements [e0, e1) of the box's pivot-major layout. */
typedef struct psim_piece {
  int64_t kind;
  int64_t offset; /* first value in psim_out_t.vals */
  int64_t count;
  int64_t v[8];
} psim_piece_t;

/* Traffic (TrafficStats, engine.py:51-75): send-side messages / elements /
 * bytes per reference phase (metrics2.py:34-39: 0 BLOCK, 1 BLOCK_K, 2 SUM,
 * 3 SUM_K, 4 TASK, 5 PIPE). */
#define PSIM_PHASES 6
typedef struct psim_traffic {
  int64_t messages[PSIM_PHASES], elements[PSIM_PHASES], nbytes[PSIM_PHASES];
} psim_traffic_t;

typedef struct psim_out {
  /* caller-provided (may be NULL): */
  void* vals;                  /* >= plan n_vals values (device or pinned host) */
  psim_piece_t* pieces;        /* host, >= plan n_pieces entries */
  void* sums;                  /* n_v global column sums (device or host) */
  psim_traffic_t* rank_traffic; /* host, world entries (every rank's traffic) */
  /* filled by the run: */
  int64_t n_pieces, n_vals;  /* this rank */
  uint64_t checksum[2];      /* global 128-bit checksum (lo, hi) */
  int64_t count, degenerate; /* global */
  int64_t local_count;       /* values this rank holds */
  double elapsed;            /* device time of the run, max over ranks (s) */
  psim_traffic_t traffic;    /* this rank */
  double kernel_seconds;     /* this rank: CUDA-event time of its fused min-plus launches */
  int64_t kernel_grids;      /* ... and how many launch groups (task groups / boxes) */
  /* PSIM_RUN_VALUES_SCRATCH runs of psim_run3: the piece whose values the
   * workspace scratch holds when the call returns (-1: none) and their
   * device address (pivot-major, as out->vals would hold that piece). */
  int64_t scratch_piece;
  const void* scratch_vals;
} psim_out_t;

typedef struct psim_plan {
  int64_t n_pieces, n_vals, workspace_bytes;
} psim_plan_t;

/* One point-to-point message of a run (psim_run_comms): in NCCL group
 * `group` (groups are issued in ascending order), a send (op 0) to or a
 * receive (op 1) from rank `peer` of `bytes` bytes carrying `what` (PSIM_MSG_*)
 * for `slot`: the slab whose block / sums travel (BLOCK, SUMS), the task /
 * table / box index (TASK, TABLE, BOX). */
#define PSIM_MSG_BLOCK 0
#define PSIM_MSG_SUMS 1
#define PSIM_MSG_TASK 2
#define PSIM_MSG_TABLE 3
#define PSIM_MSG_BOX 4
typedef struct psim_msg {
  int32_t group, op, peer, what;
  int64_t bytes, slot;
} psim_msg_t;

/* 128-byte NCCL unique id (rank 0 creates it, every rank passes it on). */
int psim_nccl_unique_id(uint8_t* id);
/* Collective over all ranks when world > 1 (ncclCommInitRank). device -1
 * makes a planning-only context (psim_run_plan works, no CUDA / NCCL). */
int psim_ctx_create(int device, int rank, int world, const uint8_t* nccl_id, psim_ctx** ctx);
int psim_ctx_destroy(psim_ctx* ctx);
/* Sizes this rank's run needs (host-only): pieces, values, workspace bytes.
 * stage: 3-way stage (-1: all stages), ignored for 2-way. */
int psim_run_plan(const psim_ctx* ctx, const psim_problem_t* problem, const psim_grid_t* grid,
                  int stage, int flags, psim_plan_t* plan);
/* psim_run_plan plus this rank's value pieces (host-only; cap >= n_pieces):
 * exactly the pieces psim_run2 / psim_run3 will report. */
int psim_run_pieces(const psim_ctx* ctx, const psim_problem_t* problem, const psim_grid_t* grid,
                    int stage, int flags, psim_plan_t* plan, psim_piece_t* pieces, int64_t cap);
/* The point-to-point messages this rank's psim_run2 / psim_run3 issues, in
 * order (host-only, any context): *n = count; up to cap written to msgs. */
int psim_run_comms(const psim_ctx* ctx, const psim_problem_t* problem, const psim_grid_t* grid,
                   int stage, int flags, psim_msg_t* msgs, int64_t cap, int64_t* n);
/* run_2way / run_3way for this rank (see above). workspace: device memory of
 * at least plan.workspace_bytes (256-byte aligned). stream: the compute
 * stream (the caller's order is respected). */
int psim_run2(psim_ctx* ctx, const psim_problem_t* problem, const psim_grid_t* grid, int flags,
              void* workspace, int64_t workspace_bytes, psim_out_t* out, void* stream);
int psim_run3(psim_ctx* ctx, const psim_problem_t* problem, const psim_grid_t* grid, int stage,
              int flags, void* workspace, int64_t workspace_bytes, psim_out_t* out, void* stream);
/* Memory helpers for callers without a CUDA allocator of their own (the
 * reference-side ctypes binding): device (pinned_host = 0)
 * or page-locked host memory; psim_memcpy is a synchronous cudaMemcpyDefault. */
int psim_malloc(void** ptr, int64_t bytes, int pinned_host);
int psim_free(void* ptr, int pinned_host);
int psim_memcpy(void* dst, const void* src, int64_t bytes);
/* checksum (verify.py:86-96) of `count` values with canonical indices
 * idx[e] (idx == NULL: idx0 + e): acc[0..1] += sum mix64(t) * (mix64(bits)
 * | 1) mod 2^128 (FP32 bits zero-extended, verify.py:58-65); acc[2] is not
 * touched. vals / idx / acc on the device. */
int psim_checksum(int dtype, const void* vals, const int64_t* idx, int64_t idx0, int64_t count,
                  unsigned long long* acc, void* stream);

/* --- measurement ----------------------------------------------------------- */
/* Min+add issue-rate microbenchmark of the mainloop mix (roofline
 * denominator). Synchronous. */
int psim_peak_minplus(int dtype, int variant, int64_t iters, double* cmp_per_s,
                      double* cmp_per_clk_sm, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSIM_H */
