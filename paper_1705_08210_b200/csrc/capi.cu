// extern "C" boundary of libpsim (declared in include/psim.h): argument
// validation, error-status mapping and the host-side planning of 3-way
// boxes. No kernel code lives here.
#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "box3_plan.cuh"
#include "psim_internal.h"

namespace psim {

static std::atomic<unsigned long long> g_launches{0};

void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

}  // namespace psim

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PSIM_OK;
  if (e == cudaErrorInvalidConfiguration)
    return fail(PSIM_ECONFIG, "%s: launch shape exceeds device limits", what);
  return fail(PSIM_ERUNTIME, "%s: CUDA error %s (%s)", what, cudaGetErrorName(e),
              cudaGetErrorString(e));
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

inline int esize(int dtype) { return dtype == psim::kF64 ? 8 : 4; }

int check_dtype(int dtype) {
  if (dtype != psim::kF32 && dtype != psim::kF64)
    return fail(PSIM_ECONFIG, "dtype must be PSIM_F32 (0) or PSIM_F64 (1), got %d", dtype);
  return PSIM_OK;
}

// Operand contract of the min-plus mainloop: 16-byte aligned base, leading
// dimension covering n_f and a multiple of one 16-byte chunk.
int check_operand(int dtype, const void* p, int64_t ld, int64_t n_f, const char* name) {
  if (!p) return fail(PSIM_ECONFIG, "%s is NULL", name);
  if (reinterpret_cast<uintptr_t>(p) % 16)
    return fail(PSIM_ECONFIG, "%s must be 16-byte aligned", name);
  const int vec = 16 / esize(dtype);
  if (ld < n_f || ld % vec)
    return fail(PSIM_ECONFIG, "%s: ld=%lld must be >= n_f=%lld and a multiple of %d", name,
                (long long)ld, (long long)n_f, vec);
  return PSIM_OK;
}

// Per-pivot tile and output counts of a 3-way box (see psim_box3_t);
// *n_packed = CTAs of the packed-pair grid (box3_plan.cuh).
void box3_counts(int dtype, const psim_box3_t& b, std::vector<int64_t>* tile_pref,
                 std::vector<int64_t>* out_pref, int64_t* n_packed = nullptr,
                 std::vector<int64_t>* packed_pref = nullptr) {
  int bm = 0, bn = 0;
  psim::tile_shape(dtype, &bm, &bn);
  const int64_t nJ = b.j1 > b.j0 ? b.j1 - b.j0 : 0;
  tile_pref->assign(nJ + 1, 0);
  out_pref->assign(nJ + 1, 0);
  int64_t packed = 0;
  if (packed_pref) packed_pref->assign(nJ + 1, 0);
  for (int64_t jj = 0; jj < nJ; ++jj) {
    const psim::Pivot3 g = psim::pivot3(b.i0, b.i1, b.j0, b.j1, b.k0, b.k1, bm, bn, b.j0 + jj);
    (*tile_pref)[jj + 1] = (*tile_pref)[jj] + g.tiles;
    (*out_pref)[jj + 1] = (*out_pref)[jj] + g.nrows * g.ncols;
    packed += g.packed;
    if (packed_pref) (*packed_pref)[jj + 1] = packed;
  }
  if (n_packed) *n_packed = packed;
}

}  // namespace

namespace psim {
// Error reporting for the other host translation units (runtime.cu).
int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
}  // namespace psim

extern "C" {

int psim_version(void) { return PSIM_VERSION; }

int psim_abi_layout(int64_t* out, int n) {
  const int64_t t[] = {
      (int64_t)sizeof(psim_block2_t),  (int64_t)offsetof(psim_block2_t, acc),
      (int64_t)sizeof(psim_box3_t),    (int64_t)offsetof(psim_box3_t, acc),
      (int64_t)sizeof(psim_problem_t), (int64_t)offsetof(psim_problem_t, ld),
      (int64_t)sizeof(psim_grid_t),    (int64_t)offsetof(psim_grid_t, n_st),
      (int64_t)sizeof(psim_piece_t),   (int64_t)offsetof(psim_piece_t, v),
      (int64_t)sizeof(psim_traffic_t), (int64_t)offsetof(psim_traffic_t, nbytes),
      (int64_t)sizeof(psim_out_t),     (int64_t)offsetof(psim_out_t, scratch_vals),
      (int64_t)sizeof(psim_plan_t),    (int64_t)offsetof(psim_plan_t, workspace_bytes),
      (int64_t)sizeof(psim_msg_t),     (int64_t)offsetof(psim_msg_t, slot),
  };
  constexpr int kStructs = (int)(sizeof(t) / sizeof(t[0]) / 2);
  for (int k = 0; out && k < 2 * std::min(n, kStructs); ++k) out[k] = t[k];
  return kStructs;
}

const char* psim_last_error(void) { return g_err; }

int psim_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (sm_count) cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  return cuda_status(cudaGetLastError(), "psim_device_info");
}

int psim_tile_shape(int dtype, int* rows, int* cols) {
  if (int r = check_dtype(dtype)) return r;
  int bm = 0, bn = 0;
  psim::tile_shape(dtype, &bm, &bn);
  if (rows) *rows = bm;
  if (cols) *cols = bn;
  return PSIM_OK;
}

int psim_gen_random_exact(int dtype, uint64_t seed, int bits, int64_t n_v_total, int64_t f0,
                          int64_t v0, int64_t n_fp, int64_t n_vp, void* V, int64_t ld,
                          void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (bits < 0 || bits > 53) return fail(PSIM_ECONFIG, "bits must be in [0, 53], got %d", bits);
  if (!V || ld < n_fp) return fail(PSIM_ECONFIG, "bad output buffer / ld");
  return cuda_status(
      psim::gen_random_exact(dtype, seed, bits, n_v_total, f0, v0, n_fp, n_vp, V, ld, S(stream)),
      "psim_gen_random_exact");
}

int psim_gen_analytic(int dtype, int64_t n_v_total, int64_t f0, int64_t v0, int64_t n_fp,
                      int64_t n_vp, void* V, int64_t ld, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!V || ld < n_fp) return fail(PSIM_ECONFIG, "bad output buffer / ld");
  return cuda_status(psim::gen_analytic(dtype, n_v_total, f0, v0, n_fp, n_vp, V, ld, S(stream)),
                     "psim_gen_analytic");
}

int psim_gen_uniform(int dtype, uint64_t seed, int64_t n_v_total, int64_t f0, int64_t v0,
                     int64_t n_fp, int64_t n_vp, void* V, int64_t ld, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!V || ld < n_fp) return fail(PSIM_ECONFIG, "bad output buffer / ld");
  return cuda_status(
      psim::gen_uniform(dtype, seed, n_v_total, f0, v0, n_fp, n_vp, V, ld, S(stream)),
      "psim_gen_uniform");
}

int psim_check_block(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                     unsigned long long* flags, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!V || !flags || ld < n_fp) return fail(PSIM_ECONFIG, "bad block / flags / ld");
  return cuda_status(psim::check_block(dtype, V, n_fp, n_vp, ld, flags, S(stream)),
                     "psim_check_block");
}

int psim_column_sums(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                     void* out, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!V || !out || ld < n_fp) return fail(PSIM_ECONFIG, "bad block / output / ld");
  return cuda_status(psim::column_sums(dtype, V, n_fp, n_vp, ld, out, S(stream)),
                     "psim_column_sums");
}

int psim_mgemm(int dtype, const void* W, int64_t ldw, const void* V, int64_t ldv, int64_t n_f,
               int64_t m, int64_t n, int symmetric, void* M, int64_t ldm, int packed,
               void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (n_f < 0 || m < 0 || n < 0) return fail(PSIM_ECONFIG, "negative extent");
  if (int r = check_operand(dtype, W, ldw, n_f, "W")) return r;
  if (int r = check_operand(dtype, V, ldv, n_f, "V")) return r;
  if (!M) return fail(PSIM_ECONFIG, "M is NULL");
  if (symmetric && (W != V || m != n || ldw != ldv))
    return fail(PSIM_ECONFIG, "symmetric mGEMM needs W == V and m == n");
  if (!packed && ldm < m) return fail(PSIM_ECONFIG, "ldm=%lld < m=%lld", (long long)ldm, (long long)m);
  return cuda_status(psim::mgemm(dtype, W, ldw, V, ldv, n_f, m, n, symmetric, M, ldm, packed,
                                 S(stream)),
                     "psim_mgemm");
}

static int check_task2(int dtype, const psim_block2_t* t);

int psim_czek2_block(int dtype, const psim_block2_t* t, void* stream) {
  if (int r = check_task2(dtype, t)) return r;
  return cuda_status(psim::czek2_block(dtype, *t, S(stream)), "psim_czek2_block");
}

int psim_czek2_tasks(int dtype, const psim_block2_t* tasks, int ntasks, void* stream) {
  if (ntasks < 0 || (ntasks && !tasks)) return fail(PSIM_ECONFIG, "bad task list");
  for (int k = 0; k < ntasks; ++k) {
    if (int r = check_task2(dtype, tasks + k)) return r;
    if (tasks[k].n_f != tasks[0].n_f || tasks[k].n_v != tasks[0].n_v)
      return fail(PSIM_ECONFIG, "tasks of one launch must share n_f and n_v");
  }
  return cuda_status(psim::czek2_tasks(dtype, tasks, ntasks, S(stream)), "psim_czek2_tasks");
}

int psim_pack_bits(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                   uint32_t* words, int64_t ldw, unsigned long long* flags, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!V || !words || !flags || ld < n_fp) return fail(PSIM_ECONFIG, "bad block / words / ld");
  if (ldw < (n_fp + 31) / 32 || ldw % 4)
    return fail(PSIM_ECONFIG, "ldw=%lld must hold ceil(n_fp/32) words and be a multiple of 4",
                (long long)ldw);
  return cuda_status(psim::pack_bits(dtype, V, n_fp, n_vp, ld, words, ldw, flags, S(stream)),
                     "psim_pack_bits");
}

int psim_mgemm_bits(const uint32_t* W, int64_t ldw, const uint32_t* V, int64_t ldv,
                    int64_t n_rows, int64_t m, int64_t n, int64_t* M, int64_t ldm, void* stream) {
  if (n_rows < 0 || m < 0 || n < 0) return fail(PSIM_ECONFIG, "negative extent");
  if (m == 0 || n == 0) return PSIM_OK;
  if (!W || !V || !M) return fail(PSIM_ECONFIG, "NULL operand");
  const int64_t nw = (n_rows + 31) / 32;
  if (ldw < nw || ldv < nw || ldw % 4 || ldv % 4 || reinterpret_cast<uintptr_t>(W) % 16 ||
      reinterpret_cast<uintptr_t>(V) % 16)
    return fail(PSIM_ECONFIG, "packed operands need 16-byte alignment and ld >= ceil(n_rows/32)");
  if (ldm < m) return fail(PSIM_ECONFIG, "ldm=%lld < m=%lld", (long long)ldm, (long long)m);
  return cuda_status(psim::mgemm_bits(W, ldw, V, ldv, n_rows, m, n,
                                      reinterpret_cast<long long*>(M), ldm, S(stream)),
                     "psim_mgemm_bits");
}

int psim_min_columns(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                     const void* vj, void* out, int64_t ldo, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (n_fp < 0 || n_vp < 0) return fail(PSIM_ECONFIG, "negative extent");
  if (n_fp == 0 || n_vp == 0) return PSIM_OK;
  if (!V || !vj || !out || ld < n_fp || ldo < n_fp)
    return fail(PSIM_ECONFIG, "bad operand / leading dimension");
  return cuda_status(psim::min_columns(dtype, V, n_fp, n_vp, ld, vj, out, ldo, S(stream)),
                     "psim_min_columns");
}

int psim_sorenson2_block(int dtype, const psim_block2_t* t, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!t || !t->W || !t->V || !t->s_row || !t->s_col || !t->acc)
    return fail(PSIM_ECONFIG, "NULL task field");
  const int64_t nw = (t->n_f + 31) / 32;
  if (t->ldw < nw || t->ldv < nw || t->ldw % 4 || t->ldv % 4 ||
      reinterpret_cast<uintptr_t>(t->W) % 16 || reinterpret_cast<uintptr_t>(t->V) % 16)
    return fail(PSIM_ECONFIG, "packed operands need 16-byte alignment and ld >= ceil(n_f/32)");
  if (t->diagonal && (t->m != t->n || t->g_row != t->g_col))
    return fail(PSIM_ECONFIG, "diagonal task needs m == n and g_row == g_col");
  if (t->row_begin || t->row_end) return fail(PSIM_ECONFIG, "row bands not supported here");
  return cuda_status(psim::sorenson2_block(dtype, *t, S(stream)), "psim_sorenson2_block");
}

static int check_task2(int dtype, const psim_block2_t* t) {
  if (int r = check_dtype(dtype)) return r;
  if (!t) return fail(PSIM_ECONFIG, "task is NULL");
  if (t->n_f < 0 || t->m < 0 || t->n < 0) return fail(PSIM_ECONFIG, "negative extent");
  if (int r = check_operand(dtype, t->W, t->ldw, t->n_f, "W")) return r;
  if (int r = check_operand(dtype, t->V, t->ldv, t->n_f, "V")) return r;
  if (!t->s_row || !t->s_col || !t->acc) return fail(PSIM_ECONFIG, "sums / acc is NULL");
  if (t->diagonal && (t->m != t->n || t->g_row != t->g_col))
    return fail(PSIM_ECONFIG, "diagonal task needs m == n and g_row == g_col");
  if (t->g_row < 0 || t->g_col < 0 || t->g_row + t->m > t->n_v || t->g_col + t->n > t->n_v)
    return fail(PSIM_ECONFIG, "task outside [0, n_v)");
  int bm = 0, bn = 0;
  psim::tile_shape(dtype, &bm, &bn);
  const int64_t re = t->row_end ? t->row_end : t->m;
  if (t->row_begin < 0 || re > t->m || t->row_begin > re || t->row_begin % bm)
    return fail(PSIM_ECONFIG, "row band [%lld, %lld) invalid (begin must be a multiple of %d)",
                (long long)t->row_begin, (long long)re, bm);
  return PSIM_OK;
}

int psim_czek2_streamed(int dtype, const psim_block2_t* t, const void* host, int64_t host_ld,
                        int64_t chunk, unsigned* ready, void* compute_stream,
                        void* copy_stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!t) return fail(PSIM_ECONFIG, "task is NULL");
  if (t->n_f < 1 || t->m < 1 || t->m != t->n || !t->diagonal || t->W != t->V ||
      t->ldw != t->ldv || t->g_row != t->g_col || t->row_begin || t->row_end)
    return fail(PSIM_ECONFIG, "streamed run needs one whole diagonal task (W == V, m == n)");
  if (int r = check_operand(dtype, t->W, t->ldw, t->n_f, "W")) return r;
  if (!t->acc || !t->s_row) return fail(PSIM_ECONFIG, "acc / s_row (sums out) is NULL");
  if (t->g_row < 0 || t->g_row + t->m > t->n_v) return fail(PSIM_ECONFIG, "task outside [0, n_v)");
  if (!host || host_ld < t->n_f || !ready || chunk < 1)
    return fail(PSIM_ECONFIG, "bad host block / ready flags / chunk");
  int bm = 0, bn = 0;
  psim::tile_shape(dtype, &bm, &bn);
  if ((t->n + chunk - 1) / chunk + (t->n + bm - 1) / bm > psim::kStreamMaxFlags)
    return fail(PSIM_ECONFIG, "too many chunks / row tiles (flags > %lld)",
                (long long)psim::kStreamMaxFlags);
  if (compute_stream == copy_stream) return fail(PSIM_ECONFIG, "copy stream must differ");
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeDevice)
    return fail(PSIM_ECONFIG, "host block is device memory");
  cudaGetLastError();
  return cuda_status(psim::czek2_streamed(dtype, *t, host, host_ld, chunk, ready,
                                          S(compute_stream), S(copy_stream)),
                     "psim_czek2_streamed");
}

int psim_stream_stats(unsigned long long* out4, int reset) {
  if (!out4) return fail(PSIM_ECONFIG, "NULL argument");
  return cuda_status(psim::stream_stats(out4, reset), "psim_stream_stats");
}

int psim_launch_count(unsigned long long* out, int reset) {
  if (!out) return fail(PSIM_ECONFIG, "NULL argument");
  *out = reset ? psim::g_launches.exchange(0) : psim::g_launches.load();
  return PSIM_OK;
}

int psim_stream_error(unsigned* aborted) {
  if (!aborted) return fail(PSIM_ECONFIG, "NULL argument");
  return cuda_status(psim::stream_error(aborted, 0), "psim_stream_error");
}

int psim_czek2_from_numerators(int dtype, const void* N, int64_t r0, int64_t r1, int64_t m,
                               int64_t n, int diagonal, const void* s_row, const void* s_col,
                               int64_t g_row, int64_t g_col, int64_t n_v, void* vals,
                               unsigned long long* acc, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!N || !s_row || !s_col || !acc) return fail(PSIM_ECONFIG, "NULL argument");
  if (r0 < 0 || r1 > m || r0 > r1) return fail(PSIM_ECONFIG, "row range outside [0, m]");
  return cuda_status(psim::czek2_from_num(dtype, N, r0, r1, m, n, diagonal, s_row, s_col, g_row,
                                          g_col, n_v, vals, acc, S(stream)),
                     "psim_czek2_from_numerators");
}

int psim_fold_add(int dtype, void* dst, const void* src, int64_t count, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!dst || !src) return fail(PSIM_ECONFIG, "NULL argument");
  return cuda_status(psim::fold_add(dtype, dst, src, count, S(stream)), "psim_fold_add");
}

int psim_quantize_bytes(int dtype, const void* vals, int64_t count, uint8_t* out,
                        unsigned long long* flag, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (count < 0) return fail(PSIM_ECONFIG, "count must be >= 0");
  if (count > 0 && (!vals || !out || !flag)) return fail(PSIM_ECONFIG, "NULL argument");
  return cuda_status(psim::quantize_bytes(dtype, vals, count, out, flag, S(stream)),
                     "psim_quantize_bytes");
}

int psim_box3_plan(int dtype, const psim_box3_t* box, int64_t* n_out, int64_t* n_tiles) {
  if (int r = check_dtype(dtype)) return r;
  if (!box) return fail(PSIM_ECONFIG, "box is NULL");
  std::vector<int64_t> tp, op;
  int64_t packed = 0;
  box3_counts(dtype, *box, &tp, &op, &packed);
  if (n_out) *n_out = op.back();
  if (n_tiles) *n_tiles = tp.back() + packed;
  return PSIM_OK;
}

int psim_box3_tile(int dtype, const psim_box3_t* box, int packed, int64_t t, int64_t* out,
                   int64_t* n_grid) {
  if (int r = check_dtype(dtype)) return r;
  if (!box || !out) return fail(PSIM_ECONFIG, "box / out is NULL");
  std::vector<int64_t> tp, op, pp;
  int64_t np = 0;
  box3_counts(dtype, *box, &tp, &op, &np, &pp);
  const std::vector<int64_t>& pref = packed ? pp : tp;
  if (n_grid) *n_grid = pref.back();
  if (t < 0 || t >= pref.back()) return fail(PSIM_ECONFIG, "tile %lld outside the grid", (long long)t);
  const int64_t nJ = box->j1 - box->j0;
  psim::Tile3 d;
  int bm = 0, bn = 0;
  psim::tile_shape(dtype, &bm, &bn);
  if (bm == 128 && bn == 128)
    d = packed ? psim::box3_decode<128, 128, true>(*box, pref.data(), nJ, t)
               : psim::box3_decode<128, 128, false>(*box, pref.data(), nJ, t);
  else if (bm == 128 && bn == 64)
    d = packed ? psim::box3_decode<128, 64, true>(*box, pref.data(), nJ, t)
               : psim::box3_decode<128, 64, false>(*box, pref.data(), nJ, t);
  else
    return fail(PSIM_ERUNTIME, "psim_box3_tile: unexpected tile shape %dx%d", bm, bn);
  const int64_t v[11] = {d.p0, d.p1, d.row0, d.row1, d.col0, d.col1, d.nr0, d.nr1, d.nc0, d.nc1,
                         d.side};
  for (int x = 0; x < 11; ++x) out[x] = v[x];
  return PSIM_OK;
}

static int check_box(int dtype, const psim_box3_t* b, bool tables) {
  if (int r = check_dtype(dtype)) return r;
  if (!b) return fail(PSIM_ECONFIG, "box is NULL");
  if (b->n_f < 0) return fail(PSIM_ECONFIG, "negative n_f");
  if (int r = check_operand(dtype, b->VA, b->ldA, b->n_f, "VA")) return r;
  if (int r = check_operand(dtype, b->VB, b->ldB, b->n_f, "VB")) return r;
  if (int r = check_operand(dtype, b->VC, b->ldC, b->n_f, "VC")) return r;
  if (tables && (!b->SA || !b->SB || !b->SC || !b->NAB || !b->NAC || !b->NBC || !b->acc))
    return fail(PSIM_ECONFIG, "NULL sums / numerator table / acc");
  if (b->i0 < b->a0 || b->j0 < b->b0 || b->k0 < b->c0 || b->i1 > b->n_v || b->j1 > b->n_v ||
      b->k1 > b->n_v)
    return fail(PSIM_ECONFIG, "box intervals outside their blocks");
  return PSIM_OK;
}

// mode 0: fused values (psim_czek3_box); 1: raw n_ijk (psim_czek3_box_numerators)
static int run_box(int dtype, const psim_box3_t* b, int mode, void* stream, const char* what) {
  std::vector<int64_t> tp, op;
  int64_t n_packed = 0;
  box3_counts(dtype, *b, &tp, &op, &n_packed);
  const int64_t n_single = tp.back();
  if (n_single + n_packed == 0) return PSIM_OK;
  cudaStream_t st = S(stream);
  int64_t* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 3 * tp.size() * sizeof(int64_t), st);
  if (e != cudaSuccess) return cuda_status(e, what);
  e = mode ? psim::czek3_box_numerators(dtype, *b, d, n_single, n_packed, st)
           : psim::czek3_box(dtype, *b, d, n_single, n_packed, st);
  cudaError_t e2 = cudaFreeAsync(d, st);
  if (e == cudaSuccess) e = e2;
  return cuda_status(e, what);
}

int psim_czek3_box(int dtype, const psim_box3_t* b, void* stream) {
  if (int r = check_box(dtype, b, true)) return r;
  return run_box(dtype, b, 0, stream, "psim_czek3_box");
}

int psim_czek3_box_numerators(int dtype, const psim_box3_t* b, void* stream) {
  if (int r = check_box(dtype, b, false)) return r;
  if (!b->vals) return fail(PSIM_ECONFIG, "vals (the n_ijk output) is NULL");
  return run_box(dtype, b, 1, stream, "psim_czek3_box_numerators");
}

int psim_czek3_from_numerators(int dtype, const psim_box3_t* b, const void* n3, int64_t e0,
                               int64_t e1, void* vals, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!b || !n3) return fail(PSIM_ECONFIG, "NULL box / numerators");
  if (!b->SA || !b->SB || !b->SC || !b->NAB || !b->NAC || !b->NBC || !b->acc)
    return fail(PSIM_ECONFIG, "NULL sums / numerator table / acc");
  std::vector<int64_t> tp, op;
  box3_counts(dtype, *b, &tp, &op);
  if (e0 < 0 || e1 > op.back() || e0 > e1) return fail(PSIM_ECONFIG, "element range outside box");
  if (e1 == e0) return PSIM_OK;
  cudaStream_t st = S(stream);
  int64_t* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 3 * tp.size() * sizeof(int64_t), st);
  if (e != cudaSuccess) return cuda_status(e, "psim_czek3_from_numerators workspace");
  e = psim::czek3_from_num(dtype, *b, d, n3, e0, e1, vals, st);
  cudaError_t e2 = cudaFreeAsync(d, st);
  if (e == cudaSuccess) e = e2;
  return cuda_status(e, "psim_czek3_from_numerators");
}

int psim_peak_minplus(int dtype, int variant, int64_t iters, double* cmp_per_s,
                      double* cmp_per_clk_sm, void* stream) {
  if (int r = check_dtype(dtype)) return r;
  if (!cmp_per_s || !cmp_per_clk_sm || iters < 1) return fail(PSIM_ECONFIG, "bad arguments");
  return cuda_status(psim::peak_minplus(dtype, variant, iters, cmp_per_s, cmp_per_clk_sm,
                                        S(stream)),
                     "psim_peak_minplus");
}

}  // extern "C"
