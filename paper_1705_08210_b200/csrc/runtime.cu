// Run-level runtime: one rank's whole run_2way / run_3way on the device, with
// NCCL for every exchange (include/psim.h, "run-level runtime").
//
// Reference mapping (paths under /root/reference/pkg/src/propsim):
//   rank_fn of run_2way          metrics2.py:131-159   -> Run2::execute
//   rank_fn of run_3way          metrics3.py:82-113    -> Run3::execute
//   _execute_slice               metrics3.py:131-192   -> psim_czek3_box per box
//   slab plans                   schedule.py:116-142, 184-263 -> plan_2way / plan_3way
//   RankContext.send / receive   engine.py:177-184     -> ncclSend / ncclRecv (comm stream)
//   RankContext.reduce_field_axis engine.py:197-216    -> grouped send/recv reduce-scatter,
//                                                         then the ascending-p_f fold
//   _gather                      metrics2.py:174-203   -> ncclAllGather of per-rank totals
//   TrafficStats                 engine.py:51-75       -> psim_traffic_t
//
// NCCL is bound at run time (dlopen of the libnccl.so.2 the process already
// has -- torch's -- or the system one), so libpsim loads on machines without
// it; a world of 1 needs no NCCL at all. All transfers are byte streams
// (ncclChar); sub-group collectives (the field axis) are grouped p2p.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "psim_internal.h"

namespace psim {
int set_error(int code, const char* fmt, ...);
cudaError_t checksum(int dtype, const void* vals, const int64_t* idx, int64_t idx0, int64_t count,
                     unsigned long long* acc, cudaStream_t st);
}  // namespace psim

namespace {

using psim::set_error;

// ---------------------------------------------------------------------------
// NCCL, bound at run time

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  const char* error = nullptr;
};

const Nccl& nccl() {
  static Nccl api = [] {
    Nccl a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, if loaded
    if (!h) {
      const char* path = getenv("PSIM_NCCL_LIBRARY");
      h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      a.error = "libnccl.so.2 not found (set PSIM_NCCL_LIBRARY)";
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.Send || !a.Recv ||
        !a.GroupStart || !a.GroupEnd || !a.AllGather || !a.GetErrorString)
      a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

// Status helpers: the first failure wins and is kept in psim_last_error().
struct Status {
  int code = PSIM_OK;
  bool ok() const { return code == PSIM_OK; }
  bool cuda(cudaError_t e, const char* what) {
    if (code == PSIM_OK && e != cudaSuccess)
      code = set_error(PSIM_ERUNTIME, "%s: CUDA error %s (%s)", what, cudaGetErrorName(e),
                       cudaGetErrorString(e));
    return code == PSIM_OK;
  }
  bool nc(ncclResult_t r, const char* what) {
    if (code == PSIM_OK && r != ncclSuccess)
      code = set_error(PSIM_ERUNTIME, "%s: NCCL error %s", what, nccl().GetErrorString(r));
    return code == PSIM_OK;
  }
  bool psim(int r) {  // a libpsim entry point's status (its message is already set)
    if (code == PSIM_OK) code = r;
    return code == PSIM_OK;
  }
};

inline int64_t esize(int dtype) { return dtype == psim::kF64 ? 8 : 4; }
inline int64_t ld_for(int64_t n_fp) { return std::max<int64_t>(32, (n_fp + 31) / 32 * 32); }
inline int64_t pair_count(int64_t m, int64_t n, bool diag) {
  return diag ? m * (m - 1) / 2 : m * n;
}
inline int64_t packed_offset(int64_t row, int64_t m, int64_t n, bool diag) {
  return diag ? row * (2 * m - row - 1) / 2 : row * n;
}

// Bump allocator over the caller's workspace; a dry run only measures.
struct Arena {
  char* base = nullptr;
  int64_t off = 0;
  bool dry = true;
  void* take(int64_t bytes) {
    off = (off + 255) / 256 * 256;
    void* p = dry ? nullptr : base + off;
    off += std::max<int64_t>(bytes, 1);
    return p;
  }
};

// Spin on an event (cudaEventQuery loop): a blocking wait after a long kernel
// returned up to 650 ms late on these boxes.
cudaError_t spin(cudaEvent_t ev) {
  for (;;) {
    cudaError_t e = cudaEventQuery(ev);
    if (e != cudaErrorNotReady) return e;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// context

struct psim_ctx {
  int device = 0, rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  cudaStream_t cstream = nullptr;  // NCCL block exchanges
  cudaStream_t copy = nullptr;     // streamed uploads
  int64_t* pinned = nullptr;       // host staging for small results (4 KB + gathers)
  int64_t pinned_len = 0;
};

namespace {

// Plans (plan.py restated; identical event order).
struct Exch {
  int step, send_to, recv_from;
};
struct Task2 {
  int step, row_block, col_block;
  int64_t r0, r1, c0, c1;
  bool diag() const { return row_block == col_block; }
};

// schedule.py:116-142 with the split half-offset block (balance "split") or
// the reference's rule (balance "reference").
void plan_2way(int n_pv, int n_pr, int p, int p_r, int64_t n_vp, bool reference,
               std::vector<Exch>* ex, std::vector<Task2>* tasks) {
  const int half = n_pv / 2;
  for (int delta = 0; delta <= half; ++delta) {
    if (delta % n_pr != p_r) continue;
    if (delta == 0) {
      tasks->push_back({0, p, p, 0, n_vp, 0, n_vp});
      continue;
    }
    const int col = (p + delta) % n_pv;
    ex->push_back({delta, ((p - delta) % n_pv + n_pv) % n_pv, col});
    if (n_pv % 2 == 0 && delta == half) {
      if (reference) {
        if (p < half) tasks->push_back({delta, p, col, 0, n_vp, 0, n_vp});
      } else if (p < half) {
        tasks->push_back({delta, p, col, 0, n_vp / 2, 0, n_vp});
      } else {
        tasks->push_back({delta, p, col, 0, n_vp, n_vp / 2, n_vp});
      }
      continue;
    }
    tasks->push_back({delta, p, col, 0, n_vp, 0, n_vp});
  }
}

struct Box {
  int A, B, C;  // slabs holding I, J, K
  int64_t i0, i1, j0, j1, k0, k1;
  bool edge;
};

int perm_rank(int I, int J, int K) {
  int o[3] = {I, J, K};
  std::sort(o, o + 3);
  const int first = I == o[0] ? 0 : (I == o[1] ? 1 : 2);
  return 2 * first + (J > K ? 1 : 0);
}

void stage_range(int s_t, int s, int64_t n_vp, int n_st, int64_t* lo, int64_t* hi) {
  *lo = ((int64_t)(s_t + n_st * s) * n_vp) / (6 * n_st);
  *hi = ((int64_t)(s_t + 1 + n_st * s) * n_vp) / (6 * n_st);
}

// schedule.py:184-214 (units) + plan.unit_boxes (schedule.py:231-263).
void plan_3way(int n_pv, int n_pr, int p, int p_r, int64_t n_vp, int n_st, int stage,
               std::vector<Box>* boxes) {
  struct Unit {
    int a, b, c, cls, slice;
  };  // cls 0 edge, 1 face, 2 volume
  std::vector<Unit> units;
  int counter = 0;
  for (int s = 0; s < 6; ++s, ++counter)
    if (counter % n_pr == p_r) units.push_back({p, p, p, 0, s});
  for (int s = 0; s < 6; ++s)
    for (int dj = 1; dj < n_pv; ++dj, ++counter)
      if (counter % n_pr == p_r) units.push_back({p, (p + dj) % n_pv, (p + dj) % n_pv, 1, s});
  for (int dk = 1; dk < n_pv; ++dk) {
    const int K = (p + dk) % n_pv;
    for (int dj = 1; dj < n_pv; ++dj, ++counter) {
      if (counter % n_pr == p_r && dj != dk) {
        const int J = (p + dj) % n_pv;
        units.push_back({p, J, K, 2, perm_rank(p, J, K)});
      }
    }
  }
  for (const Unit& u : units) {
    for (int s_t = 0; s_t < n_st; ++s_t) {
      if (stage >= 0 && s_t != stage) continue;
      int64_t lo, hi;
      stage_range(s_t, u.slice, n_vp, n_st, &lo, &hi);
      Box b{};
      if (u.cls == 0) {
        const int64_t o = (int64_t)u.a * n_vp;
        b = {u.a, u.a, u.a, o, o + n_vp, o, o + n_vp, o + lo, o + hi, true};
      } else if (u.cls == 1) {
        const int64_t bp = (int64_t)u.a * n_vp, bj = (int64_t)u.b * n_vp;
        if (u.a < u.b)
          b = {u.a, u.b, u.b, bp + lo, bp + hi, bj, bj + n_vp, bj, bj + n_vp, false};
        else
          b = {u.b, u.b, u.a, bj, bj + n_vp, bj, bj + n_vp, bp + lo, bp + hi, false};
      } else {
        int o[3] = {u.a, u.b, u.c};
        std::sort(o, o + 3);
        const int64_t ba = (int64_t)o[0] * n_vp, bb = (int64_t)o[1] * n_vp,
                      bc = (int64_t)o[2] * n_vp;
        b = {o[0], o[1], o[2], ba + lo, ba + hi, bb, bb + n_vp, bc, bc + n_vp, false};
      }
      // plan.merge_boxes: adjacent K (or I) intervals of the same box join
      if (!boxes->empty()) {
        Box& a = boxes->back();
        if (a.edge == b.edge && a.A == b.A && a.B == b.B && a.C == b.C && a.i0 == b.i0 &&
            a.i1 == b.i1 && a.j0 == b.j0 && a.j1 == b.j1 && a.k1 == b.k0) {
          a.k1 = b.k1;
          continue;
        }
        if (a.edge == b.edge && a.A == b.A && a.B == b.B && a.C == b.C && a.j0 == b.j0 &&
            a.j1 == b.j1 && a.k0 == b.k0 && a.k1 == b.k1 && a.i1 == b.i0) {
          a.i1 = b.i1;
          continue;
        }
      }
      boxes->push_back(b);
    }
  }
}

// Row chunks of a packed task with about equal element counts (field-split
// reduce-scatter: chunk f goes to field rank f).
std::vector<int64_t> row_chunks(int64_t m, int64_t n, bool diag, int parts) {
  std::vector<int64_t> b(parts + 1, 0);
  const int64_t total = pair_count(m, n, diag);
  int64_t row = 0;
  for (int p = 1; p < parts; ++p) {
    const long double target = (long double)total * p / parts;
    while (row < m && (long double)packed_offset(row, m, n, diag) < target) ++row;
    b[p] = row;
  }
  b[parts] = m;
  for (int p = 1; p <= parts; ++p) b[p] = std::max(b[p], b[p - 1]);
  return b;
}

// ---------------------------------------------------------------------------
// common per-rank state

struct Rank {
  psim_ctx* ctx;
  const psim_problem_t* pr;
  const psim_grid_t* g;
  int flags;
  cudaStream_t st;
  Status S;
  Arena A;
  int p_f = 0, p_v = 0, p_r = 0;
  int64_t n_fp = 0, n_vp = 0, ld = 0, esz = 8;
  int dtype = 1;
  // device buffers
  void* own = nullptr;  // own block (padded ld)
  int64_t own_ld = 0;
  void* s_own = nullptr;
  unsigned long long* acc = nullptr;
  unsigned long long* dflags = nullptr;  // validation flags (2 x u64)
  int64_t* gather = nullptr;             // all-gather of totals [world][kTot]
  void* sum_parts = nullptr;             // field all-gather of sums [n_pf][n_vp]
  void* all_sums = nullptr;              // [world][n_vp]
  bool validate = false;
  bool streamed = false;
  unsigned* ready = nullptr;
  int64_t chunk = 0;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_tmp = nullptr;
  psim_traffic_t traffic{};
  std::vector<psim_piece_t> pieces;
  int64_t n_vals = 0, local_count = 0;
  std::vector<cudaEvent_t> kev;  // (start, end) pairs around the fused min-plus launches
  // PSIM_RUN_VALUES_SCRATCH: the piece whose values the scratch buffer holds
  // at the end of the run, and where (reported in psim_out_t)
  int64_t scratch_piece = -1;
  const void* scratch_vals = nullptr;

  bool kmark() {  // one event on the compute stream
    cudaEvent_t e;
    if (!S.cuda(cudaEventCreate(&e), "event")) return false;
    kev.push_back(e);
    return S.cuda(cudaEventRecord(e, st), "event");
  }

  static constexpr int kTot = 8 + 3 * PSIM_PHASES;  // lo, hi, deg, count, elapsed, f0, f1, 0

  int rank_of(int pf, int pv, int prr) const { return pf + g->n_pf * (pv + g->n_pv * prr); }

  void count_send(int phase, int64_t elements, int64_t bytes) {
    traffic.messages[phase] += 1;
    traffic.elements[phase] += elements;
    traffic.nbytes[phase] += bytes;
  }

  bool setup() {
    const int world = ctx->world, rank = ctx->rank;
    p_f = rank % g->n_pf;
    p_v = (rank / g->n_pf) % g->n_pv;
    p_r = rank / (g->n_pf * g->n_pv);
    n_fp = pr->n_f / g->n_pf;
    n_vp = pr->n_v / g->n_pv;
    dtype = pr->dtype;
    esz = esize(dtype);
    ld = ld_for(n_fp);
    // the caller's device block is used in place when it has the padded pitch
    // (blocks travel between ranks as whole n_vp * ld spans)
    const bool dev_ok = pr->input == PSIM_INPUT_DEVICE && pr->block &&
                        reinterpret_cast<uintptr_t>(pr->block) % 16 == 0 && pr->ld == ld;
    if (dev_ok) {
      own = const_cast<void*>(pr->block);
      own_ld = pr->ld;
    } else {
      own = A.take(n_vp * ld * esz);
      own_ld = ld;
    }
    validate = pr->input == PSIM_INPUT_DEVICE || pr->input == PSIM_INPUT_HOST;
    s_own = A.take(n_vp * esz);
    acc = static_cast<unsigned long long*>(A.take(3 * 8));
    dflags = static_cast<unsigned long long*>(A.take(2 * 8));
    gather = static_cast<int64_t*>(A.take((int64_t)world * kTot * 8));
    if (g->n_pf > 1) sum_parts = A.take((int64_t)g->n_pf * n_vp * esz);
    all_sums = A.take((int64_t)world * n_vp * esz);
    return true;
  }

  // Own block on the device: generated, uploaded, or the caller's.
  bool load(bool allow_stream) {
    const int64_t f0 = p_f * n_fp, v0 = p_v * n_vp;
    switch (pr->input) {
      case PSIM_INPUT_RANDOM_EXACT:
        return S.cuda(psim::gen_random_exact(dtype, pr->seed, pr->bits, pr->n_v, f0, v0, n_fp,
                                             n_vp, own, own_ld, st), "generate block");
      case PSIM_INPUT_ANALYTIC:
        return S.cuda(psim::gen_analytic(dtype, pr->n_v, f0, v0, n_fp, n_vp, own, own_ld, st),
                      "generate block");
      case PSIM_INPUT_UNIFORM:
        return S.cuda(psim::gen_uniform(dtype, pr->seed, pr->n_v, f0, v0, n_fp, n_vp, own,
                                        own_ld, st), "generate block");
      case PSIM_INPUT_DEVICE:
        if (own == pr->block) return true;
        return S.cuda(cudaMemcpy2DAsync(own, own_ld * esz, pr->block, pr->ld * esz, n_fp * esz,
                                        n_vp, cudaMemcpyDeviceToDevice, st), "copy block");
      default: {  // host
        if (allow_stream) return true;  // uploaded by the streamed kernel
        return S.cuda(cudaMemcpy2DAsync(own, own_ld * esz, pr->block, pr->ld * esz, n_fp * esz,
                                        n_vp, cudaMemcpyHostToDevice, st), "upload block");
      }
    }
  }

  // --- point-to-point plumbing -------------------------------------------
  // Every NCCL send / recv of a run goes through send() / recv() inside a
  // gstart() / gend() group, and is appended to `log` (psim_run_comms returns
  // it; with `trace` set nothing is issued -- the CPU tests replay the log over
  // gloo to check the schedule for every grid, N = 8 included).
  std::vector<psim_msg_t> log;
  int group = 0;
  bool trace = false;

  bool gstart() { return trace || S.nc(nccl().GroupStart(), "ncclGroupStart"); }
  bool gend() {
    ++group;
    return trace || S.nc(nccl().GroupEnd(), "ncclGroupEnd");
  }
  bool send(const void* p, int64_t bytes, int peer, cudaStream_t s, int phase, int64_t elems,
            int what, int64_t slot) {
    log.push_back({group, 0, peer, what, bytes, slot});
    count_send(phase, elems, bytes);
    return trace || S.nc(nccl().Send(p, bytes, ncclChar, peer, ctx->comm, s), "ncclSend");
  }
  bool recv(void* p, int64_t bytes, int peer, cudaStream_t s, int what, int64_t slot) {
    log.push_back({group, 1, peer, what, bytes, slot});
    return trace || S.nc(nccl().Recv(p, bytes, ncclChar, peer, ctx->comm, s), "ncclRecv");
  }

  // Grouped p2p all-gather of `bytes` from every field rank of this slab
  // (p_f order) into dst[n_pf][bytes]; dst[p_f] already holds ours.
  bool field_allgather(const void* mine, void* dst, int64_t bytes, int phase, int64_t elems,
                       int what, int64_t slot) {
    char* d = static_cast<char*>(dst);
    if (!trace && d + p_f * bytes != mine &&
        !S.cuda(cudaMemcpyAsync(d + p_f * bytes, mine, bytes, cudaMemcpyDeviceToDevice, st),
                "stage field part"))
      return false;
    if (!gstart()) return false;
    for (int f = 0; f < g->n_pf; ++f) {
      if (f == p_f) continue;
      const int peer = rank_of(f, p_v, p_r);
      send(mine, bytes, peer, st, phase, elems, what, slot);
      recv(d + f * bytes, bytes, peer, st, what, slot);
    }
    return gend();
  }

  // Ordered reduce-scatter over the field group (reduce_field_axis,
  // engine.py:197-216): element range [off[f], off[f+1]) of `part` goes to
  // field rank f; ours lands in rbuf[f][mine] from every f.
  bool field_scatter(const void* part, void* rbuf_, const std::vector<int64_t>& off, int phase,
                     int what, int64_t slot) {
    const int64_t mine = off[p_f + 1] - off[p_f];
    char* rb = static_cast<char*>(rbuf_);
    const char* pp = static_cast<const char*>(part);
    if (!gstart()) return false;
    for (int f = 0; f < g->n_pf; ++f) {
      const int64_t cnt = off[f + 1] - off[f];
      if (f == p_f) {
        if (!trace && cnt)
          S.cuda(cudaMemcpyAsync(rb + f * mine * esz, pp + off[f] * esz, cnt * esz,
                                 cudaMemcpyDeviceToDevice, st), "stage part");
        continue;
      }
      const int peer = rank_of(f, p_v, p_r);
      if (cnt) send(pp + off[f] * esz, cnt * esz, peer, st, phase, cnt, what, slot);
      if (mine) recv(rb + f * mine * esz, mine * esz, peer, st, what, slot);
    }
    return gend();
  }

  // reduce_field_axis (engine.py:197-216): ((P0 + P1) + P2) + ... in p_f order.
  bool fold_parts(void* dst, const void* parts, int64_t count) {
    const char* p = static_cast<const char*>(parts);
    if (!S.cuda(cudaMemcpyAsync(dst, p, count * esz, cudaMemcpyDeviceToDevice, st), "fold"))
      return false;
    for (int f = 1; f < g->n_pf; ++f)
      if (!S.cuda(psim::fold_add(dtype, dst, p + f * count * esz, count, st), "fold")) return false;
    return true;
  }

  bool sums() {
    if (!S.cuda(psim::column_sums(dtype, own, n_fp, n_vp, own_ld, s_own, st), "column sums"))
      return false;
    if (g->n_pf == 1) return true;
    return field_allgather(s_own, sum_parts, n_vp * esz, 2, n_vp, PSIM_MSG_SUMS, p_v) &&
           fold_parts(s_own, sum_parts, n_vp);
  }

  // _gather (metrics2.py:174-203): every rank's totals, one all-gather.
  int finish(psim_out_t* out, int64_t count) {
    const int world = ctx->world;
    if (!S.cuda(cudaEventRecord(ev_end, st), "event")) return S.code;
    int64_t* h = ctx->pinned;  // [0, kTot): mine; [64, 64 + world * kTot): all
    if (!S.cuda(cudaMemcpyAsync(h, acc, 24, cudaMemcpyDeviceToHost, st), "acc D2H")) return S.code;
    if (validate && !S.cuda(cudaMemcpyAsync(h + 5, dflags, 16, cudaMemcpyDeviceToHost, st), "D2H"))
      return S.code;
    if (!S.cuda(cudaEventRecord(ev_tmp, st), "event") || !S.cuda(spin(ev_tmp), "run"))
      return S.code;
    if (streamed) {  // the streamed kernel gave up waiting for an upload (czek2.cu)
      unsigned aborted = 0;
      if (!S.psim(psim_stream_error(&aborted))) return S.code;
      if (aborted) h[5] = -1;  // reported after the gather, on every rank
    }
    float ms = 0.f;
    S.cuda(cudaEventElapsedTime(&ms, ev_start, ev_end), "elapsed");
    double el = ms * 1e-3;
    h[3] = count;
    std::memcpy(&h[4], &el, 8);
    if (!validate) h[5] = h[6] = 0;
    h[7] = h[5] < 0 ? 1 : 0;
    if (h[5] < 0) h[5] = 0;
    for (int ph = 0; ph < PSIM_PHASES; ++ph) {
      h[8 + 3 * ph] = traffic.messages[ph];
      h[9 + 3 * ph] = traffic.elements[ph];
      h[10 + 3 * ph] = traffic.nbytes[ph];
    }
    int64_t* all = h + 64;
    if (world > 1) {
      int64_t* dmine = gather;  // reuse: [0] row as the send buffer is not allowed (in place ok)
      int64_t* drow = gather + (int64_t)ctx->rank * kTot;
      S.cuda(cudaMemcpyAsync(drow, h, kTot * 8, cudaMemcpyHostToDevice, st), "totals H2D");
      S.nc(nccl().AllGather(drow, dmine, kTot * 8, ncclChar, ctx->comm, st), "ncclAllGather");
      S.cuda(cudaMemcpyAsync(all, gather, (int64_t)world * kTot * 8, cudaMemcpyDeviceToHost, st),
             "totals D2H");
      if (out->sums) {
        S.nc(nccl().AllGather(s_own, all_sums, n_vp * esz, ncclChar, ctx->comm, st),
             "ncclAllGather sums");
        for (int pv = 0; pv < g->n_pv; ++pv)
          S.cuda(cudaMemcpyAsync(static_cast<char*>(out->sums) + pv * n_vp * esz,
                                 static_cast<char*>(all_sums) + rank_of(0, pv, 0) * n_vp * esz,
                                 n_vp * esz, cudaMemcpyDefault, st), "sums");
      }
      S.cuda(cudaEventRecord(ev_tmp, st), "event");
      S.cuda(spin(ev_tmp), "gather");
      if (!S.ok()) return S.code;
    } else {
      std::memcpy(all, h, kTot * 8);
      if (out->sums &&
          !S.cuda(cudaMemcpyAsync(out->sums, s_own, n_vp * esz, cudaMemcpyDefault, st), "sums"))
        return S.code;
      S.cuda(cudaEventRecord(ev_tmp, st), "event");
      if (!S.cuda(spin(ev_tmp), "sums")) return S.code;
    }
    unsigned __int128 total = 0;
    int64_t deg = 0, cnt = 0, bad0 = 0, bad1 = 0, stalled = 0;
    double emax = 0;
    for (int r = 0; r < world; ++r) {
      const int64_t* t = all + (int64_t)r * kTot;
      total += ((unsigned __int128)(uint64_t)t[1] << 64) | (uint64_t)t[0];
      deg += t[2];
      cnt += t[3];
      double e;
      std::memcpy(&e, &t[4], 8);
      emax = std::max(emax, e);
      bad0 += t[5];
      bad1 += t[6];
      stalled += t[7];
      if (out->rank_traffic) {
        for (int ph = 0; ph < PSIM_PHASES; ++ph) {
          out->rank_traffic[r].messages[ph] = t[8 + 3 * ph];
          out->rank_traffic[r].elements[ph] = t[9 + 3 * ph];
          out->rank_traffic[r].nbytes[ph] = t[10 + 3 * ph];
        }
      }
    }
    out->checksum[0] = (uint64_t)total;
    out->checksum[1] = (uint64_t)(total >> 64);
    out->degenerate = deg;
    out->count = cnt;
    out->elapsed = emax;
    out->traffic = traffic;
    out->kernel_seconds = 0;
    out->kernel_grids = (int64_t)kev.size() / 2;
    for (size_t k = 0; k + 1 < kev.size(); k += 2) {
      float kms = 0.f;
      if (cudaEventElapsedTime(&kms, kev[k], kev[k + 1]) == cudaSuccess)
        out->kernel_seconds += kms * 1e-3;
    }
    out->local_count = local_count;
    out->scratch_piece = scratch_piece;
    out->scratch_vals = scratch_vals;
    out->n_vals = n_vals;
    out->n_pieces = (int64_t)pieces.size();
    if (out->pieces) std::copy(pieces.begin(), pieces.end(), out->pieces);
    if (stalled)
      return set_error(PSIM_ERUNTIME, "streamed input did not arrive within 20 s on %lld rank(s); "
                       "results discarded", (long long)stalled);
    if (bad0) return set_error(PSIM_EDATA, "vector data must be finite (%lld non-finite)",
                               (long long)bad0);
    if (bad1) return set_error(PSIM_EDATA, "vector data must be nonnegative (%lld negative)",
                               (long long)bad1);
    return PSIM_OK;
  }

  bool begin() {
    if (!S.cuda(cudaEventCreate(&ev_start), "event") || !S.cuda(cudaEventCreate(&ev_end), "event") ||
        !S.cuda(cudaEventCreateWithFlags(&ev_tmp, cudaEventDisableTiming), "event"))
      return false;
    S.cuda(cudaEventRecord(ev_start, st), "event");
    S.cuda(cudaMemsetAsync(acc, 0, 24, st), "acc");
    if (validate) S.cuda(cudaMemsetAsync(dflags, 0, 16, st), "flags");
    return S.ok();
  }
  ~Rank() {
    for (cudaEvent_t e : kev) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_end) cudaEventDestroy(ev_end);
    if (ev_tmp) cudaEventDestroy(ev_tmp);
  }
};

int check_common(const psim_ctx* ctx, const psim_problem_t* p, const psim_grid_t* g, int arity) {
  if (!ctx || !p || !g) return set_error(PSIM_ECONFIG, "NULL context / problem / grid");
  if (p->arity != arity) return set_error(PSIM_ECONFIG, "problem arity %d != %d", p->arity, arity);
  if (p->dtype != psim::kF32 && p->dtype != psim::kF64)
    return set_error(PSIM_ECONFIG, "dtype must be PSIM_F32 or PSIM_F64");
  if (g->n_pf < 1 || g->n_pv < 1 || g->n_pr < 1 || g->n_st < 1)
    return set_error(PSIM_ECONFIG, "grid axes must be >= 1");
  if ((int64_t)g->n_pf * g->n_pv * g->n_pr != ctx->world)
    return set_error(PSIM_ECONFIG, "world size %d != n_pf * n_pv * n_pr = %d", ctx->world,
                     g->n_pf * g->n_pv * g->n_pr);
  if (p->n_f < 1 || p->n_v < arity)
    return set_error(PSIM_ECONFIG, "need n_f >= 1 and n_v >= %d", arity);
  if (p->n_f % g->n_pf || p->n_v % g->n_pv)
    return set_error(PSIM_ECONFIG, "n_pf must divide n_f and n_pv must divide n_v");
  if (p->n_f / g->n_pf < 1 || p->n_v / g->n_pv < 1)
    return set_error(PSIM_ECONFIG, "empty slab");
  if (p->input < PSIM_INPUT_RANDOM_EXACT || p->input > PSIM_INPUT_HOST)
    return set_error(PSIM_ECONFIG, "unknown input kind %d", p->input);
  if ((p->input == PSIM_INPUT_DEVICE || p->input == PSIM_INPUT_HOST) &&
      (!p->block || p->ld < p->n_f / g->n_pf))
    return set_error(PSIM_ECONFIG, "input block is NULL or ld < n_f / n_pf");
  if (p->input == PSIM_INPUT_RANDOM_EXACT && (p->bits < 0 || p->bits > 64))
    return set_error(PSIM_ECONFIG, "bits must be in [0, 64]");
  if (arity == 3 && (p->n_v / g->n_pv) % 6)
    return set_error(PSIM_ECONFIG, "3-way needs n_v / n_pv divisible by 6 (schedule.py:96-100)");
  return PSIM_OK;
}

// ---------------------------------------------------------------------------
// 2-way

struct Run2 : Rank {
  std::vector<Exch> ex;
  std::vector<Task2> tasks;
  std::vector<void*> rblock, rsums;  // one per exchange
  // field split
  void *part = nullptr, *rbuf = nullptr, *tot = nullptr;
  void* scratch = nullptr;

  bool layout(psim_out_t* out) {
    setup();
    plan_2way(g->n_pv, g->n_pr, p_v, p_r, n_vp, flags & PSIM_RUN_BALANCE_REFERENCE, &ex, &tasks);
    // received blocks back to back: consecutive full-width tasks then form one
    // contiguous V operand (flattened into one grid with TMA staging)
    char* ring = static_cast<char*>(A.take((int64_t)ex.size() * n_vp * ld * esz));
    for (size_t k = 0; k < ex.size(); ++k) {
      rblock.push_back(ring ? ring + k * n_vp * ld * esz : nullptr);
      rsums.push_back(A.take(n_vp * esz));
    }
    // host input (pinned, or pageable staged through a pinned ring) with a
    // diagonal task on this rank: streamed upload under the diagonal kernel
    streamed = pr->input == PSIM_INPUT_HOST && g->n_pf == 1 && !(flags & PSIM_RUN_NO_STREAM) &&
               n_vp >= 2 && !tasks.empty() && tasks[0].diag();
    if (streamed) {
      int bm = 0, bn = 0;
      psim::tile_shape(dtype, &bm, &bn);
      chunk = std::max<int64_t>(64, (n_vp + 255) / 256);  // <= 256 chunks (engine2.stream_chunk)
      ready = static_cast<unsigned*>(A.take(((n_vp + chunk - 1) / chunk + (n_vp + bm - 1) / bm) * 4));
      scratch_sums = A.take(n_vp * esz);
    }
    // values / pieces
    int64_t max_cnt = 0, max_mine = 0;
    for (const Task2& t : tasks) {
      const int64_t m = t.r1 - t.r0, n = t.c1 - t.c0;
      const int64_t c = pair_count(m, n, t.diag());
      psim_piece_t pc{};
      pc.kind = 2;
      pc.v[0] = (int64_t)t.row_block * n_vp + t.r0;
      pc.v[1] = (int64_t)t.col_block * n_vp + t.c0;
      pc.v[2] = m;
      pc.v[3] = n;
      pc.v[4] = t.diag();
      if (g->n_pf == 1) {
        pc.v[5] = 0;
        pc.v[6] = m;
        pc.count = c;
      } else {
        const std::vector<int64_t> b = row_chunks(m, n, t.diag(), g->n_pf);
        pc.v[5] = b[p_f];
        pc.v[6] = b[p_f + 1];
        pc.count = packed_offset(b[p_f + 1], m, n, t.diag()) - packed_offset(b[p_f], m, n, t.diag());
        for (int f = 0; f < g->n_pf; ++f)
          max_mine = std::max(max_mine, packed_offset(b[f + 1], m, n, t.diag()) -
                                            packed_offset(b[f], m, n, t.diag()));
      }
      max_cnt = std::max(max_cnt, c);
      pc.offset = n_vals;
      n_vals += pc.count;
      pieces.push_back(pc);
    }
    local_count = n_vals;
    if (g->n_pf > 1) {
      part = A.take(max_cnt * esz);
      rbuf = A.take(max_mine * g->n_pf * esz);
      tot = A.take(max_mine * esz);
    }
    if (flags & PSIM_RUN_VALUES_SCRATCH) scratch = A.take(n_vals * esz);
    (void)out;
    return true;
  }

  void* vals_at(psim_out_t* out, int64_t offset) {
    void* base = scratch ? scratch : (out ? out->vals : nullptr);
    return base ? static_cast<char*>(base) + offset * esz : nullptr;
  }

  psim_block2_t task_struct(const Task2& t, const void* V, int64_t ldv, const void* s_col,
                            void* vals) {
    psim_block2_t b{};
    b.W = static_cast<const char*>(own) + t.r0 * own_ld * esz;
    b.ldw = own_ld;
    b.V = static_cast<const char*>(V) + t.c0 * ldv * esz;
    b.ldv = ldv;
    b.n_f = n_fp;
    b.m = t.r1 - t.r0;
    b.n = t.c1 - t.c0;
    b.diagonal = t.diag();
    b.s_row = static_cast<const char*>(s_own) + t.r0 * esz;
    b.s_col = static_cast<const char*>(s_col) + t.c0 * esz;
    b.g_row = (int64_t)t.row_block * n_vp + t.r0;
    b.g_col = (int64_t)t.col_block * n_vp + t.c0;
    b.n_v = pr->n_v;
    b.vals = vals;
    b.acc = acc;
    return b;
  }

  // Post every block exchange (metrics2.py:140-147) on the comm stream once
  // `ready` (the own block and its sums) has been reached on `after`.
  bool post_exchanges(cudaStream_t after) {
    if (ex.empty()) return true;
    if (!trace && (!S.cuda(cudaEventRecord(ev_tmp, after), "event") ||
                   !S.cuda(cudaStreamWaitEvent(ctx->cstream, ev_tmp, 0), "wait")))
      return false;
    for (size_t k = 0; k < ex.size(); ++k) {
      const int to = rank_of(p_f, ex[k].send_to, p_r), from = rank_of(p_f, ex[k].recv_from, p_r);
      cudaStream_t cs = ctx->cstream;
      gstart();
      send(own, n_vp * own_ld * esz, to, cs, 0, n_fp * n_vp, PSIM_MSG_BLOCK, p_v);
      send(s_own, n_vp * esz, to, cs, 2, n_vp, PSIM_MSG_SUMS, p_v);
      recv(rblock[k], n_vp * ld * esz, from, cs, PSIM_MSG_BLOCK, ex[k].recv_from);
      recv(rsums[k], n_vp * esz, from, cs, PSIM_MSG_SUMS, ex[k].recv_from);
      if (!gend()) return false;
    }
    return true;
  }

  // The comm schedule alone (psim_run_comms): execute()'s groups, in order.
  void comm_trace() {
    if (g->n_pf > 1) field_allgather(s_own, sum_parts, n_vp * esz, 2, n_vp, PSIM_MSG_SUMS, p_v);
    post_exchanges(st);
    if (g->n_pf > 1)
      for (size_t k = 0; k < tasks.size(); ++k) field_scatter(part, rbuf, task_offsets(k), 4,
                                                               PSIM_MSG_TASK, (int64_t)k);
  }

  std::vector<int64_t> task_offsets(size_t k) const {
    const Task2& t = tasks[k];
    const int64_t m = t.r1 - t.r0, n = t.c1 - t.c0;
    const std::vector<int64_t> b = row_chunks(m, n, t.diag(), g->n_pf);
    std::vector<int64_t> off(g->n_pf + 1);
    for (int f = 0; f <= g->n_pf; ++f) off[f] = packed_offset(b[f], m, n, t.diag());
    return off;
  }

  int slot_of(int step) const {
    for (size_t k = 0; k < ex.size(); ++k)
      if (ex[k].step == step) return (int)k;
    return -1;
  }

  bool run_tasks(const std::vector<psim_block2_t>& v) {
    for (size_t k = 0; k < v.size(); k += 16) {
      const int n = (int)std::min<size_t>(16, v.size() - k);
      if (!kmark() || !S.psim(psim_czek2_tasks(dtype, v.data() + k, n, st)) || !kmark())
        return false;
    }
    return true;
  }

  bool execute(psim_out_t* out) {
    if (!begin()) return false;
    if (streamed) return execute_streamed(out);
    if (!load(false)) return false;
    if (validate && !S.cuda(psim::check_block(dtype, own, n_fp, n_vp, own_ld, dflags, st), "check"))
      return false;
    if (!sums()) return false;
    if (g->n_pf == 1) {
      if (!post_exchanges(st)) return false;
      std::vector<psim_block2_t> diag, rest;
      for (size_t k = 0; k < tasks.size(); ++k) {
        const Task2& t = tasks[k];
        void* v = vals_at(out, pieces[k].offset);
        if (t.diag()) {
          diag.push_back(task_struct(t, own, own_ld, s_own, v));
        } else {
          const int s = slot_of(t.step);
          rest.push_back(task_struct(t, rblock[s], ld, rsums[s], v));
        }
      }
      if (!run_tasks(diag)) return false;  // overlaps the exchanges
      if (!ex.empty() && (!S.cuda(cudaEventRecord(ev_tmp, ctx->cstream), "event") ||
                          !S.cuda(cudaStreamWaitEvent(st, ev_tmp, 0), "wait")))
        return false;
      return run_tasks(rest);
    }
    // field split: every exchange first, then per task the partial numerators,
    // the ordered reduce-scatter and the epilogue of this rank's row chunk
    if (!post_exchanges(st)) return false;
    if (!ex.empty() && (!S.cuda(cudaEventRecord(ev_tmp, ctx->cstream), "event") ||
                        !S.cuda(cudaStreamWaitEvent(st, ev_tmp, 0), "wait")))
      return false;
    for (size_t k = 0; k < tasks.size(); ++k) {
      const Task2& t = tasks[k];
      const int64_t m = t.r1 - t.r0, n = t.c1 - t.c0;
      const void* V = own;
      int64_t ldv = own_ld;
      const void* s_col = s_own;
      if (!t.diag()) {
        const int s = slot_of(t.step);
        V = rblock[s];
        ldv = ld;
        s_col = rsums[s];
      }
      const char* W = static_cast<const char*>(own) + t.r0 * own_ld * esz;
      const char* Vc = static_cast<const char*>(V) + t.c0 * ldv * esz;
      if (!kmark() ||
          !S.psim(psim_mgemm(dtype, W, own_ld, Vc, ldv, n_fp, m, n, t.diag(), part, 0, 1, st)) ||
          !kmark())
        return false;
      const std::vector<int64_t> off = task_offsets(k);
      const int64_t mine = off[p_f + 1] - off[p_f];
      if (!field_scatter(part, rbuf, off, 4, PSIM_MSG_TASK, (int64_t)k)) return false;
      if (mine == 0) continue;
      if (!fold_parts(tot, rbuf, mine)) return false;
      const psim_piece_t& pc = pieces[k];
      if (!S.psim(psim_czek2_from_numerators(
              dtype, tot, pc.v[5], pc.v[6], m, n, t.diag(), static_cast<const char*>(s_own) + t.r0 * esz,
              static_cast<const char*>(s_col) + t.c0 * esz, pc.v[0], pc.v[1], pr->n_v,
              vals_at(out, pc.offset), acc, st)))
        return false;
    }
    return S.ok();
  }

  // Pinned host input, no field split: the diagonal task is the streamed
  // kernel (the copy engine uploads the block in chunks while the kernel
  // starts on the tiles that have landed); sums, validation and the block
  // exchanges queue on the copy stream behind the upload; the other tasks
  // follow as one grid once their blocks are in.
  bool execute_streamed(psim_out_t* out) {
    cudaStream_t cp = ctx->copy;
    if (!S.cuda(cudaEventRecord(ev_tmp, st), "event") ||
        !S.cuda(cudaStreamWaitEvent(cp, ev_tmp, 0), "wait"))
      return false;
    psim_block2_t d = task_struct(tasks[0], own, own_ld, s_own, vals_at(out, pieces[0].offset));
    void* s_kernel = scratch_sums;  // the streamed kernel writes its own copy of the sums
    d.s_row = s_kernel;
    if (!kmark() || !S.psim(psim_czek2_streamed(dtype, &d, pr->block, pr->ld, chunk, ready, st, cp)) ||
        !kmark())
      return false;
    // behind the upload on the copy stream: sums (bitwise the kernel's),
    // validation, then the exchanges
    if (!S.cuda(psim::column_sums(dtype, own, n_fp, n_vp, own_ld, s_own, cp), "column sums") ||
        !S.cuda(psim::check_block(dtype, own, n_fp, n_vp, own_ld, dflags, cp), "check"))
      return false;
    if (!post_exchanges(cp)) return false;
    if (!S.cuda(cudaEventRecord(ev_tmp, ex.empty() ? cp : ctx->cstream), "event") ||
        !S.cuda(cudaStreamWaitEvent(st, ev_tmp, 0), "wait"))
      return false;
    std::vector<psim_block2_t> rest;
    for (size_t k = 1; k < tasks.size(); ++k) {
      const int s = slot_of(tasks[k].step);
      rest.push_back(task_struct(tasks[k], rblock[s], ld, rsums[s], vals_at(out, pieces[k].offset)));
    }
    return run_tasks(rest);
  }

  void* scratch_sums = nullptr;
};

// ---------------------------------------------------------------------------
// 3-way

struct Run3 : Rank {
  int stage = -1;
  std::vector<Box> boxes;
  std::vector<void*> blocks, bsums;  // by slab
  struct Tab {
    int X, Y;
    void* data;
  };
  std::vector<Tab> tabs;
  void *tab_parts = nullptr, *part = nullptr, *rbuf = nullptr, *tot = nullptr, *scratch = nullptr;
  std::vector<int64_t> n_out;
  std::vector<int> piece_of;  // box -> index into pieces (-1: no values here)

  void* table(int X, int Y) {
    for (Tab& t : tabs)
      if (t.X == X && t.Y == Y) return t.data;
    return nullptr;
  }

  psim_box3_t box_struct(const Box& b, void* vals, bool with_tables) {
    psim_box3_t s{};
    s.n_f = with_tables ? pr->n_f : n_fp;
    s.n_v = pr->n_v;
    s.VA = blocks[b.A];
    s.ldA = ld;
    s.a0 = (int64_t)b.A * n_vp;
    s.VB = blocks[b.B];
    s.ldB = ld;
    s.b0 = (int64_t)b.B * n_vp;
    s.VC = blocks[b.C];
    s.ldC = ld;
    s.c0 = (int64_t)b.C * n_vp;
    s.i0 = b.i0;
    s.i1 = b.i1;
    s.j0 = b.j0;
    s.j1 = b.j1;
    s.k0 = b.k0;
    s.k1 = b.k1;
    s.vals = vals;
    s.acc = acc;
    if (with_tables) {
      s.SA = bsums[b.A];
      s.SB = bsums[b.B];
      s.SC = bsums[b.C];
      s.NAB = table(b.A, b.B);
      s.ldAB = n_vp;
      s.NAC = table(b.A, b.C);
      s.ldAC = n_vp;
      s.NBC = table(b.B, b.C);
      s.ldBC = n_vp;
    }
    return s;
  }

  bool layout(psim_out_t* out) {
    setup();
    plan_3way(g->n_pv, g->n_pr, p_v, p_r, n_vp, g->n_st, stage, &boxes);
    blocks.assign(g->n_pv, nullptr);
    bsums.assign(g->n_pv, nullptr);
    blocks[p_v] = own;
    bsums[p_v] = s_own;
    for (int d = 1; d < g->n_pv; ++d) {
      const int s = (p_v + d) % g->n_pv;
      blocks[s] = A.take(n_vp * ld * esz);
      bsums[s] = A.take(n_vp * esz);
    }
    for (const Box& b : boxes) {
      const int pairs[3][2] = {{b.A, b.B}, {b.A, b.C}, {b.B, b.C}};
      for (auto& xy : pairs)
        if (!std::any_of(tabs.begin(), tabs.end(),
                         [&](const Tab& t) { return t.X == xy[0] && t.Y == xy[1]; }))
          tabs.push_back({xy[0], xy[1], nullptr});
    }
    for (Tab& t : tabs) t.data = A.take(n_vp * n_vp * esz);
    if (g->n_pf > 1) tab_parts = A.take((int64_t)g->n_pf * n_vp * n_vp * esz);
    int64_t max_out = 0;
    for (const Box& b : boxes) {
      psim_box3_t s = box_struct(b, nullptr, false);
      int64_t no = 0, nt = 0;
      psim_box3_plan(dtype, &s, &no, &nt);
      n_out.push_back(no);
      max_out = std::max(max_out, no);
      psim_piece_t pc{};
      pc.kind = 3;
      pc.v[0] = b.i0;
      pc.v[1] = b.i1;
      pc.v[2] = b.j0;
      pc.v[3] = b.j1;
      pc.v[4] = b.k0;
      pc.v[5] = b.k1;
      int64_t e0 = 0, e1 = no;
      if (g->n_pf > 1) {
        e0 = no * p_f / g->n_pf;
        e1 = no * (p_f + 1) / g->n_pf;
      }
      pc.v[6] = e0;
      pc.v[7] = e1;
      pc.count = e1 - e0;
      pc.offset = n_vals;
      piece_of.push_back(-1);
      if (no > 0 && pc.count > 0) {
        piece_of.back() = (int)pieces.size();
        n_vals += pc.count;
        pieces.push_back(pc);
      }
    }
    local_count = n_vals;
    if (g->n_pf > 1) {
      part = A.take(max_out * esz);
      const int64_t mine = (max_out + g->n_pf - 1) / g->n_pf + 1;
      rbuf = A.take(mine * g->n_pf * esz);
      tot = A.take(mine * esz);
    }
    if (flags & PSIM_RUN_VALUES_SCRATCH) scratch = A.take(max_out * esz);
    (void)out;
    return true;
  }

  bool blocks_group() {
    if (g->n_pv == 1) return true;
    cudaStream_t cs = ctx->cstream;
    if (!gstart()) return false;
    for (int d = 1; d < g->n_pv; ++d) {
      const int to = rank_of(p_f, (p_v - d + g->n_pv) % g->n_pv, p_r);
      const int fs = (p_v + d) % g->n_pv;
      const int from = rank_of(p_f, fs, p_r);
      send(own, n_vp * ld * esz, to, cs, 0, n_fp * n_vp, PSIM_MSG_BLOCK, p_v);
      send(s_own, n_vp * esz, to, cs, 2, n_vp, PSIM_MSG_SUMS, p_v);
      recv(blocks[fs], n_vp * ld * esz, from, cs, PSIM_MSG_BLOCK, fs);
      recv(bsums[fs], n_vp * esz, from, cs, PSIM_MSG_SUMS, fs);
    }
    return gend();
  }

  bool table_group(size_t t, const void* mine) {
    return field_allgather(mine, tab_parts, n_vp * n_vp * esz, 4, n_vp * n_vp, PSIM_MSG_TABLE,
                           (int64_t)t);
  }

  std::vector<int64_t> box_offsets(size_t bi) const {
    std::vector<int64_t> off(g->n_pf + 1);
    for (int f = 0; f <= g->n_pf; ++f) off[f] = n_out[bi] * f / g->n_pf;
    return off;
  }

  // The comm schedule alone (psim_run_comms): execute()'s groups, in order.
  void comm_trace() {
    if (g->n_pf > 1) field_allgather(s_own, sum_parts, n_vp * esz, 2, n_vp, PSIM_MSG_SUMS, p_v);
    blocks_group();
    std::vector<bool> done(tabs.size(), false);
    for (size_t bi = 0; bi < boxes.size(); ++bi) {
      const Box& b = boxes[bi];
      for (size_t t = 0; t < tabs.size(); ++t) {
        const Tab& T = tabs[t];
        const bool used = (T.X == b.A && T.Y == b.B) || (T.X == b.A && T.Y == b.C) ||
                          (T.X == b.B && T.Y == b.C);
        if (!used || done[t]) continue;
        if (g->n_pf > 1) table_group(t, tab_parts);
        done[t] = true;
      }
      if (n_out[bi] == 0 || g->n_pf == 1) continue;
      field_scatter(part, rbuf, box_offsets(bi), 5, PSIM_MSG_BOX, (int64_t)bi);
    }
  }

  bool execute(psim_out_t* out) {
    if (!begin() || !load(false)) return false;
    if (validate && !S.cuda(psim::check_block(dtype, own, n_fp, n_vp, own_ld, dflags, st), "check"))
      return false;
    if (!sums()) return false;
    if (g->n_pv > 1 && (!S.cuda(cudaEventRecord(ev_tmp, st), "event") ||
                        !S.cuda(cudaStreamWaitEvent(ctx->cstream, ev_tmp, 0), "wait")))
      return false;
    // the block circulation (metrics3.py:93-109, face_j / vol_k / vol_j) as one
    // circulant all-gather of blocks and sums on the comm stream, overlapped
    // with the diagonal-edge boxes that need only the own block
    if (!blocks_group()) return false;
    bool gathered = g->n_pv == 1;
    std::vector<bool> tab_done(tabs.size(), false);
    for (size_t bi = 0; bi < boxes.size(); ++bi) {
      const Box& b = boxes[bi];
      if (!b.edge && !gathered) {
        if (!S.cuda(cudaEventRecord(ev_tmp, ctx->cstream), "event") ||
            !S.cuda(cudaStreamWaitEvent(st, ev_tmp, 0), "wait"))
          return false;
        gathered = true;
      }
      // numerator tables this box reads (2-way mGEMM of a block pair; with a
      // field split, every field rank's table folded in p_f order)
      for (size_t t = 0; t < tabs.size(); ++t) {
        const Tab& T = tabs[t];
        const bool used = (T.X == b.A && T.Y == b.B) || (T.X == b.A && T.Y == b.C) ||
                          (T.X == b.B && T.Y == b.C);
        if (!used || tab_done[t]) continue;
        void* dst = g->n_pf > 1 ? static_cast<char*>(tab_parts) + p_f * n_vp * n_vp * esz : T.data;
        if (!S.psim(psim_mgemm(dtype, blocks[T.X], ld, blocks[T.Y], ld, n_fp, n_vp, n_vp,
                               T.X == T.Y, dst, n_vp, 0, st)))
          return false;
        if (g->n_pf > 1) {
          if (!table_group(t, dst)) return false;
          if (!fold_parts(T.data, tab_parts, n_vp * n_vp)) return false;
        }
        tab_done[t] = true;
      }
      if (n_out[bi] == 0) continue;
      const psim_piece_t* pc = piece_of[bi] >= 0 ? &pieces[piece_of[bi]] : nullptr;
      void* vals = scratch ? scratch
                           : (out && out->vals && pc ? static_cast<char*>(out->vals) + pc->offset * esz
                                                     : nullptr);
      if (g->n_pf == 1) {
        psim_box3_t s = box_struct(b, vals, true);
        if (!kmark() || !S.psim(psim_czek3_box(dtype, &s, st)) || !kmark()) return false;
        if (scratch) {
          scratch_piece = piece_of[bi];
          scratch_vals = scratch;
        }
        continue;
      }
      // field split (metrics3.py:163-164): raw n_ijk of this slab, the ordered
      // reduce-scatter over the field group, then values for this rank's range
      psim_box3_t raw = box_struct(b, part, false);
      if (!kmark() || !S.psim(psim_czek3_box_numerators(dtype, &raw, st)) || !kmark()) return false;
      const std::vector<int64_t> off = box_offsets(bi);
      const int64_t mine = off[p_f + 1] - off[p_f];
      if (!field_scatter(part, rbuf, off, 5, PSIM_MSG_BOX, (int64_t)bi)) return false;
      if (mine == 0) continue;
      if (!fold_parts(tot, rbuf, mine)) return false;
      psim_box3_t s = box_struct(b, nullptr, true);
      if (!S.psim(psim_czek3_from_numerators(dtype, &s, tot, off[p_f], off[p_f + 1], vals, st)))
        return false;
    }
    if (!gathered && (!S.cuda(cudaEventRecord(ev_tmp, ctx->cstream), "event") ||
                      !S.cuda(cudaStreamWaitEvent(st, ev_tmp, 0), "wait")))
      return false;
    return S.ok();
  }
};

template <class R>
int plan_or_run(psim_ctx* ctx, const psim_problem_t* p, const psim_grid_t* g, int stage, int flags,
                void* ws, int64_t ws_bytes, psim_out_t* out, void* stream, psim_plan_t* plan,
                psim_piece_t* plan_pieces = nullptr, int64_t cap = 0,
                std::vector<psim_msg_t>* comms = nullptr) {
  R r;
  r.ctx = ctx;
  r.pr = p;
  r.g = g;
  r.flags = flags;
  r.st = static_cast<cudaStream_t>(stream);
  if constexpr (std::is_same<R, Run3>::value) r.stage = stage;
  // dry layout: sizes only
  r.A.dry = true;
  r.layout(out);
  if (comms) {  // the message schedule only
    r.trace = true;
    r.comm_trace();
    *comms = r.log;
    return PSIM_OK;
  }
  if (plan) {
    plan->n_pieces = (int64_t)r.pieces.size();
    plan->n_vals = r.n_vals;
    plan->workspace_bytes = r.A.off + 256;
    if (plan_pieces) {
      if (cap < plan->n_pieces)
        return set_error(PSIM_ECONFIG, "pieces capacity %lld < %lld", (long long)cap,
                         (long long)plan->n_pieces);
      std::copy(r.pieces.begin(), r.pieces.end(), plan_pieces);
    }
    return PSIM_OK;
  }
  if (r.A.off + 256 > ws_bytes || (!ws && r.A.off > 0))
    return set_error(PSIM_ECONFIG, "workspace of %lld bytes < the %lld this run needs",
                     (long long)ws_bytes, (long long)(r.A.off + 256));
  if (reinterpret_cast<uintptr_t>(ws) % 256)
    return set_error(PSIM_ECONFIG, "workspace must be 256-byte aligned");
  R run;
  run.ctx = ctx;
  run.pr = p;
  run.g = g;
  run.flags = flags;
  run.st = r.st;
  if constexpr (std::is_same<R, Run3>::value) run.stage = stage;
  run.A.dry = false;
  run.A.base = static_cast<char*>(ws);
  run.layout(out);
  if (run.A.off > ws_bytes) return set_error(PSIM_ECONFIG, "workspace too small");
  if (!run.execute(out)) return run.S.code;
  return run.finish(out, run.local_count);
}

}  // namespace

extern "C" {

int psim_nccl_unique_id(uint8_t* id) {
  if (!id) return set_error(PSIM_ECONFIG, "NULL id");
  const Nccl& N = nccl();
  if (N.error) return set_error(PSIM_ERUNTIME, "%s", N.error);
  ncclUniqueId u;
  ncclResult_t r = N.GetUniqueId(&u);
  if (r != ncclSuccess) return set_error(PSIM_ERUNTIME, "ncclGetUniqueId: %s", N.GetErrorString(r));
  static_assert(sizeof(u) == PSIM_NCCL_ID_BYTES, "NCCL unique id size");
  std::memcpy(id, &u, sizeof(u));
  return PSIM_OK;
}

int psim_ctx_create(int device, int rank, int world, const uint8_t* nccl_id, psim_ctx** out) {
  if (!out) return set_error(PSIM_ECONFIG, "NULL ctx pointer");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world)
    return set_error(PSIM_ECONFIG, "rank %d outside world %d", rank, world);
  if (device < 0) {  // planning-only context (psim_run_plan; no CUDA, no NCCL)
    psim_ctx* c = new psim_ctx;
    c->device = -1;
    c->rank = rank;
    c->world = world;
    *out = c;
    return PSIM_OK;
  }
  if (world > 1 && !nccl_id) return set_error(PSIM_ECONFIG, "world > 1 needs an NCCL unique id");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess)
    return set_error(PSIM_ERUNTIME, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  psim_ctx* c = new psim_ctx;
  c->device = device;
  c->rank = rank;
  c->world = world;
  Status S;
  S.cuda(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking), "comm stream");
  S.cuda(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking), "copy stream");
  c->pinned_len = 64 + (int64_t)world * 64;
  S.cuda(cudaHostAlloc(&c->pinned, c->pinned_len * 8, cudaHostAllocDefault), "pinned staging");
  if (S.ok() && world > 1) {
    const Nccl& N = nccl();
    if (N.error) {
      S.code = set_error(PSIM_ERUNTIME, "%s", N.error);
    } else {
      ncclUniqueId u;
      std::memcpy(&u, nccl_id, sizeof(u));
      S.nc(N.CommInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
    }
  }
  if (!S.ok()) {
    psim_ctx_destroy(c);
    return S.code;
  }
  *out = c;
  return PSIM_OK;
}

int psim_ctx_destroy(psim_ctx* c) {
  if (!c) return PSIM_OK;
  if (c->comm) nccl().CommDestroy(c->comm);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->pinned) cudaFreeHost(c->pinned);
  delete c;
  return PSIM_OK;
}

int psim_run_plan(const psim_ctx* ctx, const psim_problem_t* p, const psim_grid_t* g, int stage,
                  int flags, psim_plan_t* plan) {
  return psim_run_pieces(ctx, p, g, stage, flags, plan, nullptr, 0);
}

int psim_run_pieces(const psim_ctx* ctx, const psim_problem_t* p, const psim_grid_t* g, int stage,
                    int flags, psim_plan_t* plan, psim_piece_t* pieces, int64_t cap) {
  if (!plan) return set_error(PSIM_ECONFIG, "NULL plan");
  if (int r = check_common(ctx, p, g, p ? p->arity : 0)) return r;
  if (p->arity != 2 && p->arity != 3) return set_error(PSIM_ECONFIG, "arity must be 2 or 3");
  if (p->arity == 3 && (stage < -1 || stage >= g->n_st))
    return set_error(PSIM_ECONFIG, "stage %d outside [0, %d)", stage, g->n_st);
  psim_ctx* c = const_cast<psim_ctx*>(ctx);
  return p->arity == 2
             ? plan_or_run<Run2>(c, p, g, -1, flags, nullptr, 0, nullptr, nullptr, plan, pieces, cap)
             : plan_or_run<Run3>(c, p, g, stage, flags, nullptr, 0, nullptr, nullptr, plan, pieces,
                                 cap);
}

int psim_run_comms(const psim_ctx* ctx, const psim_problem_t* p, const psim_grid_t* g, int stage,
                   int flags, psim_msg_t* msgs, int64_t cap, int64_t* n) {
  if (!n) return set_error(PSIM_ECONFIG, "NULL count");
  if (int r = check_common(ctx, p, g, p ? p->arity : 0)) return r;
  if (p->arity != 2 && p->arity != 3) return set_error(PSIM_ECONFIG, "arity must be 2 or 3");
  if (p->arity == 3 && (stage < -1 || stage >= g->n_st))
    return set_error(PSIM_ECONFIG, "stage %d outside [0, %d)", stage, g->n_st);
  std::vector<psim_msg_t> log;
  psim_ctx* c = const_cast<psim_ctx*>(ctx);
  const int r = p->arity == 2
                    ? plan_or_run<Run2>(c, p, g, -1, flags, nullptr, 0, nullptr, nullptr, nullptr,
                                        nullptr, 0, &log)
                    : plan_or_run<Run3>(c, p, g, stage, flags, nullptr, 0, nullptr, nullptr,
                                        nullptr, nullptr, 0, &log);
  if (r) return r;
  *n = (int64_t)log.size();
  if (msgs) std::copy(log.begin(), log.begin() + std::min<int64_t>(cap, *n), msgs);
  return PSIM_OK;
}

int psim_run2(psim_ctx* ctx, const psim_problem_t* p, const psim_grid_t* g, int flags, void* ws,
              int64_t ws_bytes, psim_out_t* out, void* stream) {
  if (int r = check_common(ctx, p, g, 2)) return r;
  if (!out) return set_error(PSIM_ECONFIG, "NULL out");
  if (ctx->device < 0) return set_error(PSIM_ECONFIG, "planning-only context (device -1)");
  if (ctx->world > 1 && nccl().error) return set_error(PSIM_ERUNTIME, "%s", nccl().error);
  cudaSetDevice(ctx->device);
  return plan_or_run<Run2>(ctx, p, g, -1, flags, ws, ws_bytes, out, stream, nullptr);
}

int psim_run3(psim_ctx* ctx, const psim_problem_t* p, const psim_grid_t* g, int stage, int flags,
              void* ws, int64_t ws_bytes, psim_out_t* out, void* stream) {
  if (int r = check_common(ctx, p, g, 3)) return r;
  if (!out) return set_error(PSIM_ECONFIG, "NULL out");
  if (ctx->device < 0) return set_error(PSIM_ECONFIG, "planning-only context (device -1)");
  if (stage < -1 || stage >= g->n_st)
    return set_error(PSIM_ECONFIG, "stage %d outside [0, %d)", stage, g->n_st);
  if (ctx->world > 1 && nccl().error) return set_error(PSIM_ERUNTIME, "%s", nccl().error);
  cudaSetDevice(ctx->device);
  return plan_or_run<Run3>(ctx, p, g, stage, flags, ws, ws_bytes, out, stream, nullptr);
}

int psim_malloc(void** ptr, int64_t bytes, int pinned_host) {
  if (!ptr || bytes < 0) return set_error(PSIM_ECONFIG, "bad allocation request");
  *ptr = nullptr;
  if (bytes == 0) return PSIM_OK;
  cudaError_t e = pinned_host ? cudaHostAlloc(ptr, bytes, cudaHostAllocDefault)
                              : cudaMalloc(ptr, bytes);
  if (e != cudaSuccess)
    return set_error(PSIM_ERUNTIME, "allocation of %lld bytes failed: %s", (long long)bytes,
                     cudaGetErrorString(e));
  return PSIM_OK;
}

int psim_free(void* ptr, int pinned_host) {
  if (!ptr) return PSIM_OK;
  cudaError_t e = pinned_host ? cudaFreeHost(ptr) : cudaFree(ptr);
  return e == cudaSuccess ? PSIM_OK : set_error(PSIM_ERUNTIME, "free: %s", cudaGetErrorString(e));
}

int psim_memcpy(void* dst, const void* src, int64_t bytes) {
  if (bytes < 0 || (bytes && (!dst || !src))) return set_error(PSIM_ECONFIG, "bad copy");
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
  return e == cudaSuccess ? PSIM_OK : set_error(PSIM_ERUNTIME, "copy: %s", cudaGetErrorString(e));
}

int psim_checksum(int dtype, const void* vals, const int64_t* idx, int64_t idx0, int64_t count,
                  unsigned long long* acc, void* stream) {
  if (dtype != psim::kF32 && dtype != psim::kF64) return set_error(PSIM_ECONFIG, "bad dtype");
  if (count < 0 || (count && (!vals || !acc))) return set_error(PSIM_ECONFIG, "bad arguments");
  cudaError_t e = psim::checksum(dtype, vals, idx, idx0, count, acc, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_error(PSIM_ERUNTIME, "psim_checksum: %s", cudaGetErrorString(e));
  return PSIM_OK;
}

}  // extern "C"
