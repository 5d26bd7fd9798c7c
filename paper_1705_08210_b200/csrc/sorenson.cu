// Sorenson (0/1 data) 2-way path: bit-packed vectors, AND + POPC mainloop
// (SURVEY 8f, row f3).
//
// Reference: pack_bits (mingemm.py:279-291) packs each 0/1 column into
// 64-bit words; mgemm_bitpacked (mingemm.py:294-312) counts popcount(a & b)
// per column pair; run_2way converts the counts to the run dtype and applies
// the Czekanowski expression (metrics2.py:126-129, 85-89). On 0/1 data the
// count equals sum_q min(a_q, b_q) exactly, so values and checksums equal the
// dense kernel's bit for bit (pinned by test_acceptance.py:240-257).
//
// Here 32 fields share one uint32 word; the min-plus tiling / cp.async
// pipeline of minplus.cuh is reused with T = uint32_t, and one LDS.128 brings
// 128 fields: the mainloop costs LOP3 + POPC + IADD per 32 comparisons.
#include "minplus.cuh"
#include "psim_internal.h"

namespace psim {

// POPC-bound (16 per clock per SM): a 128 x 64 tile at 2 CTAs/SM keeps the
// register budget at 128 without spills.
using CfgBits = Cfg<uint32_t, 8, 4, 3, 2, 0>;

template <typename VT>
struct SorArgs {
  const uint32_t* W;  // packed words, column i at W + i*ldw
  int64_t ldw;
  const uint32_t* V;
  int64_t ldv;
  int64_t n_words;
  int64_t m, n;
  int diagonal;
  const VT* s_row;
  const VT* s_col;
  int64_t g_row, g_col, n_v;
  VT* out;
  unsigned long long* acc;
  int64_t tiles_m, tiles_n, band, nbands;
  const int64_t* row_pref;
};

template <typename VT>
__global__ void __launch_bounds__(kNT, CfgBits::MINB) k_sorenson2(const SorArgs<VT> a) {
  using C = CfgBits;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* smem = reinterpret_cast<uint32_t*>(smem_raw);
  int bi, bj;
  if (!band_tile((int64_t)blockIdx.x, a.row_pref, a.nbands, a.band, 0, a.tiles_m, C::BM, C::BN,
                 a.diagonal, bi, bj))
    return;
  const int64_t row0 = (int64_t)bi * C::BM, col0 = (int64_t)bj * C::BN;
  const int rows = (int)min64(C::BM, a.m - row0);
  const int cols = (int)min64(C::BN, a.n - col0);
  uint32_t acc[C::TM][C::TN];
  minplus_tile<C, false>(a.W + row0 * a.ldw, a.ldw, rows, a.V + col0 * a.ldv, a.ldv, cols,
                         nullptr, a.n_words, acc, smem);
  const int ty = thread_ty(), tx = thread_tx();
  Cks c;
#pragma unroll
  for (int mi = 0; mi < C::TM; ++mi) {
    const int li = ty + 16 * mi;
    if (li >= rows) continue;
    const int64_t i = row0 + li;
    const VT si = a.s_row[i];
    const uint64_t gi = (uint64_t)(a.g_row + i);
#pragma unroll
    for (int nj = 0; nj < C::TN; ++nj) {
      const int lj = tx + 16 * nj;
      const int64_t j = col0 + lj;
      if (lj >= cols || (a.diagonal && j <= i)) continue;
      const VT num = (VT)acc[mi][nj];  // int -> dt, round to nearest (numpy astype)
      const VT d = Traits<VT>::add(si, a.s_col[j]);
      const bool zero = (d == VT(0));
      const VT v = zero ? VT(0) : Traits<VT>::div(Traits<VT>::mul(VT(2), num), d);
      if (a.out) a.out[a.diagonal ? (int64_t)pair_index(i, j, a.m) : i * a.n + j] = v;
      const uint64_t gj = (uint64_t)(a.g_col + j);
      const uint64_t gidx = gi < gj ? pair_index(gi, gj, a.n_v) : pair_index(gj, gi, a.n_v);
      c.term(gidx, Traits<VT>::bits(v));
      c.deg += zero ? 1ull : 0ull;
    }
  }
  cks_block_flush<kNT>(a.acc, c);
}

// Bit packing with validation (pack_bits, mingemm.py:279-291): one warp per
// 32-field chunk of a vector; flags[0] += count of entries outside {0, 1}.
template <typename T>
__global__ void __launch_bounds__(256) k_pack_bits(const T* __restrict__ V, int64_t n_fp,
                                                   int64_t n_vp, int64_t ld,
                                                   uint32_t* __restrict__ words, int64_t ldw,
                                                   unsigned long long* flags) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (n_fp + 31) / 32;
  const int64_t total = nw * n_vp;
  unsigned long long bad = 0;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < total;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t v = w / nw, wq = w - v * nw;
    const int64_t q = wq * 32 + lane;
    T x = T(0);
    if (q < n_fp) x = V[v * ld + q];
    bad += (x == T(0) || x == T(1)) ? 0 : 1;
    const uint32_t bits = __ballot_sync(0xffffffffu, x == T(1));
    if (lane == 0) words[v * ldw + wq] = bits;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, o);
  if (lane == 0 && bad) atomicAdd(flags, bad);
}

cudaError_t pack_bits(int dtype, const void* V, int64_t n_fp, int64_t n_vp, int64_t ld,
                      uint32_t* words, int64_t ldw, unsigned long long* flags, cudaStream_t st) {
  if (n_fp <= 0 || n_vp <= 0) return cudaSuccess;
  int64_t warps = ((n_fp + 31) / 32) * n_vp;
  int64_t blocks = (warps + 7) / 8;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (dtype == kF64) {
    note_launch();
    k_pack_bits<double><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const double*>(V), n_fp,
                                                          n_vp, ld, words, ldw, flags);
  } else {
    note_launch();
    k_pack_bits<float><<<(unsigned)blocks, 256, 0, st>>>(static_cast<const float*>(V), n_fp,
                                                         n_vp, ld, words, ldw, flags);
  }
  return cudaGetLastError();
}

__host__ __device__ __forceinline__ int64_t band_count_s(int64_t b, int64_t G, int64_t tiles_m,
                                                         int64_t tiles_n, int diagonal) {
  const int64_t r0 = b * G;
  const int64_t rows = min64(G, tiles_m - r0);
  return rows * max64(0, tiles_n - first_col_tile(r0, CfgBits::BM, CfgBits::BN, diagonal));
}

__global__ void k_band_prefix_s(int64_t nbands, int64_t G, int64_t tiles_m, int64_t tiles_n,
                                int diagonal, int64_t* pref) {
  if (threadIdx.x != 0) return;  // nbands is small (<= a few hundred)
  int64_t run = 0;
  for (int64_t b = 0; b < nbands; ++b) {
    pref[b] = run;
    run += band_count_s(b, G, tiles_m, tiles_n, diagonal);
  }
  pref[nbands] = run;
}

template <typename VT>
static cudaError_t sorenson_t(const psim_block2_t& t, cudaStream_t st) {
  using C = CfgBits;
  SorArgs<VT> a{};
  a.W = static_cast<const uint32_t*>(t.W);
  a.ldw = t.ldw;
  a.V = static_cast<const uint32_t*>(t.V);
  a.ldv = t.ldv;
  a.n_words = (t.n_f + 31) / 32;
  a.m = t.m;
  a.n = t.n;
  a.diagonal = t.diagonal;
  a.s_row = static_cast<const VT*>(t.s_row);
  a.s_col = static_cast<const VT*>(t.s_col);
  a.g_row = t.g_row;
  a.g_col = t.g_col;
  a.n_v = t.n_v;
  a.out = static_cast<VT*>(t.vals);
  a.acc = t.acc;
  if (a.m <= 0 || a.n <= 0) return cudaSuccess;
  a.tiles_m = (a.m + C::BM - 1) / C::BM;
  a.tiles_n = (a.n + C::BN - 1) / C::BN;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  a.band = (int64_t)(sqrt((double)sms) + 0.5);
  a.nbands = (a.tiles_m + a.band - 1) / a.band;
  int64_t blocks = 0;
  for (int64_t b = 0; b < a.nbands; ++b)
    blocks += band_count_s(b, a.band, a.tiles_m, a.tiles_n, a.diagonal);
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(k_sorenson2<VT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int64_t* pref = nullptr;
  e = cudaMallocAsync(&pref, (a.nbands + 1) * sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  note_launch();
  k_band_prefix_s<<<1, 32, 0, st>>>(a.nbands, a.band, a.tiles_m, a.tiles_n, a.diagonal, pref);
  a.row_pref = pref;
  note_launch();
  k_sorenson2<VT><<<(unsigned)blocks, kNT, C::SMEM_BYTES, st>>>(a);
  e = cudaGetLastError();
  cudaError_t e2 = cudaFreeAsync(pref, st);
  return e != cudaSuccess ? e : e2;
}

// Raw counts (mgemm_bitpacked itself, mingemm.py:294-312): M[i + j*ldm] =
// sum over words of popc(W_i & V_j), int64, column-major; the kernel
// plug-point form (no epilogue), row-major tile order.
__global__ void __launch_bounds__(kNT, CfgBits::MINB)
    k_mgemm_bits(const uint32_t* __restrict__ W, int64_t ldw, const uint32_t* __restrict__ V,
                 int64_t ldv, int64_t n_words, int64_t m, int64_t n, int64_t tiles_n,
                 long long* __restrict__ M, int64_t ldm) {
  using C = CfgBits;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* smem = reinterpret_cast<uint32_t*>(smem_raw);
  const int64_t bi = blockIdx.x / tiles_n, bj = blockIdx.x - bi * tiles_n;
  const int64_t row0 = bi * C::BM, col0 = bj * C::BN;
  const int rows = (int)min64(C::BM, m - row0), cols = (int)min64(C::BN, n - col0);
  uint32_t acc[C::TM][C::TN];
  minplus_tile<C, false>(W + row0 * ldw, ldw, rows, V + col0 * ldv, ldv, cols, nullptr, n_words,
                         acc, smem);
  const int ty = thread_ty(), tx = thread_tx();
#pragma unroll
  for (int mi = 0; mi < C::TM; ++mi) {
    const int li = ty + 16 * mi;
#pragma unroll
    for (int nj = 0; nj < C::TN; ++nj) {
      const int lj = tx + 16 * nj;
      if (li < rows && lj < cols) M[(row0 + li) + (col0 + lj) * ldm] = (long long)acc[mi][nj];
    }
  }
}

cudaError_t mgemm_bits(const uint32_t* W, int64_t ldw, const uint32_t* V, int64_t ldv,
                       int64_t n_rows, int64_t m, int64_t n, long long* M, int64_t ldm,
                       cudaStream_t st) {
  using C = CfgBits;
  if (m <= 0 || n <= 0) return cudaSuccess;
  const int64_t tiles_n = (n + C::BN - 1) / C::BN;
  const int64_t blocks = ((m + C::BM - 1) / C::BM) * tiles_n;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(k_mgemm_bits, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  note_launch();
  k_mgemm_bits<<<(unsigned)blocks, kNT, C::SMEM_BYTES, st>>>(W, ldw, V, ldv, (n_rows + 31) / 32,
                                                             m, n, tiles_n, M, ldm);
  return cudaGetLastError();
}

cudaError_t sorenson2_block(int dtype, const psim_block2_t& t, cudaStream_t st) {
  return dtype == kF64 ? sorenson_t<double>(t, st) : sorenson_t<float>(t, st);
}

}  // namespace psim
