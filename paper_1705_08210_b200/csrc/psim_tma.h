// Host side of TMA staging (minplus.cuh: minplus_tile_tma /
// minplus_tile_pivot_ilv): tensor maps of the vector blocks. The encoder
// comes from the driver through the runtime (no libcuda link);
// PSIM_NO_TMA=1 keeps the cp.async loaders (read per launch, for A/B runs).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

namespace psim {

// TMA staging on unless PSIM_NO_TMA=1 (read per launch, so tests can A/B it).
inline bool tma_enabled() {
  const char* v = getenv("PSIM_NO_TMA");
  return !(v && v[0] == '1');
}

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return f;
  }();
  return fn;
}

template <typename T>
inline bool encode_operand(CUtensorMap* map, const T* base, int64_t n_f, int64_t vectors,
                           int64_t ld, int box_rows, int pitch) {
  auto enc = tma_encoder();
  if (!enc || !base || vectors < 1 || n_f < 1 || n_f >= (1ll << 31) || vectors >= (1ll << 31))
    return false;
  const cuuint64_t dims[2] = {(cuuint64_t)n_f, (cuuint64_t)vectors};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * (int64_t)sizeof(T))};
  const cuuint32_t box[2] = {(cuuint32_t)pitch, (cuuint32_t)box_rows}, es[2] = {1, 1};
  return enc(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
             2, const_cast<T*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace psim
