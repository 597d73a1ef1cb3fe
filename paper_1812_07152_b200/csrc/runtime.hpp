// runtime.hpp — host-side helpers shared by the translation units of libhmxg.so: the
// thread-local error message behind hmxg_last_error, CUDA status mapping, device upload
// and TMA descriptor encoding.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hmxg.h"

struct hmxg_ctx {
  std::vector<int> devs;
  hmxg_comm comm{};  // size 0: no communicator (hmxg_create)
};

namespace hmxg {

inline thread_local std::string g_err;

inline int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

inline int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear non-sticky errors
  return set_err(e == cudaErrorMemoryAllocation ? HMXG_ENOMEM : HMXG_ECUDA,
                 std::string(what) + ": " + cudaGetErrorString(e));
}

#define HMXG_CUDA(call)                                 \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

#define HMXG_TRY(call)              \
  do {                              \
    int rc_ = (call);               \
    if (rc_ != HMXG_OK) return rc_; \
  } while (0)

template <class T>
int dev_upload(T** dst, const T* src, std::size_t count, cudaStream_t st) {
  *dst = nullptr;
  if (count == 0) return HMXG_OK;
  HMXG_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), count * sizeof(T)));
  HMXG_CUDA(cudaMemcpyAsync(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return HMXG_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D map over a point-major buffer (rows x cols, cols contiguous, row pitch ld doubles):
// boxes of box_rows rows x box_cols columns, no swizzle, zero fill outside.
inline int make_map_box(CUtensorMap* map, const double* base, std::uint64_t rows, std::uint64_t cols,
                        std::uint64_t ld, std::uint32_t box_cols, std::uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_err(HMXG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * sizeof(double)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(HMXG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return HMXG_OK;
}

}  // namespace hmxg
