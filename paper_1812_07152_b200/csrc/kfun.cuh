// kfun.cuh — the kernel functions K(x, y) on the device (kernel.cpp:35-49), shared by the
// generated near field (kernels.cuh), the error oracle (krows.cu) and the GPU compression
// (compress.cu).
#pragma once

#include <cstdint>

#include "../../include/hmxg.h"

namespace hmxg {
namespace {

struct KernelParams {
  int kind;
  std::uint32_t d;
  double den;   // gaussian: 2 h h, formed as (2.0 * h) * h like kernel.cpp:42
  double invh;  // exponential: 1 / h
};

// K given the squared distance s, with the reference's operation order (kernel.cpp:42-47).
__device__ __forceinline__ double kernel_of_sqdist(const KernelParams& kp, double s) {
  if (kp.kind == HMXG_KERNEL_GAUSSIAN) return exp(__ddiv_rn(-s, kp.den));
  if (kp.kind == HMXG_KERNEL_EXPONENTIAL) return exp(__dmul_rn(-__dsqrt_rn(s), kp.invh));
  return s == 0.0 ? 1.0 : __ddiv_rn(1.0, __dsqrt_rn(s));
}
// K(x, y) with the reference's operation order: the squared distance accumulates the
// rounded products dimension by dimension (no FMA contraction, kernel.cpp:37-41).
__device__ __forceinline__ double kernel_value(const KernelParams& kp, const double* __restrict__ x,
                                               const double* __restrict__ y) {
  double s = 0.0;
  for (std::uint32_t i = 0; i < kp.d; ++i) {
    const double t = __dsub_rn(__ldg(x + i), __ldg(y + i));
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return kernel_of_sqdist(kp, s);
}

}  // namespace
}  // namespace hmxg
