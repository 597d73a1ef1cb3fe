// kernels.cuh — sm_100a kernels of the evaluator.
//
//  * grouped_gemm<TRANS_A>: one CTA per (output row tile, 64-column block); its K loop runs
//    over the tile's segment list, so a whole far+downward sum or a whole leaf row
//    (V_i S_i + sum_j D_ij Wp_j) is accumulated in registers and stored once.
//    FP64 math on the tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; tcgen05 has no
//    f64 kind). Operands are staged global->shared by a 3-stage cp.async ring
//    with zero-fill for ragged M/K/N edges (two-means leaves of 15..256 points).
//  * gather_rows / scatter_rows: the permutation into and out of tree order
//    (executor.cpp:35-39, :245-254); coalesced along the output, the scattered side is a
//    per-column gather that stays L2 resident.
#pragma once

#include <cstdint>

#include "plan.hpp"

namespace hmxg {

constexpr int kBM = 64;       // output rows per CTA tile
constexpr int kBN = 64;       // output columns per CTA tile
constexpr int kBK = 16;       // K chunk per pipeline stage
constexpr int kStages = 3;
constexpr int kThreads = 128; // 4 warps, 2 x 2 warp grid of 32 x 32 warp tiles
constexpr int kAStrideN = kBM + 8;  // A stored [k][r] (non-transposed A)
constexpr int kAStrideT = kBK + 4;  // A stored [r][k] (transposed A)
constexpr int kBStride = kBK + 4;   // B stored [n][k]
constexpr int kAStageElems = (kBK * kAStrideN > kBM * kAStrideT) ? kBK * kAStrideN : kBM * kAStrideT;
constexpr int kBStageElems = kBN * kBStride;
constexpr int kSmemBytes = kStages * (kAStageElems + kBStageElems) * 8;

struct EvalParams {
  const double* gen[3];        // D, B, V generator bases
  double* buf[kNumBufs];       // Wp, T, S, Yp
  std::uint64_t ld[kNumBufs];  // leading dimensions
  const Task* tasks;           // first task of the phase
  const Seg* segs;
  std::uint32_t q;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Uniform selects instead of dynamic indexing into the parameter arrays (which would
// copy them to local memory).
__device__ __forceinline__ const double* pick_gen(const EvalParams& p, unsigned g) {
  return g == kGenD ? p.gen[kGenD] : (g == kGenB ? p.gen[kGenB] : p.gen[kGenV]);
}
__device__ __forceinline__ double* pick_buf(const EvalParams& p, unsigned b) {
  return b == kBufWp ? p.buf[kBufWp] : (b == kBufT ? p.buf[kBufT] : (b == kBufS ? p.buf[kBufS] : p.buf[kBufYp]));
}
__device__ __forceinline__ std::uint64_t pick_ld(const EvalParams& p, unsigned b) {
  return b == kBufWp ? p.ld[kBufWp] : (b == kBufT ? p.ld[kBufT] : (b == kBufS ? p.ld[kBufS] : p.ld[kBufYp]));
}

template <bool TRANS_A>
__global__ void __launch_bounds__(kThreads) grouped_gemm(EvalParams p) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                                // kStages * kAStageElems
  double* Bs = smem + kStages * kAStageElems;       // kStages * kBStageElems

  const Task task = p.tasks[blockIdx.x];
  const std::uint32_t c0 = blockIdx.y * kBN;
  const std::uint32_t ncols = min(static_cast<std::uint32_t>(kBN), p.q - c0);
  const int m = task.m;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;

  // number of K chunks over all segments
  int nchunks = 0;
  for (std::uint32_t s = task.seg_begin; s < task.seg_end; ++s)
    nchunks += (p.segs[s].k + kBK - 1) / kBK;

  // loader cursor
  std::uint32_t ls = task.seg_begin;
  std::uint32_t lk = 0;
  auto load_stage = [&](int stage) {
    if (ls < task.seg_end) {
      const Seg sg = p.segs[ls];
      const double* a = pick_gen(p, sg.gen) + sg.a_off;
      const std::uint64_t ldb = pick_ld(p, sg.bbuf);
      const double* b = pick_buf(p, sg.bbuf) + sg.b_row + static_cast<std::uint64_t>(c0) * ldb;
      const int kr = min(kBK, static_cast<int>(sg.k - lk));
      double* as = As + stage * kAStageElems;
      double* bs = Bs + stage * kBStageElems;
      if (TRANS_A) {
        // A(r,k) = a[k + r*lda]; contiguous along k -> store [r][k]
        const int k = tid % kBK;
#pragma unroll
        for (int j = 0; j < (kBM * kBK) / kThreads; ++j) {
          const int r = tid / kBK + j * (kThreads / kBK);
          const bool ok = r < m && k < kr;
          cp_async8(as + r * kAStrideT + k, ok ? a + (lk + k) + static_cast<std::uint64_t>(r) * sg.lda : a, ok);
        }
      } else {
        // A(r,k) = a[r + k*lda]; contiguous along r -> store [k][r]
        const int r = tid % kBM;
#pragma unroll
        for (int j = 0; j < (kBM * kBK) / kThreads; ++j) {
          const int k = tid / kBM + j * (kThreads / kBM);
          const bool ok = r < m && k < kr;
          cp_async8(as + k * kAStrideN + r, ok ? a + r + static_cast<std::uint64_t>(lk + k) * sg.lda : a, ok);
        }
      }
      {
        const int k = tid % kBK;
#pragma unroll
        for (int j = 0; j < (kBN * kBK) / kThreads; ++j) {
          const int n = tid / kBK + j * (kThreads / kBK);
          const bool ok = k < kr && n < static_cast<int>(ncols);
          cp_async8(bs + n * kBStride + k, ok ? b + (lk + k) + static_cast<std::uint64_t>(n) * ldb : b, ok);
        }
      }
      lk += kBK;
      if (lk >= sg.k) {
        ++ls;
        lk = 0;
      }
    }
    cp_async_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) load_stage(st);

  for (int it = 0; it < nchunks; ++it) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int stage = it % kStages;
    const double* as = As + stage * kAStageElems;
    const double* bs = Bs + stage * kBStageElems;
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = wm * 32 + i * 8 + (lane >> 2);
        const int k = kk + (lane & 3);
        af[i] = TRANS_A ? as[r * kAStrideT + k] : as[k * kAStrideN + r];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn * 32 + j * 8 + (lane >> 2);
        bf[j] = bs[n * kBStride + kk + (lane & 3)];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j], af[i], bf[j]);
    }
    load_stage((it + kStages - 1) % kStages);
  }
  cp_async_wait<0>();

  // epilogue: every element of the tile is stored exactly once (zeros for empty tasks)
  double* C = pick_buf(p, task.cbuf);
  const std::uint64_t ldc = pick_ld(p, task.cbuf);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = wm * 32 + i * 8 + (lane >> 2);
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = wn * 32 + j * 8 + 2 * (lane & 3);
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (col + e < static_cast<int>(ncols))
          C[task.c_row + row + static_cast<std::uint64_t>(c0 + col + e) * ldc] = acc[i][j][e];
    }
  }
}

// Wp[pos, c] = W[perm[pos], c]
__global__ void gather_rows(const double* __restrict__ w, std::uint64_t ldw,
                            const std::uint32_t* __restrict__ perm, double* __restrict__ wp,
                            std::uint64_t ldwp, std::uint32_t n, std::uint32_t q) {
  const std::uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const std::uint32_t src = perm[pos];
  for (std::uint32_t c = blockIdx.y; c < q; c += gridDim.y)
    wp[pos + c * ldwp] = w[src + c * ldw];
}

// Y[r, c] = Yp[iperm[r], c]  (== Y[perm[pos], c] = Yp[pos, c])
__global__ void scatter_rows(const double* __restrict__ yp, std::uint64_t ldyp,
                             const std::uint32_t* __restrict__ iperm, double* __restrict__ y,
                             std::uint64_t ldy, std::uint32_t n, std::uint32_t q) {
  const std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const std::uint32_t src = iperm[r];
  for (std::uint32_t c = blockIdx.y; c < q; c += gridDim.y)
    y[r + c * ldy] = yp[src + c * ldyp];
}

}  // namespace hmxg
