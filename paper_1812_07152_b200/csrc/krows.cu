// krows.cu — exact kernel products on the B200: the GPU error oracle.
//
// dense_apply (/root/reference/proj/src/executor.cpp:405-429) builds K in 256-row blocks
// on the host and multiplies each block into W; relative_error_vs (:431-476) compares an
// evaluation against exact rows of K W, densely (n <= 16384) or on 256 sampled rows.
// Here the same products run as
//
//   permute_in   Wt = W, point-major (the evaluator's transpose kernel, identity order)
//   gen_ktiles   A chunks K(x_rows, x_j), generated from the points straight into the
//                swizzled 64 x 16 chunk layout the GEMM streams (the kernel matrix is
//                never read from the host; per row block it lives in HBM once)
//   grouped_gemm the evaluator's FP64 DMMA GEMM, split over K (the point index j) so a
//                few hundred sampled rows still fill every SM
//   reduce       the K splits summed in a fixed order and transposed back to column
//                major (deterministic: no atomics)
//
// and the error sums in one deterministic reduction kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/hmxg.h"
#include "kernels.cuh"
#include "runtime.hpp"

namespace hmxg {
namespace {

// A chunks of K(x_rows, x_all) for one block of output rows: chunk c = (row tile t, K
// chunk kc) holds A(r, k) = K(x_{row(t*64+r)}, x_{kc*16+k}) at a_swz(k, r), zero outside.
__global__ void __launch_bounds__(256) gen_ktiles(const double* __restrict__ pts, const KernelParams kp,
                                                  const std::uint32_t* __restrict__ rows, std::uint64_t row0,
                                                  std::uint32_t nrows, std::uint32_t nkc, std::uint32_t n,
                                                  double* __restrict__ tiles, std::uint64_t nchunks) {
  for (std::uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const std::uint32_t t = static_cast<std::uint32_t>(c / nkc), kc = static_cast<std::uint32_t>(c % nkc);
    double* out = tiles + c * kChunkElems;
    for (int e = threadIdx.x; e < kChunkElems; e += blockDim.x) {
      const int r = e % kBM, k = e / kBM;  // a warp: 32 rows against one point j
      const std::uint32_t i = t * kBM + r, j = kc * kBK + k;
      double v = 0.0;
      if (i < nrows && j < n) {
        const std::uint64_t pi = rows ? rows[row0 + i] : row0 + i;
        v = kernel_value(kp, pts + pi * kp.d, pts + static_cast<std::uint64_t>(j) * kp.d);
      }
      out[a_swz(k, r)] = v;
    }
  }
}

// Y[r, c] = sum_s part[s*split_rows + r, c] (s ascending; column c at phys_col(c)),
// point-major -> column major.
__global__ void __launch_bounds__(256) reduce_splits(const double* __restrict__ part, std::uint64_t ldp,
                                                     std::uint32_t splits, std::uint64_t split_rows,
                                                     double* __restrict__ y, std::uint64_t ldy, std::uint32_t nrows,
                                                     std::uint32_t q) {
  __shared__ double tile[kTT][kTT + 1];
  const std::uint32_t r0 = blockIdx.x * kTT, c0 = blockIdx.y * kTT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + ty + k, c = c0 + tx;
    double v = 0.0;
    if (r < nrows && c < q)
      for (std::uint32_t s = 0; s < splits; ++s) v += part[(s * split_rows + r) * ldp + phys_col(c)];
    tile[ty + k][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + tx, c = c0 + ty + k;
    if (r < nrows && c < q) y[r + static_cast<std::uint64_t>(c) * ldy] = tile[tx][ty + k];
  }
}

// out[i + c*nrows] = ya[rows[i] + c*ldya]
__global__ void gather_rows(const double* __restrict__ ya, std::uint64_t ldya, const std::uint32_t* __restrict__ rows,
                            std::uint32_t nrows, std::uint32_t q, double* __restrict__ out) {
  const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<std::uint64_t>(nrows) * q) return;
  const std::uint32_t i = static_cast<std::uint32_t>(idx % nrows), c = static_cast<std::uint32_t>(idx / nrows);
  out[idx] = ya[rows[i] + static_cast<std::uint64_t>(c) * ldya];
}

// Per-block partial sums of (ya - acc)^2 and acc^2 over nrows x q entries, each block in a
// fixed order (grid-stride, then a shared-memory tree): deterministic for a fixed grid.
constexpr unsigned kErrBlocks = 592, kErrThreads = 256;
__global__ void __launch_bounds__(kErrThreads) err_sums(const double* __restrict__ ya, std::uint64_t ldya,
                                                        const double* __restrict__ acc, std::uint64_t lda,
                                                        std::uint64_t nrows, std::uint64_t q,
                                                        double* __restrict__ partial) {
  __shared__ double sn[kErrThreads], sd[kErrThreads];
  double num = 0.0, den = 0.0;
  const std::uint64_t total = nrows * q;
  for (std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(kErrThreads) + threadIdx.x; idx < total;
       idx += static_cast<std::uint64_t>(gridDim.x) * kErrThreads) {
    const std::uint64_t r = idx % nrows, c = idx / nrows;
    const double a = acc[r + c * lda];
    const double diff = ya[r + c * ldya] - a;
    num += diff * diff;
    den += a * a;
  }
  sn[threadIdx.x] = num;
  sd[threadIdx.x] = den;
  __syncthreads();
  for (unsigned w = kErrThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sn[threadIdx.x] += sn[threadIdx.x + w];
      sd[threadIdx.x] += sd[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = sn[0];
    partial[2 * blockIdx.x + 1] = sd[0];
  }
}

// hmx::mix64 / hmx::Rng (proj/include/hmx/rng.hpp:9-41): splitmix64 and xoshiro256**.
std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
struct Xoshiro {
  std::uint64_t s[4];
  explicit Xoshiro(std::uint64_t seed) {
    std::uint64_t x = seed;
    for (auto& si : s) si = x = mix64(x);
  }
  static std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  std::uint64_t next() {
    const std::uint64_t result = rotl(s[1] * 5, 7) * 9;
    const std::uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
};

constexpr std::uint64_t kTileBudgetBytes = 2ull << 30;  // generated K chunks per row block
constexpr std::uint64_t kDenseGuard = 16384;            // executor.cpp:442-443

template <class T>
int ensure(T** p, std::size_t& cap, std::size_t count, bool zero = false) {
  if (count <= cap) return HMXG_OK;
  cudaFree(*p);
  *p = nullptr;
  cap = 0;
  HMXG_CUDA(cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
  if (zero) {
    HMXG_CUDA(cudaMemset(*p, 0, count * sizeof(T)));
    HMXG_CUDA(cudaDeviceSynchronize());  // legacy-stream memset vs the non-blocking streams
  }
  cap = count;
  return HMXG_OK;
}

}  // namespace
}  // namespace hmxg

struct hmxg_points {
  int dev = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::uint64_t n = 0, npad = 0;
  hmxg::KernelParams kp{};
  unsigned gemm_grid = 0;
  double* pts = nullptr;
  std::uint32_t* ident = nullptr;  // identity order for the transpose kernel
  double* wdev = nullptr;          // host W staged on the device (n x q, column major)
  std::size_t wdev_cap = 0;
  double* wt = nullptr;            // point-major W (npad x phys_cols(q)); pad rows stay zero
  std::size_t wt_cap = 0;
  double* ktiles = nullptr;
  std::size_t ktiles_cap = 0;
  double* part = nullptr;          // K-split partial products (point-major)
  std::size_t part_cap = 0;
  double* ydev = nullptr;          // exact rows (nrows x q, column major)
  std::size_t ydev_cap = 0;
  double* yadev = nullptr;         // the approximation's rows (error oracle)
  std::size_t yadev_cap = 0;
  std::uint32_t* rows_dev = nullptr;
  std::size_t rows_cap = 0;
  hmxg::Task* tasks = nullptr;
  std::size_t tasks_cap = 0;
  hmxg::SegDev* segs = nullptr;
  std::size_t segs_cap = 0;
  std::uint32_t* counter = nullptr;
  double* err_part = nullptr;
  std::mutex mu;

  ~hmxg_points() {
    if (cudaSetDevice(dev) != cudaSuccess) return;
    if (st) cudaStreamSynchronize(st);
    for (void* p : {static_cast<void*>(pts), static_cast<void*>(ident), static_cast<void*>(wdev),
                    static_cast<void*>(wt), static_cast<void*>(ktiles), static_cast<void*>(part),
                    static_cast<void*>(ydev), static_cast<void*>(yadev), static_cast<void*>(rows_dev),
                    static_cast<void*>(tasks), static_cast<void*>(segs), static_cast<void*>(counter),
                    static_cast<void*>(err_part)})
      cudaFree(p);
    for (cudaEvent_t e : {ev0, ev1})
      if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
  }
};

namespace hmxg {
namespace {

// Y (nrows x q, column major, ldy) = K(x_rows, x_all) W for device W (n x q, ldw); rows is
// a host array or null (every point in order).
int kernel_rows_dev(hmxg_points& P, const std::uint32_t* rows, std::uint64_t nrows, const double* w,
                    std::size_t ldw, double* y, std::size_t ldy, std::size_t q, cudaStream_t st,
                    std::uint32_t* launches) {
  const std::uint64_t n = P.n, npad = P.npad;
  const std::uint32_t nkc = static_cast<std::uint32_t>(npad / kBK);
  const std::uint32_t qq = static_cast<std::uint32_t>(q);
  const std::uint64_t ldq = phys_cols(q);
  if (npad * ldq > P.wt_cap) {
    HMXG_CUDA(cudaStreamSynchronize(st));
    HMXG_TRY(ensure(&P.wt, P.wt_cap, npad * ldq, true));
  }
  const dim3 tgrid(static_cast<unsigned>((n + kTT - 1) / kTT), (qq + kTT - 1) / kTT);
  if (tgrid.y > 65535) return set_err(HMXG_EINVAL, "hmxg_kernel_rows: too many columns for one call");
  // rows n .. npad of Wt meet the zero A columns past the last point; clear what an
  // earlier call with another pitch may have left there
  if (npad > n) HMXG_CUDA(cudaMemsetAsync(P.wt + n * ldq, 0, (npad - n) * ldq * sizeof(double), st));
  permute_in<<<tgrid, 256, 0, st>>>(w, ldw, P.ident, P.wt, ldq, static_cast<std::uint32_t>(n), qq, nullptr, 0);
  ++*launches;
  if (rows) {
    HMXG_CUDA(cudaStreamSynchronize(st));
    HMXG_TRY(ensure(&P.rows_dev, P.rows_cap, nrows));
    HMXG_CUDA(cudaMemcpyAsync(P.rows_dev, rows, nrows * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
  }
  CUtensorMap tm;
  HMXG_TRY(make_map_box(&tm, P.wt, npad, ldq, ldq, kBPitch, kBK));
  const std::uint64_t rb_budget = std::max<std::uint64_t>(kBM, kTileBudgetBytes / (npad * 8) / kBM * kBM);
  const std::uint64_t rb = std::min<std::uint64_t>((nrows + kBM - 1) / kBM * kBM, rb_budget);
  const std::uint32_t ncb = (qq + kBN - 1) / kBN;
  std::vector<Task> tasks;
  std::vector<SegDev> segs;
  for (std::uint64_t r0 = 0; r0 < nrows; r0 += rb) {
    const std::uint32_t nb = static_cast<std::uint32_t>(std::min<std::uint64_t>(rb, nrows - r0));
    const std::uint32_t ntr = (nb + kBM - 1) / kBM;
    // K splits: about two items per resident CTA, at least 16 chunks per split
    std::uint64_t splits = (2ull * P.gemm_grid + std::uint64_t(ntr) * ncb - 1) / (std::uint64_t(ntr) * ncb);
    splits = std::max<std::uint64_t>(1, std::min<std::uint64_t>({splits, std::max<std::uint32_t>(1, nkc / 16), 64}));
    const std::uint32_t per = static_cast<std::uint32_t>((nkc + splits - 1) / splits);
    const std::uint32_t S = (nkc + per - 1) / per;
    tasks.clear();
    segs.clear();
    for (std::uint32_t s = 0; s < S; ++s)
      for (std::uint32_t t = 0; t < ntr; ++t) {
        Task tk{};
        tk.id_off = tk.id_node0 = tk.id_node1 = kNoMap;
        tk.c_row = (s * ntr + t) * kBM;
        tk.cbuf = kBufYp;
        tk.m = static_cast<std::uint16_t>(std::min<std::uint32_t>(kBM, nb - t * kBM));
        tk.seg_begin = static_cast<std::uint32_t>(segs.size());
        for (std::uint32_t kc = s * per; kc < std::min(nkc, (s + 1) * per); kc += 32768) {
          SegDev sg{};
          const std::uint32_t cnt = std::min<std::uint32_t>(32768, std::min(nkc, (s + 1) * per) - kc);
          sg.tile_off = (std::uint64_t(t) * nkc + kc) * kChunkElems;
          sg.b_row = kc * kBK;
          sg.nchunks = static_cast<std::uint16_t>(cnt);
          sg.bbuf = kBufWp;
          segs.push_back(sg);
        }
        tk.seg_end = static_cast<std::uint32_t>(segs.size());
        tasks.push_back(tk);
      }
    // the previous block's launches read the task tables and buffers being reused
    HMXG_CUDA(cudaStreamSynchronize(st));
    HMXG_TRY(ensure(&P.tasks, P.tasks_cap, tasks.size()));
    HMXG_TRY(ensure(&P.segs, P.segs_cap, segs.size()));
    HMXG_CUDA(cudaMemcpyAsync(P.tasks, tasks.data(), tasks.size() * sizeof(Task), cudaMemcpyHostToDevice, st));
    HMXG_CUDA(cudaMemcpyAsync(P.segs, segs.data(), segs.size() * sizeof(SegDev), cudaMemcpyHostToDevice, st));
    const std::uint64_t nchunks = std::uint64_t(ntr) * nkc;
    HMXG_TRY(ensure(&P.ktiles, P.ktiles_cap, nchunks * kChunkElems));
    HMXG_TRY(ensure(&P.part, P.part_cap, std::uint64_t(S) * ntr * kBM * ldq));
    gen_ktiles<<<static_cast<unsigned>(std::min<std::uint64_t>(nchunks, 148ull * 16)), 256, 0, st>>>(
        P.pts, P.kp, rows ? P.rows_dev : nullptr, r0, nb, nkc, static_cast<std::uint32_t>(n), P.ktiles, nchunks);
    ++*launches;
    GemmParams gp{};
    gp.tiles = P.ktiles;
    gp.tasks = P.tasks;
    gp.segs = P.segs;
    gp.buf[kBufWp] = P.wt;
    gp.buf[kBufT] = P.wt;
    gp.buf[kBufS] = P.wt;
    gp.buf[kBufYp] = P.part;
    for (auto& l : gp.ld) l = ldq;
    gp.q = qq;
    const std::uint64_t items = std::uint64_t(tasks.size()) * ncb;
    HMXG_CUDA(cudaMemsetAsync(P.counter, 0, sizeof(std::uint32_t), st));
    grouped_gemm<<<static_cast<unsigned>(std::min<std::uint64_t>(items, P.gemm_grid)), kThreads, kSmemBytes, st>>>(
        tm, tm, tm, gp, static_cast<std::uint32_t>(tasks.size()), P.counter);
    ++*launches;
    const dim3 rgrid((nb + kTT - 1) / kTT, (qq + kTT - 1) / kTT);
    reduce_splits<<<rgrid, 256, 0, st>>>(P.part, ldq, S, std::uint64_t(ntr) * kBM, y + r0, ldy, nb, qq);
    ++*launches;
    HMXG_CUDA(cudaGetLastError());
  }
  return HMXG_OK;
}

int copy_cols(double* dst, std::size_t lddst, const double* src, std::size_t ldsrc, std::size_t rows,
              std::size_t cols, cudaMemcpyKind kind, cudaStream_t st) {
  if (rows == 0 || cols == 0) return HMXG_OK;
  HMXG_CUDA(cudaMemcpy2DAsync(dst, lddst * sizeof(double), src, ldsrc * sizeof(double), rows * sizeof(double), cols,
                              kind, st));
  return HMXG_OK;
}

}  // namespace
}  // namespace hmxg

using namespace hmxg;

extern "C" {

int hmxg_points_upload(hmxg_ctx* ctx, const double* coords, uint64_t n, uint32_t d, int32_t kernel, double h,
                       hmxg_points** out) {
  if (!ctx || !out || (n && !coords) || ctx->devs.empty()) return set_err(HMXG_EINVAL, "hmxg_points_upload: null argument");
  *out = nullptr;
  if (n == 0 || d == 0) return set_err(HMXG_EINVAL, "hmxg_points_upload: empty point set");
  if (n > 0xffffff00ull) return set_err(HMXG_EINVAL, "hmxg_points_upload: too many points");
  if (kernel < HMXG_KERNEL_GAUSSIAN || kernel > HMXG_KERNEL_INVDIST)
    return set_err(HMXG_EINVAL, "hmxg_points_upload: unknown kernel");
  if (kernel != HMXG_KERNEL_INVDIST && !(h > 0.0))  // Kernel::validate, kernel.cpp:8-11
    return set_err(HMXG_EINVAL, "Gaussian kernel: bandwidth must be > 0");
  auto P = std::make_unique<hmxg_points>();
  P->dev = ctx->devs[0];
  P->n = n;
  P->npad = (n + kBK - 1) / kBK * kBK;
  P->kp.kind = kernel;
  P->kp.d = d;
  P->kp.den = 2.0 * h * h;
  P->kp.invh = 1.0 / h;
  HMXG_CUDA(cudaSetDevice(P->dev));
  HMXG_CUDA(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
  HMXG_CUDA(cudaEventCreate(&P->ev0));
  HMXG_CUDA(cudaEventCreate(&P->ev1));
  HMXG_CUDA(cudaFuncSetAttribute(grouped_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  int per_sm = 0, sms = 0;
  HMXG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grouped_gemm, kThreads, kSmemBytes));
  HMXG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->dev));
  P->gemm_grid = static_cast<unsigned>(std::max(1, std::min(per_sm, 3)) * sms);
  HMXG_TRY(dev_upload(&P->pts, coords, n * d, P->st));
  std::vector<std::uint32_t> ident(n);
  for (std::uint64_t i = 0; i < n; ++i) ident[i] = static_cast<std::uint32_t>(i);
  HMXG_TRY(dev_upload(&P->ident, ident.data(), n, P->st));
  HMXG_CUDA(cudaMalloc(&P->counter, sizeof(std::uint32_t)));
  HMXG_CUDA(cudaMalloc(&P->err_part, 2 * kErrBlocks * sizeof(double)));
  HMXG_CUDA(cudaStreamSynchronize(P->st));
  *out = P.release();
  return HMXG_OK;
}

int hmxg_points_free(hmxg_points* pts) {
  delete pts;
  return HMXG_OK;
}

int hmxg_kernel_rows(hmxg_points* pts, const uint32_t* rows, uint64_t nrows, const double* W, size_t n, size_t q,
                     size_t ldw, double* Y, size_t ldy, unsigned flags, void* stream, hmxg_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!pts) return set_err(HMXG_EINVAL, "hmxg_kernel_rows: null points");
  if (stats) std::memset(stats, 0, sizeof *stats);
  if (n != pts->n) return set_err(HMXG_EINVAL, "dense_apply: W row count mismatch");
  if (!rows && nrows != n) return set_err(HMXG_EINVAL, "hmxg_kernel_rows: nrows must be n without a row list");
  if (q == 0 || nrows == 0) return HMXG_OK;
  if (!W || !Y || ldw < n || ldy < nrows) return set_err(HMXG_EINVAL, "hmxg_kernel_rows: bad W/Y or leading dimension");
  if (nrows > 0xffffffffull || q > 0xffffffffull) return set_err(HMXG_EINVAL, "hmxg_kernel_rows: too large");
  if (rows)
    for (std::uint64_t i = 0; i < nrows; ++i)
      if (rows[i] >= n) return set_err(HMXG_EINVAL, "dense_block: row index out of range");
  std::lock_guard<std::mutex> lock(pts->mu);
  hmxg_points& P = *pts;
  HMXG_CUDA(cudaSetDevice(P.dev));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.st;
  std::uint32_t launches = 0;
  HMXG_CUDA(cudaEventRecord(P.ev0, st));
  if (flags & HMXG_F_DEVICE_PTRS) {
    HMXG_TRY(kernel_rows_dev(P, rows, nrows, W, ldw, Y, ldy, q, st, &launches));
  } else {
    HMXG_CUDA(cudaStreamSynchronize(st));
    HMXG_TRY(ensure(&P.wdev, P.wdev_cap, n * q));
    HMXG_TRY(ensure(&P.ydev, P.ydev_cap, nrows * q));
    HMXG_TRY(copy_cols(P.wdev, n, W, ldw, n, q, cudaMemcpyHostToDevice, st));
    HMXG_TRY(kernel_rows_dev(P, rows, nrows, P.wdev, n, P.ydev, nrows, q, st, &launches));
    HMXG_TRY(copy_cols(Y, ldy, P.ydev, nrows, nrows, q, cudaMemcpyDeviceToHost, st));
  }
  HMXG_CUDA(cudaEventRecord(P.ev1, st));
  HMXG_CUDA(cudaEventSynchronize(P.ev1));
  if (stats) {
    float ms = 0.f;
    HMXG_CUDA(cudaEventElapsedTime(&ms, P.ev0, P.ev1));
    stats->device_ms = ms;
    stats->launches = launches;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return HMXG_OK;
}

uint64_t hmxg_sample_rows(uint64_t n, uint64_t seed, uint32_t* rows) {
  // executor.cpp:446-451: iota, then swap(rows[i], rows[i + below(n - i)]) for i < min(n, 256)
  const std::uint64_t nr = std::min<std::uint64_t>(n, 256);
  if (!rows || nr == 0) return 0;
  std::vector<std::uint32_t> all(n);
  for (std::uint64_t i = 0; i < n; ++i) all[i] = static_cast<std::uint32_t>(i);
  Xoshiro rng(mix64(seed ^ mix64(0xe44a11ULL)));
  for (std::uint64_t i = 0; i < nr; ++i) std::swap(all[i], all[i + rng.next() % (n - i)]);
  std::memcpy(rows, all.data(), nr * sizeof(std::uint32_t));
  return nr;
}

int hmxg_relative_error(hmxg_points* pts, const double* Y_approx, size_t ldya, const double* W, size_t n, size_t q,
                        size_t ldw, int mode, uint64_t seed, unsigned flags, double* eps) {
  if (!pts || !eps) return set_err(HMXG_EINVAL, "hmxg_relative_error: null argument");
  if (n != pts->n) return set_err(HMXG_EINVAL, "relative_error: shape mismatch");
  if (mode != HMXG_ERR_DENSE && mode != HMXG_ERR_SAMPLED) return set_err(HMXG_EINVAL, "relative_error: bad mode");
  *eps = 0.0;
  if (q == 0) return HMXG_OK;  // executor.cpp:437-440 (0 by convention)
  if (!W || !Y_approx || ldw < n || ldya < n) return set_err(HMXG_EINVAL, "relative_error: bad W/Y or leading dimension");
  if (mode == HMXG_ERR_DENSE && n > kDenseGuard)
    return set_err(HMXG_EGUARD, "dense error oracle limited to n <= 16384; use sampled mode");
  std::vector<std::uint32_t> rows;
  if (mode == HMXG_ERR_SAMPLED) {
    rows.resize(std::min<std::uint64_t>(n, 256));
    hmxg_sample_rows(n, seed, rows.data());
  }
  const std::uint64_t nr = mode == HMXG_ERR_SAMPLED ? rows.size() : n;
  const bool dev_ptrs = flags & HMXG_F_DEVICE_PTRS;
  std::lock_guard<std::mutex> lock(pts->mu);
  hmxg_points& P = *pts;
  HMXG_CUDA(cudaSetDevice(P.dev));
  cudaStream_t st = P.st;
  std::uint32_t launches = 0;
  const double* wd = W;
  std::size_t ldwd = ldw;
  if (!dev_ptrs) {
    HMXG_TRY(ensure(&P.wdev, P.wdev_cap, n * q));
    HMXG_TRY(copy_cols(P.wdev, n, W, ldw, n, q, cudaMemcpyHostToDevice, st));
    wd = P.wdev;
    ldwd = n;
  }
  HMXG_TRY(ensure(&P.ydev, P.ydev_cap, nr * q));
  HMXG_TRY(kernel_rows_dev(P, rows.empty() ? nullptr : rows.data(), nr, wd, ldwd, P.ydev, nr, q, st, &launches));
  // the approximation's rows, column major with leading dimension `lda`
  const double* ya = Y_approx;
  std::size_t lda = ldya;
  if (mode == HMXG_ERR_SAMPLED) {
    HMXG_TRY(ensure(&P.yadev, P.yadev_cap, nr * q));
    if (dev_ptrs) {
      // P.rows_dev holds the sampled rows (uploaded by kernel_rows_dev)
      const std::uint64_t cells = nr * q;
      gather_rows<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, st>>>(
          Y_approx, ldya, P.rows_dev, static_cast<std::uint32_t>(nr), static_cast<std::uint32_t>(q), P.yadev);
    } else {
      std::vector<double> host(nr * q);
      for (std::size_t c = 0; c < q; ++c)
        for (std::uint64_t i = 0; i < nr; ++i) host[i + c * nr] = Y_approx[rows[i] + c * ldya];
      HMXG_CUDA(cudaMemcpyAsync(P.yadev, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, st));
      HMXG_CUDA(cudaStreamSynchronize(st));  // `host` goes out of scope
    }
    ya = P.yadev;
    lda = nr;
  } else if (!dev_ptrs) {
    HMXG_TRY(ensure(&P.yadev, P.yadev_cap, n * q));
    HMXG_TRY(copy_cols(P.yadev, n, Y_approx, ldya, n, q, cudaMemcpyHostToDevice, st));
    ya = P.yadev;
    lda = n;
  }
  err_sums<<<kErrBlocks, kErrThreads, 0, st>>>(ya, lda, P.ydev, nr, nr, q, P.err_part);
  HMXG_CUDA(cudaGetLastError());
  std::vector<double> part(2 * kErrBlocks);
  HMXG_CUDA(cudaMemcpyAsync(part.data(), P.err_part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  HMXG_CUDA(cudaStreamSynchronize(st));
  double num2 = 0.0, den2 = 0.0;
  for (unsigned b = 0; b < kErrBlocks; ++b) {
    num2 += part[2 * b];
    den2 += part[2 * b + 1];
  }
  *eps = den2 == 0.0 ? 0.0 : std::sqrt(num2 / den2);
  return HMXG_OK;
}

}  // extern "C"
