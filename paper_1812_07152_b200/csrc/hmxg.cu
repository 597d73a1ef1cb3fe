// hmxg.cu — C-ABI of the B200 evaluator (include/hmxg.h): device residency of the CDS,
// workspace management, column sharding over devices and the launch sequence.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hmxg.h"
#include "kernels.cuh"
#include "plan.hpp"

namespace hmxg {
namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  return set_err(e == cudaErrorMemoryAllocation ? HMXG_ENOMEM : HMXG_ECUDA,
                 std::string(what) + ": " + cudaGetErrorString(e));
}

#define HMXG_CUDA(call)                                   \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

template <class T>
int dev_upload(T** dst, const T* src, std::size_t count, cudaStream_t st) {
  *dst = nullptr;
  if (count == 0) return HMXG_OK;
  HMXG_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), count * sizeof(T)));
  HMXG_CUDA(cudaMemcpyAsync(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return HMXG_OK;
}

struct DevState {
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double* gen[3] = {nullptr, nullptr, nullptr};
  Task* tasks = nullptr;
  Seg* segs = nullptr;
  std::uint32_t* perm = nullptr;
  std::uint32_t* iperm = nullptr;
  std::size_t cap_q = 0;  // evaluation workspace capacity in columns
  double* wp = nullptr;
  double* yp = nullptr;
  double* t = nullptr;
  double* s = nullptr;
  std::size_t stage_q = 0;  // host-mode staging capacity in columns
  double* w_stage = nullptr;
  double* y_stage = nullptr;
  std::uint64_t resident_bytes = 0;

  void release_workspace() {
    cudaFree(wp);
    cudaFree(yp);
    cudaFree(t);
    cudaFree(s);
    wp = yp = t = s = nullptr;
    cap_q = 0;
  }
  void release_stage() {
    cudaFree(w_stage);
    cudaFree(y_stage);
    w_stage = y_stage = nullptr;
    stage_q = 0;
  }
  void release() {
    if (cudaSetDevice(dev) != cudaSuccess) return;
    if (stream) cudaStreamSynchronize(stream);
    release_workspace();
    release_stage();
    for (auto*& g : gen) {
      cudaFree(g);
      g = nullptr;
    }
    cudaFree(tasks);
    cudaFree(segs);
    cudaFree(perm);
    cudaFree(iperm);
    tasks = nullptr;
    segs = nullptr;
    perm = iperm = nullptr;
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
    ev0 = ev1 = nullptr;
    stream = nullptr;
  }
};

}  // namespace
}  // namespace hmxg

struct hmxg_ctx {
  std::vector<int> devs;
};

struct hmxg_mat {
  hmxg_ctx* ctx = nullptr;
  hmxg::Plan plan;
  std::vector<hmxg::DevState> devs;
  std::mutex mu;  // one in-flight evaluate per matrix
};

namespace hmxg {
namespace {

int ensure_workspace(const Plan& plan, DevState& d, std::size_t q) {
  if (q <= d.cap_q) return HMXG_OK;
  d.release_workspace();
  const std::size_t n = plan.n, r = std::max<std::uint64_t>(plan.skel_rows, 1);
  HMXG_CUDA(cudaMalloc(&d.wp, n * q * sizeof(double)));
  HMXG_CUDA(cudaMalloc(&d.yp, n * q * sizeof(double)));
  HMXG_CUDA(cudaMalloc(&d.t, r * q * sizeof(double)));
  HMXG_CUDA(cudaMalloc(&d.s, r * q * sizeof(double)));
  d.cap_q = q;
  return HMXG_OK;
}

int ensure_stage(const Plan& plan, DevState& d, std::size_t q) {
  if (q <= d.stage_q) return HMXG_OK;
  d.release_stage();
  HMXG_CUDA(cudaMalloc(&d.w_stage, plan.n * q * sizeof(double)));
  HMXG_CUDA(cudaMalloc(&d.y_stage, plan.n * q * sizeof(double)));
  d.stage_q = q;
  return HMXG_OK;
}

// Enqueue one full evaluation of q columns on d.stream: W (ldw) -> Y (ldy), device ptrs.
int enqueue_eval(const Plan& plan, DevState& d, const double* w, std::size_t ldw, double* y,
                 std::size_t ldy, std::size_t q, cudaStream_t st, std::uint32_t* launches) {
  const std::uint32_t n = static_cast<std::uint32_t>(plan.n);
  const std::uint32_t qq = static_cast<std::uint32_t>(q);
  const dim3 eblk(256);
  const dim3 egrid((n + 255) / 256, std::min<std::uint32_t>(qq, 65535));
  gather_rows<<<egrid, eblk, 0, st>>>(w, ldw, d.perm, d.wp, plan.n, n, qq);
  ++*launches;

  EvalParams p{};
  p.gen[kGenD] = d.gen[kGenD];
  p.gen[kGenB] = d.gen[kGenB];
  p.gen[kGenV] = d.gen[kGenV];
  p.buf[kBufWp] = d.wp;
  p.buf[kBufT] = d.t;
  p.buf[kBufS] = d.s;
  p.buf[kBufYp] = d.yp;
  p.ld[kBufWp] = plan.n;
  p.ld[kBufT] = plan.skel_rows;
  p.ld[kBufS] = plan.skel_rows;
  p.ld[kBufYp] = plan.n;
  p.segs = d.segs;
  p.q = qq;
  const std::uint32_t col_blocks = (qq + kBN - 1) / kBN;
  for (const Phase& ph : plan.phases) {
    p.tasks = d.tasks + ph.task_begin;
    const dim3 grid(ph.task_end - ph.task_begin, col_blocks);
    if (ph.trans_a)
      grouped_gemm<true><<<grid, kThreads, kSmemBytes, st>>>(p);
    else
      grouped_gemm<false><<<grid, kThreads, kSmemBytes, st>>>(p);
    ++*launches;
  }
  scatter_rows<<<egrid, eblk, 0, st>>>(d.yp, plan.n, d.iperm, y, ldy, n, qq);
  ++*launches;
  HMXG_CUDA(cudaGetLastError());
  return HMXG_OK;
}

}  // namespace
}  // namespace hmxg

using namespace hmxg;

extern "C" {

const char* hmxg_last_error(void) { return g_err.c_str(); }
const char* hmxg_version(void) { return "hmxg 0.1 sm_100a fp64-dmma grouped-gemm"; }

int hmxg_create(const int* devs, int ndev, hmxg_ctx** out) {
  if (!out) return set_err(HMXG_EINVAL, "hmxg_create: null out");
  *out = nullptr;
  int count = 0;
  HMXG_CUDA(cudaGetDeviceCount(&count));
  auto ctx = std::make_unique<hmxg_ctx>();
  if (ndev <= 0 || !devs) {
    ctx->devs.push_back(0);
  } else {
    for (int i = 0; i < ndev; ++i) {
      if (devs[i] < 0 || devs[i] >= count)
        return set_err(HMXG_EINVAL, "hmxg_create: device id out of range");
      ctx->devs.push_back(devs[i]);
    }
  }
  if (count == 0) return set_err(HMXG_ECUDA, "hmxg_create: no CUDA device");
  for (int dv : ctx->devs) {
    cudaDeviceProp prop{};
    HMXG_CUDA(cudaGetDeviceProperties(&prop, dv));
    if (prop.major != 10) return set_err(HMXG_ECUDA, "hmxg_create: built for sm_100a (B200) only");
  }
  *out = ctx.release();
  return HMXG_OK;
}

int hmxg_destroy(hmxg_ctx* ctx) {
  delete ctx;
  return HMXG_OK;
}

int hmxg_upload(hmxg_ctx* ctx, const hmxg_cds_view* cds, hmxg_mat** out) {
  if (!ctx || !cds || !out) return set_err(HMXG_EINVAL, "hmxg_upload: null argument");
  *out = nullptr;
  auto mat = std::make_unique<hmxg_mat>();
  mat->ctx = ctx;
  std::string err;
  if (!build_plan(*cds, kBM, mat->plan, err)) return set_err(HMXG_EINVAL, err);
  const Plan& plan = mat->plan;
  std::vector<std::uint32_t> iperm(plan.n);
  for (std::uint64_t pos = 0; pos < plan.n; ++pos) iperm[cds->perm[pos]] = static_cast<std::uint32_t>(pos);
  mat->devs.resize(ctx->devs.size());
  for (std::size_t g = 0; g < ctx->devs.size(); ++g) {
    DevState& d = mat->devs[g];
    d.dev = ctx->devs[g];
    HMXG_CUDA(cudaSetDevice(d.dev));
    HMXG_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    HMXG_CUDA(cudaEventCreate(&d.ev0));
    HMXG_CUDA(cudaEventCreate(&d.ev1));
    HMXG_CUDA(cudaFuncSetAttribute(grouped_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    HMXG_CUDA(cudaFuncSetAttribute(grouped_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    int rc;
    if ((rc = dev_upload(&d.gen[kGenD], cds->dgen, plan.d_elems, d.stream))) return rc;
    if ((rc = dev_upload(&d.gen[kGenB], cds->bgen, plan.b_elems, d.stream))) return rc;
    if ((rc = dev_upload(&d.gen[kGenV], cds->vgen, plan.v_elems, d.stream))) return rc;
    if ((rc = dev_upload(&d.tasks, plan.tasks.data(), plan.tasks.size(), d.stream))) return rc;
    if ((rc = dev_upload(&d.segs, plan.segs.data(), plan.segs.size(), d.stream))) return rc;
    if ((rc = dev_upload(&d.perm, cds->perm, plan.n, d.stream))) return rc;
    if ((rc = dev_upload(&d.iperm, iperm.data(), plan.n, d.stream))) return rc;
    HMXG_CUDA(cudaStreamSynchronize(d.stream));
    d.resident_bytes = 8 * (plan.d_elems + plan.b_elems + plan.v_elems) +
                       sizeof(Task) * plan.tasks.size() + sizeof(Seg) * plan.segs.size() + 8 * plan.n;
  }
  *out = mat.release();
  return HMXG_OK;
}

int hmxg_validate(const hmxg_cds_view* cds, hmxg_info* info) {
  if (!cds) return set_err(HMXG_EINVAL, "hmxg_validate: null view");
  Plan plan;
  std::string err;
  if (!build_plan(*cds, kBM, plan, err)) return set_err(HMXG_EINVAL, err);
  if (info) {
    std::memset(info, 0, sizeof *info);
    info->n = plan.n;
    info->d_elems = plan.d_elems;
    info->b_elems = plan.b_elems;
    info->v_elems = plan.v_elems;
    info->skel_rows = plan.skel_rows;
    info->launches_per_eval = static_cast<std::uint32_t>(plan.phases.size() + 2);
    info->flops_per_col = 2.0 * (2.0 * plan.v_elems + plan.b_elems + plan.d_elems);
  }
  return HMXG_OK;
}

int hmxg_free(hmxg_mat* mat) {
  if (!mat) return HMXG_OK;
  for (auto& d : mat->devs) d.release();
  delete mat;
  return HMXG_OK;
}

int hmxg_info_get(const hmxg_mat* mat, hmxg_info* info) {
  if (!mat || !info) return set_err(HMXG_EINVAL, "hmxg_info_get: null argument");
  const Plan& p = mat->plan;
  std::memset(info, 0, sizeof *info);
  info->n = p.n;
  info->d_elems = p.d_elems;
  info->b_elems = p.b_elems;
  info->v_elems = p.v_elems;
  info->skel_rows = p.skel_rows;
  info->num_devices = static_cast<std::uint32_t>(mat->devs.size());
  info->launches_per_eval = static_cast<std::uint32_t>(p.phases.size() + 2);
  info->flops_per_col = 2.0 * (2.0 * p.v_elems + p.b_elems + p.d_elems);
  info->device_bytes = mat->devs.empty() ? 0 : mat->devs[0].resident_bytes;
  return HMXG_OK;
}

int hmxg_evaluate(hmxg_mat* mat, const double* W, size_t n, size_t q, size_t ldw, double* Y,
                  size_t ldy, unsigned flags, void* stream, hmxg_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!mat) return set_err(HMXG_EINVAL, "hmxg_evaluate: null matrix");
  if (n != mat->plan.n)
    return set_err(HMXG_EINVAL, "evaluate: W row count does not match the point count");
  if (stats) std::memset(stats, 0, sizeof *stats);
  if (q == 0) return HMXG_OK;  // executor.cpp:279-282
  if (!W || !Y || ldw < n || ldy < n) return set_err(HMXG_EINVAL, "hmxg_evaluate: bad W/Y or leading dimension");
  if (q > 0xffffffffull) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many columns");
  std::lock_guard<std::mutex> lock(mat->mu);
  const Plan& plan = mat->plan;
  std::uint32_t launches = 0;
  float dev_ms = 0.f;

  if (flags & HMXG_F_DEVICE_PTRS) {
    if (mat->devs.size() != 1)
      return set_err(HMXG_EINVAL, "hmxg_evaluate: device pointers need a single-device context");
    DevState& d = mat->devs[0];
    HMXG_CUDA(cudaSetDevice(d.dev));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    int rc = ensure_workspace(plan, d, q);
    if (rc) return rc;
    const bool sync = !(flags & HMXG_F_NO_SYNC);
    if (sync) HMXG_CUDA(cudaEventRecord(d.ev0, st));
    if ((rc = enqueue_eval(plan, d, W, ldw, Y, ldy, q, st, &launches))) return rc;
    if (sync) {
      HMXG_CUDA(cudaEventRecord(d.ev1, st));
      HMXG_CUDA(cudaEventSynchronize(d.ev1));
      HMXG_CUDA(cudaEventElapsedTime(&dev_ms, d.ev0, d.ev1));
    }
  } else {
    // column sharding over the context's devices: Y[:,c] depends only on W[:,c]
    const std::size_t G = mat->devs.size();
    std::vector<std::size_t> c0(G + 1);
    for (std::size_t g = 0; g <= G; ++g) c0[g] = q * g / G;
    for (std::size_t g = 0; g < G; ++g) {
      DevState& d = mat->devs[g];
      const std::size_t qg = c0[g + 1] - c0[g];
      if (qg == 0) continue;
      HMXG_CUDA(cudaSetDevice(d.dev));
      int rc = ensure_workspace(plan, d, qg);
      if (!rc) rc = ensure_stage(plan, d, qg);
      if (rc) return rc;
      HMXG_CUDA(cudaMemcpy2DAsync(d.w_stage, n * sizeof(double), W + c0[g] * ldw, ldw * sizeof(double),
                                  n * sizeof(double), qg, cudaMemcpyHostToDevice, d.stream));
      HMXG_CUDA(cudaEventRecord(d.ev0, d.stream));
      if ((rc = enqueue_eval(plan, d, d.w_stage, n, d.y_stage, n, qg, d.stream, &launches))) return rc;
      HMXG_CUDA(cudaEventRecord(d.ev1, d.stream));
      HMXG_CUDA(cudaMemcpy2DAsync(Y + c0[g] * ldy, ldy * sizeof(double), d.y_stage, n * sizeof(double),
                                  n * sizeof(double), qg, cudaMemcpyDeviceToHost, d.stream));
    }
    for (std::size_t g = 0; g < G; ++g) {
      DevState& d = mat->devs[g];
      if (c0[g + 1] == c0[g]) continue;
      HMXG_CUDA(cudaSetDevice(d.dev));
      HMXG_CUDA(cudaStreamSynchronize(d.stream));
      float ms = 0.f;
      HMXG_CUDA(cudaEventElapsedTime(&ms, d.ev0, d.ev1));
      dev_ms = std::max(dev_ms, ms);
    }
  }
  if (stats) {
    stats->locked_pairs = 0;
    stats->device_ms = dev_ms;
    stats->launches = launches;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return HMXG_OK;
}

}  // extern "C"
