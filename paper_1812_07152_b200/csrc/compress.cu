// compress.cu — GPU compression: the interpolative decomposition of every participating
// node (/root/reference/proj/src/compress.cpp:17-148).
//
// The reference compresses bottom-up by tree level. For each node it forms the sampled
// block K(sample rows, columns), where the columns are the node's points (leaf) or its
// children's skeletons. It then runs a column-pivoted Householder QR that recomputes the
// exact trailing column norms every step, stops at tol * ||block||_F or max_rank, and
// interpolates the non-skeleton columns with T = R11^{-1} R12.
//
// Here one CTA runs one node's decomposition and one launch covers a tree level. The
// per-column arithmetic (sampled kernel entries, column norms, Householder dot products and
// updates, triangular solves) runs sequentially per column in the reference's order
// without FMA contraction. The pivots, ranks, skeletons and bases therefore follow the
// reference's, and are bit-identical for kernels built from correctly rounded operations
// (inverse distance). The two whole-block sums that only feed the stopping test (||A||_F^2
// and the remaining trailing mass) are parallel reductions; a different outcome needs the
// test to sit within an ulp of its threshold.
//
// Layout: the block is row major in a per-node global scratch (A(i, j) at i*c + j), so the
// threads of a warp, one column each, read consecutive addresses for every row.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hmxg.h"
#include "kfun.cuh"
#include "runtime.hpp"

namespace hmxg {
namespace {

constexpr unsigned kIdThreads = 256;
constexpr double kRankFloor = 1e-14;  // compress.cpp:13
constexpr int kChain = 16;            // column-chain loads per block (two blocks in flight)

// One node's decomposition.
struct IdJob {
  std::uint64_t a_off;     // r x c block (row major) in the scratch
  std::uint64_t v_off;     // Householder vector scratch (r doubles)
  std::uint64_t out_off;   // V (c x cap, column major) in the output buffer
  std::uint64_t samp_off;  // sample rows in the sample index array
  std::uint64_t cols_off;  // column point indices in the column index array
  std::uint64_t piv_off;   // column permutation (c entries)
  std::uint32_t r, c, cap;
  std::uint32_t pad;
};

__device__ __forceinline__ void block_reduce_max_sum(double& best, std::uint32_t& best_j, double& sum, double* s_val,
                                                     std::uint32_t* s_idx, double* s_sum) {
  // (max value, lowest index among maxima) and a sum over the CTA's threads
  const unsigned t = threadIdx.x;
  s_val[t] = best;
  s_idx[t] = best_j;
  s_sum[t] = sum;
  __syncthreads();
  for (unsigned w = blockDim.x / 2; w > 0; w >>= 1) {
    if (t < w) {
      const double ov = s_val[t + w];
      const std::uint32_t oj = s_idx[t + w];
      if (ov > s_val[t] || (ov == s_val[t] && oj < s_idx[t])) {
        s_val[t] = ov;
        s_idx[t] = oj;
      }
      s_sum[t] += s_sum[t + w];
    }
    __syncthreads();
  }
  best = s_val[0];
  best_j = s_idx[0];
  sum = s_sum[0];
  __syncthreads();
}

// s (+)= f(x_i) over rows [k, r) of one column (stride c), in row order (the reference's
// sum), with the next kChain rows' loads in flight while the current block is added: the
// chain is bound by the add latency, not by an L2 round trip per block.
template <class F>
__device__ __forceinline__ double chain_sum(const double* __restrict__ col, std::uint32_t c, std::uint32_t k,
                                            std::uint32_t r, F&& f) {
  double s = 0.0;
  std::uint32_t i = k;
  if (i + kChain <= r) {
    double x0[kChain], x1[kChain];
#pragma unroll
    for (int u = 0; u < kChain; ++u) x0[u] = col[static_cast<std::uint64_t>(i + u) * c];
    for (;;) {
      const bool more = i + 2 * kChain <= r;
      if (more) {
#pragma unroll
        for (int u = 0; u < kChain; ++u) x1[u] = col[static_cast<std::uint64_t>(i + kChain + u) * c];
      }
#pragma unroll
      for (int u = 0; u < kChain; ++u) s = __dadd_rn(s, f(i + u, x0[u]));
      i += kChain;
      if (!more) break;
#pragma unroll
      for (int u = 0; u < kChain; ++u) x0[u] = x1[u];
    }
  }
  for (; i < r; ++i) s = __dadd_rn(s, f(i, col[static_cast<std::uint64_t>(i) * c]));
  return s;
}

__global__ void __launch_bounds__(kIdThreads) id_level(const double* __restrict__ pts, const KernelParams kp,
                                                      const IdJob* __restrict__ jobs,
                                                      const std::uint32_t* __restrict__ samp,
                                                      const std::uint32_t* __restrict__ cols, double tol,
                                                      double* __restrict__ scratch, double* __restrict__ vout,
                                                      std::uint32_t* __restrict__ piv_out,
                                                      std::uint32_t* __restrict__ rank_out) {
  extern __shared__ unsigned char smem[];
  const IdJob job = jobs[blockIdx.x];
  const std::uint32_t r = job.r, c = job.c, cap = job.cap;
  double* a = scratch + job.a_off;
  (void)job.v_off;  // (the Householder vector lives in shared memory)
  std::uint32_t* piv = piv_out + job.piv_off;
  double* norms2 = reinterpret_cast<double*>(smem);               // c
  double* red_val = norms2 + c;                                   // blockDim
  double* red_sum = red_val + blockDim.x;                         // blockDim
  double* vs = red_sum + blockDim.x;                              // r: the Householder vector
  std::uint32_t* red_idx = reinterpret_cast<std::uint32_t*>(vs + r);  // blockDim
  __shared__ double s_v2, s_xnorm;
  const unsigned t = threadIdx.x, nt = blockDim.x;

  // the sampled block: A(i, j) = K(x_{samp[i]}, x_{cols[j]}) (dense_block, kernel.cpp:52-65)
  const std::uint32_t* sr = samp + job.samp_off;
  const std::uint32_t* cl = cols + job.cols_off;
  for (std::uint64_t e = t; e < static_cast<std::uint64_t>(r) * c; e += nt) {
    const std::uint32_t i = static_cast<std::uint32_t>(e / c), j = static_cast<std::uint32_t>(e % c);
    a[e] = kernel_value(kp, pts + static_cast<std::uint64_t>(sr[i]) * kp.d,
                        pts + static_cast<std::uint64_t>(cl[j]) * kp.d);
  }
  for (std::uint32_t j = t; j < c; j += nt) piv[j] = j;
  __syncthreads();
  // ||A||_F^2 (stopping threshold only)
  double part = 0.0;
  for (std::uint64_t e = t; e < static_cast<std::uint64_t>(r) * c; e += nt) part += a[e] * a[e];
  {
    double dummy = 0.0;
    std::uint32_t dj = 0;
    block_reduce_max_sum(dummy, dj, part, red_val, red_idx, red_sum);
  }
  const double tol_eff = fmax(tol, kRankFloor);
  const double stop2 = tol_eff * tol_eff * part;

  std::uint32_t k = 0;
  for (; k < cap; ++k) {
    // exact trailing column norms (compress.cpp:33-46), one column per thread, rows in order
    double best = -1.0, rem = 0.0;
    std::uint32_t best_j = 0xffffffffu;
    for (std::uint32_t j = k + t; j < c; j += nt) {
      // rows in order (the reference's sum), loads issued kChain ahead of the adds: the
      // chain is bound by the add latency, not by one L2 round trip per row
      const double s = chain_sum(a + j, c, k, r, [](std::uint32_t, double x) { return __dmul_rn(x, x); });
      norms2[j] = s;
      rem += s;
      if (s > best) {  // strictly greater: the first maximum of this thread's columns
        best = s;
        best_j = j;
      }
    }
    block_reduce_max_sum(best, best_j, rem, red_val, red_idx, red_sum);
    if (rem <= stop2 || best <= 0.0) break;
    const std::uint32_t pivot = best_j;
    if (pivot != k) {
      for (std::uint32_t i = t; i < r; i += nt) {
        double* row = a + static_cast<std::uint64_t>(i) * c;
        const double tmp = row[k];
        row[k] = row[pivot];
        row[pivot] = tmp;
      }
      if (t == 0) {
        const std::uint32_t tp = piv[k];
        piv[k] = piv[pivot];
        piv[pivot] = tp;
      }
    }
    __syncthreads();
    // Householder reflector zeroing column k below the diagonal (compress.cpp:55-76)
    for (std::uint32_t i = k + 1 + t; i < r; i += nt) vs[i - k] = a[static_cast<std::uint64_t>(i) * c + k];
    if (t == 0) {
      const double ckk = a[static_cast<std::uint64_t>(k) * c + k];
      double xnorm = __dsqrt_rn(norms2[pivot]);
      if (ckk > 0) xnorm = -xnorm;
      vs[0] = __dsub_rn(ckk, xnorm);
      s_xnorm = xnorm;
    }
    __syncthreads();
    if (t == 0) {  // ||v||^2 in order; the shared-memory loads run kChain ahead of the adds
      s_v2 = chain_sum(vs, 1, 0, r - k, [](std::uint32_t, double x) { return __dmul_rn(x, x); });
      a[static_cast<std::uint64_t>(k) * c + k] = s_xnorm;
    }
    for (std::uint32_t i = k + 1 + t; i < r; i += nt) a[static_cast<std::uint64_t>(i) * c + k] = 0.0;
    __syncthreads();
    const double v2 = s_v2;
    if (v2 > 0.0) {
      for (std::uint32_t j = k + 1 + t; j < c; j += nt) {
        double* col = a + j;
        const double dot = chain_sum(col, c, k, r, [&](std::uint32_t i, double x) { return __dmul_rn(vs[i - k], x); });
        const double f = __ddiv_rn(__dmul_rn(2.0, dot), v2);
#pragma unroll 16
        for (std::uint32_t i2 = k; i2 < r; ++i2) {
          double* x = col + static_cast<std::uint64_t>(i2) * c;
          *x = __dsub_rn(*x, __dmul_rn(f, vs[i2 - k]));
        }
      }
    }
    __syncthreads();
  }

  // V (c x k): identity on the skeleton, T = R11^{-1} R12 elsewhere (compress.cpp:79-96)
  double* V = vout + job.out_off;
  for (std::uint64_t e = t; e < static_cast<std::uint64_t>(c) * k; e += nt) V[e] = 0.0;
  __syncthreads();
  for (std::uint32_t j = t; j < k; j += nt) V[piv[j] + static_cast<std::uint64_t>(j) * c] = 1.0;
  for (std::uint32_t tc = k + t; tc < c; tc += nt) {
    double* row_out = V + piv[tc];  // x[j] lives at V(piv[tc], j)
    for (std::uint32_t i = k; i-- > 0;) {
      double s = a[static_cast<std::uint64_t>(i) * c + tc];
      for (std::uint32_t j = i + 1; j < k; ++j)
        s = __dsub_rn(s, __dmul_rn(a[static_cast<std::uint64_t>(i) * c + j], row_out[static_cast<std::uint64_t>(j) * c]));
      row_out[static_cast<std::uint64_t>(i) * c] = __ddiv_rn(s, a[static_cast<std::uint64_t>(i) * c + i]);
    }
  }
  if (t == 0) rank_out[blockIdx.x] = k;
}

template <class T>
int grow(T** p, std::size_t& cap, std::size_t count) {
  if (count <= cap) return HMXG_OK;
  cudaFree(*p);
  *p = nullptr;
  cap = 0;
  HMXG_CUDA(cudaMalloc(reinterpret_cast<void**>(p), std::max<std::size_t>(count, 1) * sizeof(T)));
  cap = count;
  return HMXG_OK;
}

}  // namespace
}  // namespace hmxg

struct hmxg_compressed {
  std::vector<std::uint32_t> srank;
  std::vector<std::uint64_t> skel_ptr, v_ptr, v_rows;
  std::vector<std::uint32_t> skel;
  std::vector<double> v;
};

using namespace hmxg;

extern "C" {

int hmxg_compress(hmxg_ctx* ctx, const double* coords, uint64_t n, uint32_t d, int32_t kernel, double h,
                  uint32_t num_nodes, const uint32_t* lchild, const uint32_t* rchild, const uint32_t* start,
                  const uint32_t* end, const uint32_t* level, const uint32_t* perm, const uint8_t* participating,
                  const uint64_t* sample_ptr, const uint32_t* sample_idx, double bacc, uint32_t max_rank,
                  hmxg_compressed** out) {
  if (!ctx || !out || !coords || !lchild || !rchild || !start || !end || !level || !perm || !participating ||
      !sample_ptr || ctx->devs.empty())
    return set_err(HMXG_EINVAL, "hmxg_compress: null argument");
  *out = nullptr;
  if (n == 0 || d == 0 || num_nodes == 0) return set_err(HMXG_EINVAL, "hmxg_compress: empty input");
  if (bacc < 0.0) return set_err(HMXG_EINVAL, "compress: bacc must be >= 0");
  if (kernel < HMXG_KERNEL_GAUSSIAN || kernel > HMXG_KERNEL_INVDIST)
    return set_err(HMXG_EINVAL, "hmxg_compress: unknown kernel");
  if (kernel != HMXG_KERNEL_INVDIST && !(h > 0.0)) return set_err(HMXG_EINVAL, "Gaussian kernel: bandwidth must be > 0");
  const std::uint64_t total_samples = sample_ptr[num_nodes];
  if (total_samples && !sample_idx) return set_err(HMXG_EINVAL, "hmxg_compress: null sample rows");
  for (std::uint64_t s = 0; s < total_samples; ++s)
    if (sample_idx[s] >= n) return set_err(HMXG_EINVAL, "dense_block: row index out of range");

  KernelParams kp{};
  kp.kind = kernel;
  kp.d = d;
  kp.den = 2.0 * h * h;
  kp.invh = 1.0 / h;
  auto res = std::make_unique<hmxg_compressed>();
  res->srank.assign(num_nodes, 0);
  std::vector<std::vector<std::uint32_t>> skel(num_nodes);
  std::vector<std::vector<double>> vmat(num_nodes);
  std::vector<std::uint64_t> vrows(num_nodes, 0);

  HMXG_CUDA(cudaSetDevice(ctx->devs[0]));
  cudaStream_t st = nullptr;
  HMXG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t st;
    std::vector<void*> ptrs;
    ~Guard() {
      if (st) cudaStreamSynchronize(st);
      for (void* p : ptrs) cudaFree(p);
      if (st) cudaStreamDestroy(st);
    }
  } guard{st, {}};
  double* d_pts = nullptr;
  std::uint32_t* d_samp = nullptr;
  HMXG_TRY(dev_upload(&d_pts, coords, n * d, st));
  guard.ptrs.push_back(d_pts);
  HMXG_TRY(dev_upload(&d_samp, sample_idx, total_samples, st));
  guard.ptrs.push_back(d_samp);

  std::uint32_t height = 0;
  for (std::uint32_t i = 0; i < num_nodes; ++i) height = std::max(height, level[i]);
  std::vector<std::vector<std::uint32_t>> by_level(height + 1);
  for (std::uint32_t i = 0; i < num_nodes; ++i)
    if (participating[i]) by_level[level[i]].push_back(i);

  // per-level buffers, grown as needed and freed on every exit path
  struct LevelBufs {
    IdJob* jobs = nullptr;
    std::uint32_t* cols = nullptr;
    double *scratch = nullptr, *vout = nullptr;
    std::uint32_t *piv = nullptr, *rank = nullptr;
    ~LevelBufs() {
      cudaFree(jobs);
      cudaFree(cols);
      cudaFree(scratch);
      cudaFree(vout);
      cudaFree(piv);
      cudaFree(rank);
    }
  } lb;
  IdJob*& d_jobs = lb.jobs;
  std::uint32_t*& d_cols = lb.cols;
  double*& d_scratch = lb.scratch;
  double*& d_vout = lb.vout;
  std::uint32_t*& d_piv = lb.piv;
  std::uint32_t*& d_rank = lb.rank;
  std::size_t cap_jobs = 0, cap_cols = 0, cap_scratch = 0, cap_vout = 0, cap_piv = 0, cap_rank = 0;
  // per level: its device V buffer and where every node's V sits in it
  struct LevelV {
    double* vout = nullptr;
    std::uint64_t elems = 0;
    struct Part {
      std::uint32_t node;
      std::uint64_t off, count;
    };
    std::vector<Part> parts;
    LevelV() = default;
    LevelV(LevelV&& o) noexcept : vout(o.vout), elems(o.elems), parts(std::move(o.parts)) { o.vout = nullptr; }
    LevelV(const LevelV&) = delete;
    ~LevelV() { cudaFree(vout); }
  };
  std::vector<LevelV> levels_v;
  for (std::uint32_t lvl = height + 1; lvl-- > 0;) {  // deepest level first (compress.cpp:117-121)
    std::vector<IdJob> jobs;
    std::vector<std::uint32_t> job_node, colbuf;
    std::uint64_t scratch = 0, vsize = 0, pivsize = 0;
    std::uint32_t max_c = 0, max_r = 0;
    for (std::uint32_t node : by_level[lvl]) {
      const std::uint64_t r = sample_ptr[node + 1] - sample_ptr[node];
      std::vector<std::uint32_t> cl;
      const bool leaf = lchild[node] == HMXG_NO_NODE;
      if (leaf) {
        cl.assign(perm + start[node], perm + end[node]);
      } else {
        cl = skel[lchild[node]];
        cl.insert(cl.end(), skel[rchild[node]].begin(), skel[rchild[node]].end());
      }
      if (cl.empty()) continue;  // both children collapsed to srank 0 (compress.cpp:132-136)
      if (r == 0)
        return set_err(HMXG_EINVAL, "compress: participating node " + std::to_string(node) +
                                        " has no sample rows (sampling contract violation)");
      if (cl.size() > 0xffffffffull || r > 0xffffffffull) return set_err(HMXG_EINVAL, "hmxg_compress: block too large");
      IdJob j{};
      j.r = static_cast<std::uint32_t>(r);
      j.c = static_cast<std::uint32_t>(cl.size());
      j.cap = static_cast<std::uint32_t>(std::min<std::uint64_t>({r, cl.size(), max_rank}));
      j.a_off = scratch;
      scratch += r * cl.size();
      j.v_off = scratch;
      scratch += r;
      j.out_off = vsize;
      vsize += static_cast<std::uint64_t>(j.c) * j.cap;
      j.samp_off = sample_ptr[node];
      j.cols_off = colbuf.size();
      colbuf.insert(colbuf.end(), cl.begin(), cl.end());
      j.piv_off = pivsize;
      pivsize += j.c;
      max_c = std::max(max_c, j.c);
      max_r = std::max(max_r, j.r);
      jobs.push_back(j);
      job_node.push_back(node);
      skel[node] = std::move(cl);  // the node's columns; replaced by its skeleton below
    }
    if (jobs.empty()) continue;
    HMXG_TRY(grow(&d_jobs, cap_jobs, jobs.size()));
    HMXG_TRY(grow(&d_cols, cap_cols, colbuf.size()));
    HMXG_TRY(grow(&d_scratch, cap_scratch, scratch));
    HMXG_TRY(grow(&d_vout, cap_vout, vsize));
    HMXG_TRY(grow(&d_piv, cap_piv, pivsize));
    HMXG_TRY(grow(&d_rank, cap_rank, jobs.size()));
    HMXG_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), jobs.size() * sizeof(IdJob), cudaMemcpyHostToDevice, st));
    HMXG_CUDA(cudaMemcpyAsync(d_cols, colbuf.data(), colbuf.size() * 4, cudaMemcpyHostToDevice, st));
    const std::size_t smem =
        (max_c + max_r) * sizeof(double) + kIdThreads * (2 * sizeof(double) + sizeof(std::uint32_t));
    if (smem > 200 * 1024) return set_err(HMXG_EINVAL, "hmxg_compress: too many columns in one block");
    if (smem > 48 * 1024) HMXG_CUDA(cudaFuncSetAttribute(id_level, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t te0 = nullptr, te1 = nullptr;
    const bool trace = std::getenv("HMXG_COMPRESS_TRACE") != nullptr;
    if (trace) {
      cudaEventCreate(&te0);
      cudaEventCreate(&te1);
      cudaEventRecord(te0, st);
    }
    id_level<<<static_cast<unsigned>(jobs.size()), kIdThreads, smem, st>>>(d_pts, kp, d_jobs, d_samp, d_cols, bacc,
                                                                          d_scratch, d_vout, d_piv, d_rank);
    if (trace) {
      cudaEventRecord(te1, st);
      cudaEventSynchronize(te1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, te0, te1);
      std::fprintf(stderr, "[hmxg_compress] level %u: %zu nodes, max r %u, max c %u, kernel %.3f ms\n", lvl,
                   jobs.size(), max_r, max_c, ms);
      cudaEventDestroy(te0);
      cudaEventDestroy(te1);
    }
    HMXG_CUDA(cudaGetLastError());
    // only the ranks and pivots come back per level (the next level's columns are the
    // skeletons); the bases stay on the device until the end
    std::vector<std::uint32_t> ranks(jobs.size()), piv(pivsize);
    HMXG_CUDA(cudaMemcpyAsync(ranks.data(), d_rank, ranks.size() * 4, cudaMemcpyDeviceToHost, st));
    HMXG_CUDA(cudaMemcpyAsync(piv.data(), d_piv, piv.size() * 4, cudaMemcpyDeviceToHost, st));
    HMXG_CUDA(cudaStreamSynchronize(st));
    LevelV lv;
    lv.vout = d_vout;  // this level's V buffer is kept; the next level allocates its own
    d_vout = nullptr;
    cap_vout = 0;
    for (std::size_t q = 0; q < jobs.size(); ++q) {
      const std::uint32_t node = job_node[q], k = ranks[q], c = jobs[q].c;
      const std::vector<std::uint32_t> cl = std::move(skel[node]);
      std::vector<std::uint32_t> sk(k);
      for (std::uint32_t j = 0; j < k; ++j) sk[j] = cl[piv[jobs[q].piv_off + j]];
      skel[node] = std::move(sk);
      res->srank[node] = k;
      vrows[node] = c;
      lv.parts.push_back({node, jobs[q].out_off, std::uint64_t(c) * k});
    }
    lv.elems = vsize;
    levels_v.push_back(std::move(lv));
  }
  // every level's bases, read back once at the end
  {
    std::uint64_t most = 0;
    for (const LevelV& lv : levels_v) most = std::max(most, lv.elems);
    std::vector<double> vh(most);
    for (const LevelV& lv : levels_v) {
      if (!lv.elems) continue;
      HMXG_CUDA(cudaMemcpyAsync(vh.data(), lv.vout, lv.elems * sizeof(double), cudaMemcpyDeviceToHost, st));
      HMXG_CUDA(cudaStreamSynchronize(st));
      for (const auto& pt : lv.parts) vmat[pt.node].assign(vh.begin() + pt.off, vh.begin() + pt.off + pt.count);
    }
  }
  // flatten
  res->skel_ptr.assign(num_nodes + 1, 0);
  res->v_ptr.assign(num_nodes + 1, 0);
  res->v_rows = vrows;
  for (std::uint32_t i = 0; i < num_nodes; ++i) {
    res->skel_ptr[i + 1] = res->skel_ptr[i] + skel[i].size();
    res->v_ptr[i + 1] = res->v_ptr[i] + vmat[i].size();
  }
  res->skel.reserve(res->skel_ptr[num_nodes]);
  res->v.reserve(res->v_ptr[num_nodes]);
  for (std::uint32_t i = 0; i < num_nodes; ++i) {
    res->skel.insert(res->skel.end(), skel[i].begin(), skel[i].end());
    res->v.insert(res->v.end(), vmat[i].begin(), vmat[i].end());
  }
  *out = res.release();
  return HMXG_OK;
}

int hmxg_compressed_get(const hmxg_compressed* c, const uint32_t** srank, const uint64_t** skel_ptr,
                        const uint32_t** skel, const uint64_t** v_ptr, const uint64_t** v_rows, const double** v) {
  if (!c) return set_err(HMXG_EINVAL, "hmxg_compressed_get: null handle");
  if (srank) *srank = c->srank.data();
  if (skel_ptr) *skel_ptr = c->skel_ptr.data();
  if (skel) *skel = c->skel.data();
  if (v_ptr) *v_ptr = c->v_ptr.data();
  if (v_rows) *v_rows = c->v_rows.data();
  if (v) *v = c->v.data();
  return HMXG_OK;
}

void hmxg_compressed_free(hmxg_compressed* c) { delete c; }

}  // extern "C"
