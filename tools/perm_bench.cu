// Microbenchmark: row permutation of an n x q column-major FP64 matrix (gather vs scatter forms).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int C>
__global__ void gather_tc(const double* __restrict__ w, const uint32_t* __restrict__ pmap, double* __restrict__ out, uint32_t n, uint32_t q) {
  uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; if (r >= n) return;
  uint32_t src = pmap[r];
  for (uint32_t c0 = blockIdx.y * C; c0 < q; c0 += gridDim.y * C) {
    double v[C];
#pragma unroll
    for (int j = 0; j < C; ++j) v[j] = __ldg(w + src + (uint64_t)(c0 + j) * n);
#pragma unroll
    for (int j = 0; j < C; ++j) out[r + (uint64_t)(c0 + j) * n] = v[j];
  }
}
template <int C>
__global__ void scatter_tc(const double* __restrict__ w, const uint32_t* __restrict__ ipmap, double* __restrict__ out, uint32_t n, uint32_t q) {
  uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; if (r >= n) return;
  uint32_t dst = ipmap[r];
  for (uint32_t c0 = blockIdx.y * C; c0 < q; c0 += gridDim.y * C) {
    double v[C];
#pragma unroll
    for (int j = 0; j < C; ++j) v[j] = w[r + (uint64_t)(c0 + j) * n];
#pragma unroll
    for (int j = 0; j < C; ++j) out[dst + (uint64_t)(c0 + j) * n] = v[j];
  }
}
// column-outer: one block per (row chunk, single column), many rows per thread
__global__ void gather_col(const double* __restrict__ w, const uint32_t* __restrict__ pmap, double* __restrict__ out, uint32_t n, uint32_t q) {
  uint32_t c = blockIdx.y;
  const double* wc = w + (uint64_t)c * n; double* oc = out + (uint64_t)c * n;
  for (uint32_t r = blockIdx.x * blockDim.x * 8 + threadIdx.x; r < n; r += blockDim.x) {
    if (r >= (blockIdx.x + 1) * blockDim.x * 8) break;
    oc[r] = __ldg(wc + pmap[r]);
  }
}
__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  const uint32_t n = 262144, q = 2048;
  std::vector<uint32_t> p(n), ip(n);
  for (uint32_t i = 0; i < n; ++i) p[i] = i;
  std::mt19937 g(1); std::shuffle(p.begin(), p.end(), g);
  for (uint32_t i = 0; i < n; ++i) ip[p[i]] = i;
  double *w, *o; uint32_t *dp, *dip;
  size_t bytes = (size_t)n * q * 8;
  cudaMalloc(&w, bytes); cudaMalloc(&o, bytes); cudaMalloc(&dp, n * 4); cudaMalloc(&dip, n * 4);
  cudaMemcpy(dp, p.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(dip, ip.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset(w, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int i = 0; i < 5; ++i) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-28s %.3f ms  %.0f GB/s (2 x %.2f GB)\n", name, ms, 2.0 * bytes / ms / 1e6, bytes / 1e9);
  };
  timeit("copy", [&] { copy_k<<<148 * 16, 256>>>((double4*)w, (double4*)o, bytes / 32); });
  timeit("gather C=1", [&] { gather_tc<1><<<dim3(n / 256, 2048), 256>>>(w, dp, o, n, q); });
  timeit("gather C=16", [&] { gather_tc<16><<<dim3(n / 256, 128), 256>>>(w, dp, o, n, q); });
  timeit("gather C=16 y=16", [&] { gather_tc<16><<<dim3(n / 256, 16), 256>>>(w, dp, o, n, q); });
  timeit("gather C=4", [&] { gather_tc<4><<<dim3(n / 256, 512), 256>>>(w, dp, o, n, q); });
  timeit("scatter C=1", [&] { scatter_tc<1><<<dim3(n / 256, 2048), 256>>>(w, dip, o, n, q); });
  timeit("scatter C=4", [&] { scatter_tc<4><<<dim3(n / 256, 512), 256>>>(w, dip, o, n, q); });
  timeit("scatter C=16", [&] { scatter_tc<16><<<dim3(n / 256, 128), 256>>>(w, dip, o, n, q); });
  timeit("gather col-outer", [&] { gather_col<<<dim3(n / 2048, q), 256>>>(w, dp, o, n, q); });
  // sorted (identity) perm for reference: a coalesced gather
  std::vector<uint32_t> idp(n); for (uint32_t i = 0; i < n; ++i) idp[i] = i;
  cudaMemcpy(dp, idp.data(), n * 4, cudaMemcpyHostToDevice);
  timeit("gather C=16 identity", [&] { gather_tc<16><<<dim3(n / 256, 128), 256>>>(w, dp, o, n, q); });
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
