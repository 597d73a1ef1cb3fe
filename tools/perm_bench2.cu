// Transpose-permute variants (W column major -> Wp point major, column blocks at pitch 80):
// the evaluator's 32x32 tile vs wider tiles with 16-byte accesses (dev tool).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__host__ __device__ inline uint64_t phys(uint64_t c) { return (c / 64) * 80 + (c % 64); }

// current: 32x32 tile, 256 threads, 8-byte accesses
__global__ void __launch_bounds__(256) perm32(const double* __restrict__ w, uint64_t ldw, const uint32_t* __restrict__ ip,
                                              double* __restrict__ wp, uint64_t ldp, uint32_t n, uint32_t q) {
  __shared__ double tile[32][33];
  const uint32_t r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const uint32_t r = r0 + tx, c = c0 + ty + k;
    tile[ty + k][tx] = (r < n && c < q) ? __ldg(w + r + (uint64_t)c * ldw) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const uint32_t r = r0 + ty + k, c = c0 + tx;
    if (r < n && c < q) wp[(uint64_t)ip[r] * ldp + phys(c)] = tile[tx][ty + k];
  }
}

// 64 points x 32 columns per CTA, 16-byte loads (2 points) and stores (2 columns)
__global__ void __launch_bounds__(256) perm64v(const double* __restrict__ w, uint64_t ldw, const uint32_t* __restrict__ ip,
                                               double* __restrict__ wp, uint64_t ldp, uint32_t n, uint32_t q) {
  __shared__ double tile[32][64 + 2];  // [col][point]
  const uint32_t r0 = blockIdx.x * 64, c0 = blockIdx.y * 32;
  const int t = threadIdx.x;
  // load: 32 columns x 64 points = 1024 double2 -> 4 per thread; a warp covers one column
  // (32 lanes x 2 points = 64 points, 512 B contiguous)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int col = (t >> 5) + 8 * k, pp = (t & 31) * 2;
    const uint32_t c = c0 + col, r = r0 + pp;
    double2 v = make_double2(0.0, 0.0);
    if (c < q && r + 1 < n) v = __ldg(reinterpret_cast<const double2*>(w + r + (uint64_t)c * ldw));
    else if (c < q && r < n) v.x = __ldg(w + r + (uint64_t)c * ldw);
    tile[col][pp] = v.x;
    tile[col][pp + 1] = v.y;
  }
  __syncthreads();
  // store: 64 points x 32 columns = 1024 double2 -> 4 per thread; 16 lanes cover one
  // point's 32 columns (256 B contiguous), a warp two points
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int pt = (t >> 4) + 16 * k, cc = (t & 15) * 2;
    const uint32_t r = r0 + pt, c = c0 + cc;
    if (r < n && c + 1 < q)
      *reinterpret_cast<double2*>(wp + (uint64_t)ip[r] * ldp + phys(c)) = make_double2(tile[cc][pt], tile[cc + 1][pt]);
    else if (r < n && c < q)
      wp[(uint64_t)ip[r] * ldp + phys(c)] = tile[cc][pt];
  }
}

int main() {
  const uint32_t n = 262144, q = 2048;
  const uint64_t ldp = (q + 63) / 64 * 80;
  std::vector<uint32_t> p(n);
  for (uint32_t i = 0; i < n; ++i) p[i] = i;
  std::mt19937 g(1);
  std::shuffle(p.begin(), p.end(), g);
  double *w, *wp, *wp2;
  uint32_t* ip;
  cudaMalloc(&w, (size_t)n * q * 8);
  cudaMalloc(&wp, (size_t)n * ldp * 8);
  cudaMalloc(&wp2, (size_t)n * ldp * 8);
  cudaMalloc(&ip, n * 4);
  cudaMemcpy(ip, p.data(), n * 4, cudaMemcpyHostToDevice);
  std::vector<double> hw((size_t)n * 4);
  for (size_t i = 0; i < hw.size(); ++i) hw[i] = (double)i;
  cudaMemset(w, 0, (size_t)n * q * 8);
  cudaMemcpy(w, hw.data(), hw.size() * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 10;
    printf("%-10s %.3f ms  %.2f TB/s (16 B per element moved)\n", name, ms, 16.0 * n * q / ms / 1e9);
  };
  run("perm32", [&] { perm32<<<dim3(n / 32, q / 32), 256>>>(w, n, ip, wp, ldp, n, q); });
  run("perm64v", [&] { perm64v<<<dim3(n / 64, q / 32), 256>>>(w, n, ip, wp2, ldp, n, q); });
  std::vector<double> h1((size_t)n * ldp), h2((size_t)n * ldp);
  cudaMemcpy(h1.data(), wp, h1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), wp2, h2.size() * 8, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (uint32_t r = 0; r < n; ++r)
    for (uint32_t c = 0; c < q; ++c) bad += h1[(size_t)r * ldp + phys(c)] != h2[(size_t)r * ldp + phys(c)];
  printf("mismatches: %zu\n", bad);
  return 0;
}
