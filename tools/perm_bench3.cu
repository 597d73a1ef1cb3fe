// Transpose-permute variants, both directions, against a plain copy of the same bytes (dev tool):
// the evaluator's 32 x 32 tiles vs tiles that move a point's whole 64-column block row (512 B).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/perm_bench3 tools/perm_bench3.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__host__ __device__ inline uint64_t phys(uint64_t c) { return (c / 64) * 80 + (c % 64); }

__global__ void __launch_bounds__(256) in32(const double* __restrict__ w, uint64_t ldw, const uint32_t* __restrict__ ip,
                                            double* __restrict__ wp, uint64_t ldp, uint32_t n, uint32_t q) {
  __shared__ double tile[32][33];
  const uint32_t r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) tile[ty + k][tx] = __ldg(w + r0 + tx + (uint64_t)(c0 + ty + k) * ldw);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) wp[(uint64_t)ip[r0 + ty + k] * ldp + phys(c0 + tx)] = tile[tx][ty + k];
}
__global__ void __launch_bounds__(256) out32(const double* __restrict__ yp, uint64_t ldp, const uint32_t* __restrict__ ip,
                                             double* __restrict__ y, uint64_t ldy, uint32_t n, uint32_t q) {
  __shared__ double tile[32][33];
  const uint32_t r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) tile[ty + k][tx] = __ldg(yp + (uint64_t)ip[r0 + ty + k] * ldp + phys(c0 + tx));
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) y[r0 + tx + (uint64_t)(c0 + ty + k) * ldy] = tile[tx][ty + k];
}

// P points x 64 columns per CTA (one column block): columns read as P*8-byte segments, point rows
// written as whole 512-byte block rows (a warp per row, two 256-byte stores).
template <int P>
__global__ void __launch_bounds__(256) in_blk(const double* __restrict__ w, uint64_t ldw, const uint32_t* __restrict__ ip,
                                              double* __restrict__ wp, uint64_t ldp, uint32_t n, uint32_t q) {
  __shared__ double tile[64][P + 1];  // [column][point]
  __shared__ uint32_t rows[P];
  const uint32_t r0 = blockIdx.x * P, c0 = blockIdx.y * 64;
  const int t = threadIdx.x;
  if (t < P) rows[t] = ip[r0 + t];
  constexpr int kPer = 64 * P / 256;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = k * 256 + t, pt = e % P, col = e / P;
    tile[col][pt] = __ldg(w + r0 + pt + (uint64_t)(c0 + col) * ldw);
  }
  __syncthreads();
  // a warp per point row: lane l stores columns 2l, 2l+1
  const int warp = t >> 5, lane = t & 31;
#pragma unroll
  for (int k = 0; k < P / 8; ++k) {
    const int pt = warp + 8 * k;
    double* row = wp + (uint64_t)rows[pt] * ldp + phys(c0);
    row[lane] = tile[lane][pt];  // (column pitch P + 1 doubles: conflict-free 64-bit reads)
    row[lane + 32] = tile[lane + 32][pt];
  }
}
template <int P>
__global__ void __launch_bounds__(256) out_blk(const double* __restrict__ yp, uint64_t ldp, const uint32_t* __restrict__ ip,
                                               double* __restrict__ y, uint64_t ldy, uint32_t n, uint32_t q) {
  __shared__ double tile[64][P + 1];
  __shared__ uint32_t rows[P];
  const uint32_t r0 = blockIdx.x * P, c0 = blockIdx.y * 64;
  const int t = threadIdx.x;
  if (t < P) rows[t] = ip[r0 + t];
  __syncthreads();
  const int warp = t >> 5, lane = t & 31;
#pragma unroll
  for (int k = 0; k < P / 8; ++k) {
    const int pt = warp + 8 * k;
    const double* row = yp + (uint64_t)rows[pt] * ldp + phys(c0);
    tile[lane][pt] = __ldg(row + lane);
    tile[lane + 32][pt] = __ldg(row + lane + 32);
  }
  __syncthreads();
  constexpr int kPer = 64 * P / 256;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = k * 256 + t, pt = e % P, col = e / P;
    y[r0 + pt + (uint64_t)(c0 + col) * ldy] = tile[col][pt];
  }
}
__global__ void __launch_bounds__(256) copy16(const double2* __restrict__ a, double2* __restrict__ b, uint64_t n2) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n2; i += gridDim.x * 256ull) b[i] = __ldg(a + i);
}

int main() {
  const uint32_t n = 262144, q = 2048;
  const uint64_t ldp = (q + 63) / 64 * 80;
  std::vector<uint32_t> p(n);
  for (uint32_t i = 0; i < n; ++i) p[i] = i;
  std::mt19937 g(1);
  std::shuffle(p.begin(), p.end(), g);
  double *w, *wp, *wp2, *y, *y2;
  uint32_t* ip;
  cudaMalloc(&w, (size_t)n * q * 8);
  cudaMalloc(&y, (size_t)n * q * 8);
  cudaMalloc(&y2, (size_t)n * q * 8);
  cudaMalloc(&wp, (size_t)n * ldp * 8);
  cudaMalloc(&wp2, (size_t)n * ldp * 8);
  cudaMalloc(&ip, n * 4);
  cudaMemcpy(ip, p.data(), n * 4, cudaMemcpyHostToDevice);
  std::vector<double> hw((size_t)n * q);
  for (size_t i = 0; i < hw.size(); ++i) hw[i] = (double)(i % 1000003);
  cudaMemcpy(w, hw.data(), hw.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(wp, 0, (size_t)n * ldp * 8);
  cudaMemset(wp2, 0, (size_t)n * ldp * 8);
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
    printf("%-12s %.3f ms  %.2f TB/s (16 B per element moved)  %s\n", name, ms, 16.0 * n * q / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("copy", [&] { copy16<<<148 * 16, 256>>>((const double2*)w, (double2*)y, (uint64_t)n * q / 2); });
  run("in32", [&] { in32<<<dim3(n / 32, q / 32), 256>>>(w, n, ip, wp, ldp, n, q); });
  run("in_blk<32>", [&] { in_blk<32><<<dim3(n / 32, q / 64), 256>>>(w, n, ip, wp2, ldp, n, q); });
  run("in_blk<64>", [&] { in_blk<64><<<dim3(n / 64, q / 64), 256>>>(w, n, ip, wp2, ldp, n, q); });
  run("in_blk<16>", [&] { in_blk<16><<<dim3(n / 16, q / 64), 256>>>(w, n, ip, wp2, ldp, n, q); });
  run("out32", [&] { out32<<<dim3(n / 32, q / 32), 256>>>(wp, ldp, ip, y, n, n, q); });
  run("out_blk<32>", [&] { out_blk<32><<<dim3(n / 32, q / 64), 256>>>(wp, ldp, ip, y2, n, n, q); });
  run("out_blk<64>", [&] { out_blk<64><<<dim3(n / 64, q / 64), 256>>>(wp, ldp, ip, y2, n, n, q); });
  run("out_blk<16>", [&] { out_blk<16><<<dim3(n / 16, q / 64), 256>>>(wp, ldp, ip, y2, n, n, q); });
  // checks: the block variants against the 32 x 32 ones, and the round trip against W
  std::vector<double> h1((size_t)n * 64), h2((size_t)n * 64);
  size_t bad = 0;
  for (uint32_t r = 0; r < n; r += 997)
    for (uint32_t c = 0; c < q; c += 61) {
      double v1, v2;
      cudaMemcpy(&v1, wp + (uint64_t)r * ldp + phys(c), 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&v2, wp2 + (uint64_t)r * ldp + phys(c), 8, cudaMemcpyDeviceToHost);
      bad += v1 != v2;
    }
  std::vector<double> hy((size_t)n * 8);
  cudaMemcpy(hy.data(), y2, hy.size() * 8, cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < hy.size(); ++i) bad += hy[i] != hw[i];
  cudaMemcpy(hy.data(), y, hy.size() * 8, cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < hy.size(); ++i) bad += hy[i] != hw[i];
  printf("mismatches: %zu\n", bad);
  return 0;
}
