// Dependent-issue latency of FP64 DMMA.8x8x4 and of DFMA on one warp (clock64 around a chain),
// and the chain throughput with 1, 2, 4, 8, 16 independent accumulators per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat tools/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chain(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c[C][2];
#pragma unroll
  for (int t = 0; t < C; ++t) c[t][0] = c[t][1] = 0.0;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < C; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int t = 0; t < C; ++t) s += c[t][0] + c[t][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void fchain(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 1.0000001, 1e-9);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// ns per dependent load, every warp of every CTA chasing its own chain (lane 0)
__global__ void l2lat_ns(const double* __restrict__ p, unsigned long long* ns, int n, double* out, unsigned span) {
  unsigned idx = (blockIdx.x * 7919u + threadIdx.x * 104729u) % span;
  double s = 0;
  __syncthreads();
  const unsigned long long t0 = gt();
  for (int i = 0; i < n; ++i) {
    double v = __ldcg(p + idx);
    s += v;
    idx = (idx + 4099u + static_cast<unsigned>(v)) % span;
  }
  const unsigned long long t1 = gt();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + threadIdx.x / 32] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *ns = t1 - t0;
}
// MLP: per round, 16 independent loads per thread (ld.cg / ld.global.nc / plain), then a
// dependent step; ns per round
template <int MODE>
__global__ void mlp(const double* __restrict__ p, unsigned long long* ns, int rounds, double* out, unsigned span) {
  unsigned idx = (blockIdx.x * 7919u + threadIdx.x * 104729u) % span;
  double s = 0;
  const unsigned long long t0 = gt();
  for (int r = 0; r < rounds; ++r) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double* a = p + (idx + u * 977u) % span;
      v[u] = MODE == 0 ? __ldcg(a) : (MODE == 1 ? __ldg(a) : *a);
    }
    double t = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) t += v[u];
    s += t;
    idx = (idx + 4099u + static_cast<unsigned>(t)) % span;
  }
  const unsigned long long t1 = gt();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *ns = t1 - t0;
}
__global__ void l2lat(const double* __restrict__ p, long long* cyc, int n, double* out) {
  // pointer-chase-free: dependent loads through the loaded value's bits
  unsigned idx = 0;
  double s = 0;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double v = __ldcg(p + idx);
    s += v;
    idx = (idx + 4099u + static_cast<unsigned>(v)) % (1u << 20);
  }
  const long long t1 = clock64();
  out[0] = s;
  *cyc = t1 - t0;
}
template <int C>
void run(double* out, long long* cyc) {
  const int iters = 1024;
  chain<C><<<1, 32>>>(out, cyc, 16);
  chain<C><<<1, 32>>>(out, cyc, iters);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA chains=%2d: %.1f cycles per chain step, %.1f cycles per DMMA\n", C, double(h) / iters, double(h) / iters / C);
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 << 20);
  cudaMalloc(&cyc, 8);
  cudaMemset(out, 0, 8 << 20);
  run<1>(out, cyc);
  run<2>(out, cyc);
  run<4>(out, cyc);
  run<8>(out, cyc);
  run<16>(out, cyc);
  fchain<<<1, 32>>>(out, cyc, 4096);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent: %.1f cycles\n", double(h) / 4096);
  double* buf;
  cudaMalloc(&buf, 8 << 20);
  cudaMemset(buf, 0, 8 << 20);
  l2lat<<<1, 1>>>(buf, cyc, 64, out);
  l2lat<<<1, 1>>>(buf, cyc, 4096, out);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("L2 dependent load (8 MB buffer, ld.cg): %.1f cycles\n", double(h) / 4096);
  unsigned long long* ns;
  cudaMalloc(&ns, 8);
  for (int blocks : {1, 64, 444})
    for (int threads : {32, 160}) {
      l2lat_ns<<<blocks, threads>>>(buf, ns, 64, out, 1u << 20);
      l2lat_ns<<<blocks, threads>>>(buf, ns, 2048, out, 1u << 20);
      unsigned long long hn;
      cudaMemcpy(&hn, ns, 8, cudaMemcpyDeviceToHost);
      printf("L2 dependent load, %d CTAs x %d threads (8 MB): %.1f ns\n", blocks, threads, double(hn) / 2048);
    }
  for (int mode = 0; mode < 3; ++mode) {
    unsigned long long hn;
    auto k = mode == 0 ? mlp<0> : (mode == 1 ? mlp<1> : mlp<2>);
    k<<<64, 160>>>(buf, ns, 8, out, 1u << 20);
    k<<<64, 160>>>(buf, ns, 256, out, 1u << 20);
    cudaMemcpy(&hn, ns, 8, cudaMemcpyDeviceToHost);
    printf("16 independent loads (%s), 64 x 160: %.1f ns per round\n", mode == 0 ? "ld.cg" : (mode == 1 ? "ld.nc" : "ld"), double(hn) / 256);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
