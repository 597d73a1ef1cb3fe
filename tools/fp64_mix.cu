// Do DFMA (SIMT FP64) and DMMA (mma.sync .f64) share one pipe on B200? Runs each alone and
// both together (warp-specialized: a fraction of the warps issue DFMA, the rest DMMA; and
// interleaved inside one warp). If the pipes were separate, the mixed rate would exceed
// either alone. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_block(double (&x)[8], double a, double b) {
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = fma(x[t], a, b);
}
__device__ __forceinline__ void dmma_block(double (&c)[8][2], double a, double b) {
#pragma unroll
  for (int t = 0; t < 8; ++t)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
}

// mode 0: all DMMA; 1: all DFMA; 2: warps w % split == 0 DFMA, others DMMA; 3: interleaved
__global__ void mixed(double* out, int iters, int mode, int split) {
  const int warp = threadIdx.x >> 5;
  double x[8];
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = threadIdx.x + t, c[t][0] = c[t][1] = 0.0;
  const double a = 1.0000001, b = 1e-9, ma = threadIdx.x * 1e-3, mb = 1.0 - threadIdx.x * 1e-3;
  const bool do_fma = mode == 1 || (mode == 2 && warp % split == 0);
  const bool do_mma = mode == 0 || (mode == 2 && warp % split != 0);
  if (mode == 3) {
    for (int i = 0; i < iters; ++i) {
      dmma_block(c, ma, mb);
      dfma_block(x, a, b);
    }
  } else if (do_fma) {
    for (int i = 0; i < iters; ++i) dfma_block(x, a, b);
  } else if (do_mma) {
    for (int i = 0; i < iters; ++i) dmma_block(c, ma, mb);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += x[t] + c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 4, iters = 4096;
  // flops per warp-iteration: DFMA block = 64 fma x 32 lanes x 2; DMMA block = 8 x 512
  const double f_fma = 64.0 * 32 * 2, f_mma = 8.0 * 512;
  struct Case { int mode, split; const char* name; };
  const Case cases[] = {{0, 1, "DMMA only"}, {1, 1, "DFMA only"}, {2, 2, "1/2 warps DFMA"},
                        {2, 4, "1/4 warps DFMA"}, {2, 8, "1/8 warps DFMA"}, {3, 1, "interleaved in-warp"}};
  for (const Case& cs : cases) {
    mixed<<<blocks, threads>>>(out, 16, cs.mode, cs.split);
    cudaEventRecord(e0);
    mixed<<<blocks, threads>>>(out, iters, cs.mode, cs.split);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const int warps = threads / 32;
    double fl = 0;
    for (int w = 0; w < warps; ++w) {
      bool f = cs.mode == 1 || (cs.mode == 2 && w % cs.split == 0);
      bool m = cs.mode == 0 || (cs.mode == 2 && w % cs.split != 0);
      if (cs.mode == 3) f = m = true;
      fl += (f ? f_fma : 0) + (m ? f_mma : 0);
    }
    fl *= static_cast<double>(iters) * blocks;
    printf("%-22s %.2f TFLOP/s (%.3f ms)\n", cs.name, fl / ms / 1e9, ms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
