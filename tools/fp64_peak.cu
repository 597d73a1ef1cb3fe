// FP64 peak measuring stick for the roofline denominator:
// DFMA (SIMT) vs DMMA (mma.sync .f64) throughput on one B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma884_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = (threadIdx.x + t) * 1e-3;
#pragma unroll
  for (int t = 0; t < 4; ++t) b[t] = 1.0 - (threadIdx.x + t) * 1e-3;
  double c[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) c[t][0] = c[t][1] = c[t][2] = c[t][3] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps; int iters = 4096;
      float ms;
      dfma_loop<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
      cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 64 * iters * (double)blocks * threads;
      printf("DFMA      threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
      dmma884_loop<<<blocks, threads>>>(out, 16);
      cudaEventRecord(e0); dmma884_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 8 * 256 * iters * (double)blocks * (threads / 32);
      printf("DMMA884   threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
      dmma16816_loop<<<blocks, threads>>>(out, 16);
      cudaEventRecord(e0); dmma16816_loop<<<blocks, threads>>>(out, iters / 4); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 4 * 2048 * (iters / 4) * (double)blocks * (threads / 32);
      printf("DMMA16816 threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
