// Microbenchmark: FP64 DMMA (mma.sync m8n8k4.f64) vs DFMA throughput on sm_100a.
// Used once to fix the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, iters = 4096;
      dmma_loop<<<blocks, threads>>>(d, 64);
      cudaEventRecord(e0);
      dmma_loop<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * (blocks * threads / 32);
      printf("DMMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
      dfma_loop<<<blocks, threads>>>(d, 64);
      cudaEventRecord(e0);
      dfma_loop<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * (double)iters * blocks * threads;
      printf("DFMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
