// Microbenchmark: dependent-chain latency of FP64 ops on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-9, y = b;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; i++) x = fma(x, y, 1e-3);
  t1 = clock64(); cyc[0] = t1 - t0;
  // division chain
  t0 = clock64();
  for (int i = 0; i < n; i++) x = 1.0 / (x + 1.5);
  t1 = clock64(); cyc[1] = t1 - t0;
  // shuffle chain
  t0 = clock64();
  for (int i = 0; i < n; i++) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); cyc[2] = t1 - t0;
  // independent DFMA throughput (8 chains)
  double z[8];
  for (int j = 0; j < 8; j++) z[j] = x + j;
  t0 = clock64();
  for (int i = 0; i < n; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) z[j] = fma(z[j], y, 1e-3);
  t1 = clock64(); cyc[3] = t1 - t0;
  for (int j = 0; j < 8; j++) x += z[j];
  // DMMA m8n8k4 dependent chain and 4 independent chains
  {
    double c[2] = {x, x}, c2[4][2] = {{x, x}, {x, x}, {x, x}, {x, x}};
    t0 = clock64();
    for (int i = 0; i < n; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[0]), "+d"(c[1]) : "d"(y), "d"(y));
    t1 = clock64(); cyc[5] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; i++)
#pragma unroll
      for (int j = 0; j < 4; j++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c2[j][0]), "+d"(c2[j][1]) : "d"(y), "d"(y));
    t1 = clock64(); cyc[6] = t1 - t0;
    x += c[0] + c2[0][1] + c2[3][0];
  }
  // rcp.approx
  t0 = clock64();
  for (int i = 0; i < n; i++) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.5; }
  t1 = clock64(); cyc[7] = t1 - t0;
  // bar.sync round trip (all warps of the CTA)
  t0 = clock64();
  for (int i = 0; i < n; i++) __syncthreads();
  t1 = clock64(); cyc[4] = t1 - t0;
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64 * 8);
  const int n = 1000;
  for (int nt : {32, 256}) {
    lat<<<1, nt>>>(o, c, 1.0001, 0.9999, n);
    cudaDeviceSynchronize();
    printf("threads %d: dfma lat %.1f  div lat %.1f  shfl lat %.1f  dfma x8 %.1f/iter  bar %.1f  dmma lat %.1f  dmma x4 %.1f/iter  rcp.approx+add %.1f cycles\n",
           nt, c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n,
           c[5] / (double)n, c[6] / (double)n, c[7] / (double)n);
  }
  return 0;
}
