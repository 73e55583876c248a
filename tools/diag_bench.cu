// Standalone timing of the large-front diagonal-block kernels on one synthetic
// front (m x k panel of a diagonally dominant symmetric matrix), with the
// per-phase clock stamps of CTA 0.  Build: see tools/diag_bench.sh.
#define TFB_PHASE_CLOCK 1
#include "../paper_2306_08994_b200/csrc/factor_large.cu"
#include <cstdio>
#include <vector>
namespace tfb {
int g_small_max_m = 112;
void timer_begin(int, cudaStream_t) {}
void timer_end(cudaStream_t) {}
}
using namespace tfb;
int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 1024, k = argc > 2 ? atoi(argv[2]) : 256;
  const int nf = argc > 3 ? atoi(argv[3]) : 4;
  const int kp = (k + 3) / 4 * 4;
  const long long fac = (long long)m * kp + kp;
  std::vector<int> pat(TF_PAT_WIDTH, 0);
  pat[TF_PAT_M] = m; pat[TF_PAT_K] = k; pat[TF_PAT_KP] = kp; pat[TF_PAT_FAC] = (int)fac;
  std::vector<int> pof(nf, 0);
  std::vector<long long> poff(nf);
  for (int i = 0; i < nf; i++) poff[i] = (long long)i * k;
  std::vector<double> P(fac * nf);
  for (int f = 0; f < nf; f++)
    for (int r = 0; r < m; r++)
      for (int c = 0; c < kp; c++)
        P[f * fac + (long long)r * kp + c] = (c < k && c <= r) ? (r == c ? 4.0 * m : 1.0 / (1 + r + c)) : 0.0;
  int *dpat, *dpof; long long* dpoff; double *dP, *dP0, *daux; unsigned long long* derr;
  cudaMalloc(&dpat, pat.size() * 4); cudaMalloc(&dpof, nf * 4); cudaMalloc(&dpoff, nf * 8);
  cudaMalloc(&dP, P.size() * 8); cudaMalloc(&dP0, P.size() * 8);
  const long long auxs = large_aux_doubles(k);
  cudaMalloc(&daux, auxs * nf * 8); cudaMalloc(&derr, 8);
  cudaMemcpy(dpat, pat.data(), pat.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dpof, pof.data(), nf * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dpoff, poff.data(), nf * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dP0, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
  LevelArgs L{};
  L.n_fronts = nf; L.max_m = m; L.max_k = k; L.max_upd = m - k; L.fac_stride = fac;
  L.pattern_of = dpof; L.piv_off = dpoff; L.pat = dpat; L.aux = daux; L.aux_stride = auxs;
  L.level_fronts = nf;
  cudaFuncSetAttribute(large_diag64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem);
  cudaFuncSetAttribute(large_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBlockSmem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 20;
  for (int which = 0; which < 2; which++) {
    float best = 1e9;
    for (int it = 0; it < reps; it++) {
      cudaMemcpy(dP, dP0, P.size() * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      if (which == 0)
        large_diag64_kernel<<<nf, 256, kDiagSmem>>>(L, dP, 0, 1e-300, derr);
      else
        large_block_kernel<<<dim3(nf, (m - 64 + 63) / 64), 256, kBlockSmem>>>(L, dP, 0, 1e-300, derr);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    long long clk[32];
    cudaMemcpyFromSymbol(clk, g_phase_clk, sizeof(clk));
    printf("%s: best %.2f us  (m=%d k=%d fronts=%d) err=%s\n", which ? "block" : "diag64", best * 1e3,
           m, k, nf, cudaGetErrorString(cudaGetLastError()));
    if (which == 0) {
      const char* names[] = {"start", "load", "pan0", "upd0", "pan1", "upd1", "pan2", "upd2", "pan3",
                             "upd3", "inv16", "lvl32", "lvl64", "end"};
      for (int i = 1; i < 14; i++)
        if (clk[i] > clk[0]) printf("  %-6s +%6lld cyc\n", names[i], clk[i] - clk[0]);
    }
  }
  return 0;
}
