// Level sweeps of the triangular solve, nrhs right-hand sides at once.
//
// Reference (engine.py:468-493), single RHS:
//   forward : for z in pivot order: b[x] -= l(x,z) * b[z]        (481-485)
//   scale   : b[z] /= u(z,z)                                      (486-487)
//   backward: for z reversed: b[z] -= sum_y u(z,y) * b[y]         (488-492)
// Here vectors are row-major (n x nrhs) in pivot order.  The forward sweep is
// multifrontal: a front's vector block W (m x nrhs) starts as the level's
// pivot rows of b (zeros on shared rows) plus its children's update rows,
// eliminates its k pivots, and leaves rows [k, m) as its update for the
// parent.  The backward sweep gathers the shared rows of x from the parent's
// front block through the same extend-add maps (no global index lists).
#include "common.cuh"

namespace tfb {

template <int G>
__global__ void __launch_bounds__(G) solve_fwd_kernel(LevelArgs L, LevelArgs C,
                                                      const double* __restrict__ factors,
                                                      const double* __restrict__ w_child,
                                                      long long child_rows, double* w_out,
                                                      long long out_rows, double* y, int nrhs) {
  const long long f = blockIdx.x;
  const int tid = threadIdx.x;
  const int* P = L.pat + (size_t)L.pattern_of[f] * TF_PAT_WIDTH;
  const int m = P[TF_PAT_M], k = P[TF_PAT_K], nsrc = P[TF_PAT_NSRC];
  const long long piv = L.piv_off[f];
  double* W = w_out + f * out_rows * nrhs;
  const double* Lp = factors + f * L.fac_stride;
  const long long nW = (long long)m * nrhs, nK = (long long)k * nrhs;
  for (long long e = tid; e < nW; e += G) W[e] = e < nK ? y[piv * nrhs + e] : 0.0;
  __syncthreads();
  if (!L.is_leaf) {
    for (int c = 0; c < nsrc; c++) {
      const long long ch = 2 * f + c;
      const int* PC = C.pat + (size_t)C.pattern_of[ch] * TF_PAT_WIDTH;
      const int kc = PC[TF_PAT_K];
      const int len = c == 0 ? P[TF_PAT_LEN0] : P[TF_PAT_LEN1];
      const int* mp = L.maps + (c == 0 ? P[TF_PAT_OFF0] : P[TF_PAT_OFF1]);
      const double* Wc = w_child + ch * child_rows * nrhs + (long long)kc * nrhs;
      const long long n = (long long)len * nrhs;
      for (long long e = tid; e < n; e += G) {
        const int a = (int)(e / nrhs), j = (int)(e - (long long)a * nrhs);
        W[(long long)mp[a] * nrhs + j] += Wc[e];
      }
      __syncthreads();
    }
  }
  for (int c = 0; c < k; c++) {
    const long long n = (long long)(m - c - 1) * nrhs;
    const double* Wcol = W + (long long)c * nrhs;
    for (long long e = tid; e < n; e += G) {
      const int r = c + 1 + (int)(e / nrhs), j = (int)(e % nrhs);
      W[(long long)r * nrhs + j] -= Lp[(long long)r * k + c] * Wcol[j];
    }
    __syncthreads();
  }
  for (long long e = tid; e < nK; e += G) {
    const int r = (int)(e / nrhs);
    y[piv * nrhs + e] = W[e] / Lp[(long long)r * k + r];
  }
}

template <int G>
__global__ void __launch_bounds__(G) solve_bwd_kernel(LevelArgs L, LevelArgs PA, int has_parent,
                                                      const double* __restrict__ factors,
                                                      const double* __restrict__ x_parent,
                                                      long long parent_rows, double* x_out,
                                                      long long out_rows, double* y, int nrhs) {
  const long long f = blockIdx.x;
  const int tid = threadIdx.x;
  const int* P = L.pat + (size_t)L.pattern_of[f] * TF_PAT_WIDTH;
  const int m = P[TF_PAT_M], k = P[TF_PAT_K];
  const long long piv = L.piv_off[f];
  double* X = x_out + f * out_rows * nrhs;
  const double* Lp = factors + f * L.fac_stride;
  const long long nK = (long long)k * nrhs, nW = (long long)m * nrhs;
  for (long long e = tid; e < nK; e += G) X[e] = y[piv * nrhs + e];
  if (has_parent && m > k) {
    const long long pf = f >> 1;
    const int c = (int)(f & 1);
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    const int* mp = PA.maps + (c == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    const double* Xp = x_parent + pf * parent_rows * nrhs;
    for (long long e = nK + tid; e < nW; e += G) {
      const int a = (int)((e - nK) / nrhs), j = (int)((e - nK) % nrhs);
      X[e] = Xp[(long long)mp[a] * nrhs + j];
    }
  }
  __syncthreads();
  if (m > k) {
    for (long long e = tid; e < nK; e += G) {
      const int r = (int)(e / nrhs), j = (int)(e % nrhs);
      double acc = X[e];
      for (int s = k; s < m; s++) acc -= Lp[(long long)s * k + r] * X[(long long)s * nrhs + j];
      X[e] = acc;
    }
    __syncthreads();
  }
  for (int c = k - 1; c > 0; c--) {
    const double* Xc = X + (long long)c * nrhs;
    const long long n = (long long)c * nrhs;
    for (long long e = tid; e < n; e += G) {
      const int r = (int)(e / nrhs), j = (int)(e % nrhs);
      X[e] -= Lp[(long long)c * k + r] * Xc[j];
    }
    __syncthreads();
  }
  for (long long e = tid; e < nK; e += G) y[piv * nrhs + e] = X[e];
}

__global__ void permute_rows_kernel(const int* __restrict__ idx, long long n,
                                    const double* __restrict__ in, double* __restrict__ out,
                                    int nrhs, int scatter) {
  const long long total = n * nrhs;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / nrhs;
    const int j = (int)(e - i * nrhs);
    const long long g = (long long)idx[i] - 1;
    if (scatter) out[g * nrhs + j] = in[e];
    else out[e] = in[g * nrhs + j];
  }
}

static int pick_threads(int max_m, int nrhs) {
  long long work = (long long)max_m * nrhs;
  if (work <= 64) return 32;
  if (work <= 512) return 128;
  return 256;
}

cudaError_t launch_solve_fwd(const LevelArgs& L, const LevelArgs& C, const double* factors,
                             const double* w_child, long long child_rows, double* w_out,
                             long long out_rows, double* y, int nrhs, cudaStream_t st) {
  const int G = pick_threads(L.max_m, nrhs);
  const unsigned nb = (unsigned)L.n_fronts;
  if (G == 32)
    solve_fwd_kernel<32><<<nb, 32, 0, st>>>(L, C, factors, w_child, child_rows, w_out, out_rows,
                                            y, nrhs);
  else if (G == 128)
    solve_fwd_kernel<128><<<nb, 128, 0, st>>>(L, C, factors, w_child, child_rows, w_out,
                                              out_rows, y, nrhs);
  else
    solve_fwd_kernel<256><<<nb, 256, 0, st>>>(L, C, factors, w_child, child_rows, w_out,
                                              out_rows, y, nrhs);
  return cudaGetLastError();
}

cudaError_t launch_solve_bwd(const LevelArgs& L, const LevelArgs& PA, int has_parent,
                             const double* factors, const double* x_parent, long long parent_rows,
                             double* x_out, long long out_rows, double* y, int nrhs,
                             cudaStream_t st) {
  const int G = pick_threads(L.max_m, nrhs);
  const unsigned nb = (unsigned)L.n_fronts;
  if (G == 32)
    solve_bwd_kernel<32><<<nb, 32, 0, st>>>(L, PA, has_parent, factors, x_parent, parent_rows,
                                            x_out, out_rows, y, nrhs);
  else if (G == 128)
    solve_bwd_kernel<128><<<nb, 128, 0, st>>>(L, PA, has_parent, factors, x_parent, parent_rows,
                                              x_out, out_rows, y, nrhs);
  else
    solve_bwd_kernel<256><<<nb, 256, 0, st>>>(L, PA, has_parent, factors, x_parent, parent_rows,
                                              x_out, out_rows, y, nrhs);
  return cudaGetLastError();
}

cudaError_t launch_permute_rows(const int* idx, long long n, const double* in, double* out,
                                int nrhs, int scatter, cudaStream_t st) {
  long long total = n * nrhs;
  unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148 * 16);
  if (blocks == 0) return cudaSuccess;
  permute_rows_kernel<<<blocks, 256, 0, st>>>(idx, n, in, out, nrhs, scatter);
  return cudaGetLastError();
}

}  // namespace tfb
