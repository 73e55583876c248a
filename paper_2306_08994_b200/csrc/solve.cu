// Level sweeps of the triangular solve, nrhs right-hand sides at once.
//
// Reference (engine.py:468-493), single RHS:
//   forward : for z in pivot order: b[x] -= l(x,z) * b[z]        (481-485)
//   scale   : b[z] /= u(z,z)                                      (486-487)
//   backward: for z reversed: b[z] -= sum_y u(z,y) * b[y]         (488-492)
// Vectors are row-major (n x nrhs) in pivot order.  The forward sweep is
// multifrontal: a front's block W (m x nrhs) starts as its pivot rows of b
// (zeros on shared rows) plus its children's update rows, eliminates its k
// pivots and leaves rows [k, m) as its update for the parent.  The backward
// sweep gathers the shared rows of x from the parent's block through the same
// extend-add maps.  Small fronts: one thread group per front, block in shared
// memory.  Large fronts: blocked (64-row diagonal solves + multi-CTA
// matrix-vector updates), block in global memory.
#include "common.cuh"

namespace tfb {

constexpr int SB = 64;  // diagonal block rows of the large-front sweeps

// ------------------------------------------------------------- small fronts
template <int G, int GPC>
__global__ void __launch_bounds__(G* GPC)
    solve_fwd_small(LevelArgs L, LevelArgs C, const double* __restrict__ factors,
                    const double* __restrict__ w_child, long long child_rows, double* w_out,
                    long long out_rows, double* y, int nrhs, int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / G, t = threadIdx.x - gid * G, bar = 1 + gid;
  const long long f = (long long)blockIdx.x * GPC + gid;
  if (f >= L.n_fronts) return;
  double* W = reinterpret_cast<double*>(smem_raw + (size_t)gid * smem_per_group);
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Lp = factors + f * L.fac_stride;
  const int nW = m * nrhs, nK = k * nrhs;
  for (int e = t; e < nW; e += G) W[e] = e < nK ? y[piv * nrhs + e] : 0.0;
  group_sync<G>(bar);
  if (!L.is_leaf) {
    for (int c = 0; c < s.nsrc; c++) {
      const long long ch = 2 * f + c;
      const int kc = C.pat[(size_t)C.pattern_of[ch] * TF_PAT_WIDTH + TF_PAT_K];
      const int len = c == 0 ? s.len0 : s.len1;
      const int* mp = L.maps + (c == 0 ? s.off0 : s.off1);
      const double* Wc = w_child + ch * child_rows * nrhs + (long long)kc * nrhs;
      const int n = len * nrhs;
      for (int e = t; e < n; e += G) {
        const int a = e / nrhs, j = e - a * nrhs;
        W[mp[a] * nrhs + j] += Wc[e];
      }
      group_sync<G>(bar);
    }
  }
  for (int c = 0; c < k; c++) {
    const int n = (m - c - 1) * nrhs;
    const double* Wc = W + c * nrhs;
    for (int e = t; e < n; e += G) {
      const int r = c + 1 + e / nrhs, j = e % nrhs;
      W[r * nrhs + j] -= Lp[(long long)r * kp + c] * Wc[j];
    }
    group_sync<G>(bar);
  }
  const double* dv = Lp + (long long)m * kp;
  for (int e = t; e < nK; e += G) y[piv * nrhs + e] = W[e] / dv[e / nrhs];
  double* out = w_out + f * out_rows * nrhs;
  for (int e = nK + t; e < nW; e += G) out[e] = W[e];
}

template <int G, int GPC>
__global__ void __launch_bounds__(G* GPC)
    solve_bwd_small(LevelArgs L, LevelArgs PA, int has_parent, const double* __restrict__ factors,
                    const double* __restrict__ x_parent, long long parent_rows, double* x_out,
                    long long out_rows, double* y, int nrhs, int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / G, t = threadIdx.x - gid * G, bar = 1 + gid;
  const long long f = (long long)blockIdx.x * GPC + gid;
  if (f >= L.n_fronts) return;
  double* X = reinterpret_cast<double*>(smem_raw + (size_t)gid * smem_per_group);
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Lp = factors + f * L.fac_stride;
  const int nW = m * nrhs, nK = k * nrhs;
  for (int e = t; e < nK; e += G) X[e] = y[piv * nrhs + e];
  if (has_parent && m > k) {
    const long long pf = f >> 1;
    const int c = (int)(f & 1);
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    const int* mp = PA.maps + (c == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    const double* Xp = x_parent + pf * parent_rows * nrhs;
    for (int e = nK + t; e < nW; e += G) {
      const int a = (e - nK) / nrhs, j = (e - nK) % nrhs;
      X[e] = Xp[(long long)mp[a] * nrhs + j];
    }
  }
  group_sync<G>(bar);
  if (m > k) {
    for (int e = t; e < nK; e += G) {
      const int c = e / nrhs, j = e - c * nrhs;
      double acc = X[e];
      for (int r = k; r < m; r++) acc -= Lp[(long long)r * kp + c] * X[r * nrhs + j];
      X[e] = acc;
    }
    group_sync<G>(bar);
  }
  for (int c = k - 1; c > 0; c--) {
    const double* Xc = X + c * nrhs;
    const int n = c * nrhs;
    for (int e = t; e < n; e += G) {
      const int r = e / nrhs, j = e - r * nrhs;
      X[e] -= Lp[(long long)c * kp + r] * Xc[j];
    }
    group_sync<G>(bar);
  }
  for (int e = t; e < nK; e += G) y[piv * nrhs + e] = X[e];
  if (!L.is_leaf) {
    double* out = x_out + f * out_rows * nrhs;
    for (int e = t; e < nW; e += G) out[e] = X[e];
  }
}

// ------------------------------------------------------------- large fronts
__global__ void solve_gather_fwd(LevelArgs L, LevelArgs C, const double* __restrict__ w_child,
                                 long long child_rows, double* W, long long out_rows,
                                 const double* __restrict__ y, int nrhs) {
  const long long f = blockIdx.y;
  const Shape s = front_shape(L, f);
  const long long piv = L.piv_off[f];
  const int nW = s.m * nrhs, nK = s.k * nrhs;
  int kc[2] = {0, 0};
  for (int c = 0; c < s.nsrc && !L.is_leaf; c++)
    kc[c] = C.pat[(size_t)C.pattern_of[2 * f + c] * TF_PAT_WIDTH + TF_PAT_K];
  double* Wf = W + f * out_rows * nrhs;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nW; e += gridDim.x * blockDim.x) {
    const int r = e / nrhs, j = e - r * nrhs;
    double v = e < nK ? y[piv * nrhs + e] : 0.0;
    if (!L.is_leaf) {
      for (int c = 0; c < s.nsrc; c++) {
        const int i = L.maps[s.ioff + c * s.m + r];
        if (i >= 0)
          v += w_child[(2 * f + c) * child_rows * nrhs + (long long)(kc[c] + i) * nrhs + j];
      }
    }
    Wf[e] = v;
  }
}

__global__ void __launch_bounds__(256) solve_fwd_diag(LevelArgs L, const double* __restrict__ factors,
                                                       double* W, long long out_rows, double* y,
                                                       int nrhs, int j0) {
  extern __shared__ __align__(16) double sm[];
  double* Lb = sm;                 // [SB][SB+1]
  double* Wb = sm + SB * (SB + 1); // [SB][nrhs]
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(j0 + SB, s.k) - j0;
  if (kb <= 0) return;
  const double* Lp = factors + f * L.fac_stride;
  double* Wf = W + f * out_rows * nrhs;
  for (int e = threadIdx.x; e < kb * SB; e += blockDim.x) {
    const int i = e / SB, j = e - i * SB;
    if (j < i) Lb[i * (SB + 1) + j] = Lp[(long long)(j0 + i) * s.kp + j0 + j];
  }
  const int n = kb * nrhs;
  for (int e = threadIdx.x; e < n; e += blockDim.x) Wb[e] = Wf[(long long)j0 * nrhs + e];
  __syncthreads();
  for (int c = 0; c < kb - 1; c++) {
    const int nn = (kb - c - 1) * nrhs;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      const int r = c + 1 + e / nrhs, j = e % nrhs;
      Wb[r * nrhs + j] -= Lb[r * (SB + 1) + c] * Wb[c * nrhs + j];
    }
    __syncthreads();
  }
  const double* dv = Lp + (long long)s.m * s.kp + j0;
  const long long piv = L.piv_off[f] + j0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    Wf[(long long)j0 * nrhs + e] = Wb[e];
    y[piv * nrhs + e] = Wb[e] / dv[e / nrhs];
  }
}

__global__ void __launch_bounds__(256) solve_fwd_gemv(LevelArgs L, const double* __restrict__ factors,
                                                       double* W, long long out_rows, int nrhs,
                                                       int j0) {
  extern __shared__ __align__(16) double sm[];  // Wb [SB][nrhs]
  const long long f = blockIdx.y;
  const Shape s = front_shape(L, f);
  const int kb = min(j0 + SB, s.k) - j0;
  if (kb <= 0) return;
  const int r0 = j0 + kb + blockIdx.x * SB;
  if (r0 >= s.m) return;
  const double* Lp = factors + f * L.fac_stride;
  double* Wf = W + f * out_rows * nrhs;
  for (int e = threadIdx.x; e < kb * nrhs; e += blockDim.x) sm[e] = Wf[(long long)j0 * nrhs + e];
  __syncthreads();
  const int rows = min(SB, s.m - r0);
  for (int e = threadIdx.x; e < rows * nrhs; e += blockDim.x) {
    const int rl = e / nrhs, j = e - rl * nrhs;
    const long long r = r0 + rl;
    const double* lrow = Lp + r * s.kp + j0;
    double acc = Wf[r * nrhs + j];
    for (int q = 0; q < kb; q++) acc -= lrow[q] * sm[q * nrhs + j];
    Wf[r * nrhs + j] = acc;
  }
}

__global__ void solve_gather_bwd(LevelArgs L, LevelArgs PA, int has_parent,
                                 const double* __restrict__ x_parent, long long parent_rows,
                                 double* X, long long out_rows, const double* __restrict__ y,
                                 int nrhs) {
  const long long f = blockIdx.y;
  const Shape s = front_shape(L, f);
  const long long piv = L.piv_off[f];
  const int nW = s.m * nrhs, nK = s.k * nrhs;
  double* Xf = X + f * out_rows * nrhs;
  const int* mp = nullptr;
  const double* Xp = nullptr;
  if (has_parent) {
    const long long pf = f >> 1;
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    mp = PA.maps + ((f & 1) == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    Xp = x_parent + pf * parent_rows * nrhs;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nW; e += gridDim.x * blockDim.x) {
    if (e < nK) {
      Xf[e] = y[piv * nrhs + e];
    } else {
      const int a = (e - nK) / nrhs, j = (e - nK) % nrhs;
      Xf[e] = Xp[(long long)mp[a] * nrhs + j];
    }
  }
}

// X1[c][j] -= sum_{r in [k, m)} L[r][c] X[r][j]
__global__ void solve_bwd_shared(LevelArgs L, const double* __restrict__ factors, double* X,
                                 long long out_rows, int nrhs) {
  const long long f = blockIdx.y;
  const Shape s = front_shape(L, f);
  if (s.m == s.k) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= s.k * nrhs) return;
  const int j = e / s.k, c = e - j * s.k;  // c fastest: coalesced panel reads
  const double* Lp = factors + f * L.fac_stride;
  double* Xf = X + f * out_rows * nrhs;
  double acc = Xf[(long long)c * nrhs + j];
  for (int r = s.k; r < s.m; r++) acc -= Lp[(long long)r * s.kp + c] * Xf[(long long)r * nrhs + j];
  Xf[(long long)c * nrhs + j] = acc;
}

__global__ void __launch_bounds__(256) solve_bwd_diag(LevelArgs L, const double* __restrict__ factors,
                                                       double* X, long long out_rows, double* y,
                                                       int nrhs, int j0) {
  extern __shared__ __align__(16) double sm[];
  double* Lb = sm;
  double* Xb = sm + SB * (SB + 1);
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(j0 + SB, s.k) - j0;
  if (kb <= 0) return;
  const double* Lp = factors + f * L.fac_stride;
  double* Xf = X + f * out_rows * nrhs;
  for (int e = threadIdx.x; e < kb * SB; e += blockDim.x) {
    const int i = e / SB, j = e - i * SB;
    if (j < i) Lb[i * (SB + 1) + j] = Lp[(long long)(j0 + i) * s.kp + j0 + j];
  }
  const int n = kb * nrhs;
  for (int e = threadIdx.x; e < n; e += blockDim.x) Xb[e] = Xf[(long long)j0 * nrhs + e];
  __syncthreads();
  for (int c = kb - 1; c > 0; c--) {
    const int nn = c * nrhs;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      const int r = e / nrhs, j = e - r * nrhs;
      Xb[e] -= Lb[c * (SB + 1) + r] * Xb[c * nrhs + j];
    }
    __syncthreads();
  }
  const long long piv = L.piv_off[f] + j0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    Xf[(long long)j0 * nrhs + e] = Xb[e];
    y[piv * nrhs + e] = Xb[e];
  }
}

// X[c][j] -= sum_{t < kb} L[j0+t][c] X[j0+t][j] for c < j0
__global__ void __launch_bounds__(256) solve_bwd_gemv(LevelArgs L, const double* __restrict__ factors,
                                                       double* X, long long out_rows, int nrhs,
                                                       int j0) {
  extern __shared__ __align__(16) double sm[];  // Xb [SB][nrhs]
  const long long f = blockIdx.y;
  const Shape s = front_shape(L, f);
  const int kb = min(j0 + SB, s.k) - j0;
  if (kb <= 0) return;
  const double* Lp = factors + f * L.fac_stride;
  double* Xf = X + f * out_rows * nrhs;
  const int e0 = blockIdx.x * blockDim.x;
  if (e0 >= j0 * nrhs) return;
  for (int e = threadIdx.x; e < kb * nrhs; e += blockDim.x) sm[e] = Xf[(long long)j0 * nrhs + e];
  __syncthreads();
  const int e = e0 + threadIdx.x;
  if (e >= j0 * nrhs) return;
  const int j = e / j0, c = e - j * j0;
  double acc = Xf[(long long)c * nrhs + j];
  for (int q = 0; q < kb; q++) acc -= Lp[(long long)(j0 + q) * s.kp + c] * sm[q * nrhs + j];
  Xf[(long long)c * nrhs + j] = acc;
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

// ------------------------------------------------------------------ launch
static bool small_solve_ok(const LevelArgs& L, int nrhs) {
  return L.max_m <= g_small_max_m && (size_t)L.max_m * nrhs * 8 <= 200 * 1024;
}

template <int G, int GPC, bool FWD>
static cudaError_t launch_small_solve(const LevelArgs& L, const LevelArgs& O, int flag,
                                      const double* factors, const double* w_in,
                                      long long in_rows, double* w_out, long long out_rows,
                                      double* y, int nrhs, cudaStream_t st) {
  const int per = (int)(((size_t)L.max_m * nrhs * 8 + 15) & ~(size_t)15);
  const size_t smem = (size_t)per * GPC;
  const unsigned blocks = (unsigned)((L.n_fronts + GPC - 1) / GPC);
  if (FWD) {
    auto kern = solve_fwd_small<G, GPC>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<blocks, G * GPC, smem, st>>>(L, O, factors, w_in, in_rows, w_out, out_rows, y, nrhs,
                                        per);
  } else {
    auto kern = solve_bwd_small<G, GPC>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<blocks, G * GPC, smem, st>>>(L, O, flag, factors, w_in, in_rows, w_out, out_rows, y,
                                        nrhs, per);
  }
  return cudaGetLastError();
}

template <bool FWD>
static cudaError_t dispatch_small(const LevelArgs& L, const LevelArgs& O, int flag,
                                  const double* factors, const double* w_in, long long in_rows,
                                  double* w_out, long long out_rows, double* y, int nrhs,
                                  cudaStream_t st) {
  const long long work = (long long)L.max_m * nrhs;
  const long long bytes = work * 8;
#define TFB_SMALL(G, GPC) \
  launch_small_solve<G, GPC, FWD>(L, O, flag, factors, w_in, in_rows, w_out, out_rows, y, nrhs, st)
  if (work <= 16 && bytes * 32 <= 160 * 1024) return TFB_SMALL(8, 32);
  if (work <= 64 && bytes * 16 <= 160 * 1024) return TFB_SMALL(16, 16);
  if (work <= 256 && bytes * 8 <= 160 * 1024) return TFB_SMALL(32, 8);
  if (work <= 2048 && bytes * 2 <= 160 * 1024) return TFB_SMALL(128, 2);
  return TFB_SMALL(256, 1);
#undef TFB_SMALL
}

cudaError_t launch_solve_fwd(const LevelArgs& L, const LevelArgs& C, const double* factors,
                             const double* w_child, long long child_rows, double* w_out,
                             long long out_rows, double* y, int nrhs, cudaStream_t st) {
  if (small_solve_ok(L, nrhs))
    return dispatch_small<true>(L, C, 0, factors, w_child, child_rows, w_out, out_rows, y, nrhs,
                                st);
  const unsigned nf = (unsigned)L.n_fronts;
  const long long nW = (long long)L.max_m * nrhs;
  solve_gather_fwd<<<dim3((unsigned)std::min<long long>((nW + 255) / 256, 1024), nf), 256, 0,
                     st>>>(L, C, w_child, child_rows, w_out, out_rows, y, nrhs);
  const size_t sm_diag = sizeof(double) * (SB * (SB + 1) + (size_t)SB * nrhs);
  const size_t sm_gemv = sizeof(double) * (size_t)SB * nrhs;
  cudaFuncSetAttribute(solve_fwd_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_diag);
  cudaFuncSetAttribute(solve_fwd_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_gemv);
  for (int j0 = 0; j0 < L.max_k; j0 += SB) {
    solve_fwd_diag<<<nf, 256, sm_diag, st>>>(L, factors, w_out, out_rows, y, nrhs, j0);
    const int rows = L.max_m - j0;
    solve_fwd_gemv<<<dim3((unsigned)((rows + SB - 1) / SB), nf), 256, sm_gemv, st>>>(
        L, factors, w_out, out_rows, nrhs, j0);
  }
  return cudaGetLastError();
}

cudaError_t launch_solve_bwd(const LevelArgs& L, const LevelArgs& PA, int has_parent,
                             const double* factors, const double* x_parent, long long parent_rows,
                             double* x_out, long long out_rows, double* y, int nrhs,
                             cudaStream_t st) {
  if (small_solve_ok(L, nrhs))
    return dispatch_small<false>(L, PA, has_parent, factors, x_parent, parent_rows, x_out,
                                 out_rows, y, nrhs, st);
  const unsigned nf = (unsigned)L.n_fronts;
  const long long nW = (long long)L.max_m * nrhs;
  solve_gather_bwd<<<dim3((unsigned)std::min<long long>((nW + 255) / 256, 1024), nf), 256, 0,
                     st>>>(L, PA, has_parent, x_parent, parent_rows, x_out, out_rows, y, nrhs);
  const long long nK = (long long)L.max_k * nrhs;
  solve_bwd_shared<<<dim3((unsigned)((nK + 127) / 128), nf), 128, 0, st>>>(L, factors, x_out,
                                                                            out_rows, nrhs);
  const size_t sm_diag = sizeof(double) * (SB * (SB + 1) + (size_t)SB * nrhs);
  const size_t sm_gemv = sizeof(double) * (size_t)SB * nrhs;
  cudaFuncSetAttribute(solve_bwd_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_diag);
  cudaFuncSetAttribute(solve_bwd_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_gemv);
  const int nblk = (L.max_k + SB - 1) / SB;
  for (int b = nblk - 1; b >= 0; b--) {
    const int j0 = b * SB;
    solve_bwd_diag<<<nf, 256, sm_diag, st>>>(L, factors, x_out, out_rows, y, nrhs, j0);
    if (j0 > 0) {
      const long long n = (long long)j0 * nrhs;
      solve_bwd_gemv<<<dim3((unsigned)((n + 255) / 256), nf), 256, sm_gemv, st>>>(
          L, factors, x_out, out_rows, nrhs, j0);
    }
  }
  return cudaGetLastError();
}

int solve_launches(const LevelArgs& L, int nrhs, bool fwd) {
  if (small_solve_ok(L, nrhs)) return 1;
  const int nblk = (L.max_k + SB - 1) / SB;
  return fwd ? 1 + 2 * nblk : 2 + nblk + (nblk > 0 ? nblk - 1 : 0);
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
