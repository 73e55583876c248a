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
// extend-add maps.
//   small fronts: one thread group per front, block in shared memory (RHS
//                 columns processed in slices that fit);
//   large fronts: blocked by the factorization's 64-wide diagonal blocks,
//                 using their stored unit-lower inverses M (aux): forward
//                 Y_b = M W_b then W_rows -= L_rows,b Y_b (one launch per
//                 block); backward X_b = M^T (X_b - sum_rows L_rows,b^T X_rows)
//                 with a deterministic two-pass reduction over row chunks.
#include "common.cuh"

namespace tfb {

constexpr int SB = 64;   // diagonal block rows (= factorization NB)
constexpr int RB = 128;  // rows per CTA in the large-front row sweeps

// ------------------------------------------------------------- small fronts
// Stage the front's panel (lower part, m x k, packed to leading dimension k)
// and its pivots d into shared memory with U loads in flight per thread.
template <int G>
__device__ __forceinline__ void stage_panel(double* Ls, const double* __restrict__ P, int m, int k,
                                            int kp, int t) {
  constexpr int U = 4;
  const int n = m * k;
  for (int e0 = t; e0 < n; e0 += G * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int e = e0 + u * G;
      const int r = e / k, c = e - r * k;
      v[u] = (e < n && c <= r) ? __ldg(P + (long long)r * kp + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int e = e0 + u * G;
      if (e < n) Ls[e] = v[u];
    }
  }
  for (int c = t; c < k; c += G) Ls[n + c] = __ldg(P + (long long)m * kp + c);
}

// Vectors: row stride ldr (total RHS columns); this launch handles columns
// [col0, col0 + nr).  With one column (nr == 1) every panel entry is used
// exactly once, so the panel is read straight from global memory and shared
// memory holds only the front's vector block (high occupancy); with several
// columns the panel is staged once and reused across them.
// Block conventions: the forward sweep of a small level writes a front's
// update rows only, at rows [0, m-k) of its block (no child-shape lookup for
// the parent); large levels work in place (update rows at [k, m)).  The
// backward sweep writes all m rows.
template <bool STAGE>
struct PanelRef {
  const double* p;
  int ld;
  __device__ __forceinline__ double operator()(int r, int c) const {
    return STAGE ? p[r * ld + c] : __ldg(p + (long long)r * ld + c);
  }
};

template <int G, int GPC, bool STAGE>
__global__ void __launch_bounds__(G* GPC)
    solve_fwd_small(LevelArgs L, LevelArgs C, const double* __restrict__ factors,
                    const double* __restrict__ w_child, long long child_rows, int child_at0,
                    double* w_out, long long out_rows, double* y, int nr, int ldr, int col0,
                    int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / G, t = threadIdx.x - gid * G, bar = 1 + gid;
  const long long f = (long long)blockIdx.x * GPC + gid;
  if (f >= L.n_fronts) return;
  double* W = reinterpret_cast<double*>(smem_raw + (size_t)gid * smem_per_group);
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pg = factors + f * L.fac_stride;
  PanelRef<STAGE> Lp{Pg, kp};
  const double* dv = Pg + (long long)m * kp;
  if (STAGE) {
    double* Ls = W + L.max_m * nr;  // panel staged in shared memory: Ls[r*k + c], then d
    stage_panel<G>(Ls, Pg, m, k, kp, t);
    Lp = PanelRef<STAGE>{Ls, k};
    dv = Ls + m * k;
  }
  const int nW = m * nr, nK = k * nr;
  for (int e = t; e < nW; e += G) {
    const int r = e / nr, j = e - r * nr;
    W[e] = e < nK ? y[(piv + r) * ldr + col0 + j] : 0.0;
  }
  group_sync<G>(bar);
  if (!L.is_leaf) {
    for (int c = 0; c < s.nsrc; c++) {
      const long long ch = 2 * (L.front_base + f) + c - C.front_base;
      const int off =
          child_at0 ? 0 : C.pat[(size_t)C.pattern_of[ch] * TF_PAT_WIDTH + TF_PAT_K];
      const int len = c == 0 ? s.len0 : s.len1;
      const int* mp = L.maps + (c == 0 ? s.off0 : s.off1);
      const double* Wc = w_child + (ch * child_rows + off) * ldr + col0;
      const int n = len * nr;
      for (int e = t; e < n; e += G) {
        const int a = e / nr, j = e - a * nr;
        W[mp[a] * nr + j] += Wc[(long long)a * ldr + j];
      }
      group_sync<G>(bar);
    }
  }
  // pivot block: right-looking inside the k x k triangle
  for (int c = 0; c < k; c++) {
    const int n = (k - c - 1) * nr;
    const double* Wc = W + c * nr;
    for (int e = t; e < n; e += G) {
      const int r = c + 1 + e / nr, j = e % nr;
      W[r * nr + j] -= Lp(r, c) * Wc[j];
    }
    group_sync<G>(bar);
  }
  for (int e = t; e < nK; e += G) {
    const int r = e / nr, j = e - r * nr;
    y[(piv + r) * ldr + col0 + j] = W[e] / dv[r];
  }
  // update rows: w_r - l_r . w_piv (row-contiguous panel reads), straight out
  double* out = w_out + f * out_rows * ldr + col0;
  for (int e = nK + t; e < nW; e += G) {
    const int r = e / nr, j = e - r * nr;
    double acc = W[e];
    for (int c = 0; c < k; c++) acc -= Lp(r, c) * W[c * nr + j];
    out[(long long)(r - k) * ldr + j] = acc;
  }
}

template <int G, int GPC, bool STAGE>
__global__ void __launch_bounds__(G* GPC)
    solve_bwd_small(LevelArgs L, LevelArgs PA, int has_parent, const double* __restrict__ factors,
                    const double* __restrict__ x_parent, long long parent_rows, double* x_out,
                    long long out_rows, double* y, int nr, int ldr, int col0,
                    int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / G, t = threadIdx.x - gid * G, bar = 1 + gid;
  const long long f = (long long)blockIdx.x * GPC + gid;
  if (f >= L.n_fronts) return;
  double* X = reinterpret_cast<double*>(smem_raw + (size_t)gid * smem_per_group);
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pg = factors + f * L.fac_stride;
  PanelRef<STAGE> Lp{Pg, kp};
  if (STAGE) {
    double* Ls = X + L.max_m * nr;
    stage_panel<G>(Ls, Pg, m, k, kp, t);
    Lp = PanelRef<STAGE>{Ls, k};
  }
  const int nW = m * nr, nK = k * nr;
  for (int e = t; e < nK; e += G) {
    const int r = e / nr, j = e - r * nr;
    X[e] = y[(piv + r) * ldr + col0 + j];
  }
  if (has_parent && m > k) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int c = (int)((L.front_base + f) & 1);
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    const int* mp = PA.maps + (c == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    const double* Xp = x_parent + pf * parent_rows * ldr + col0;
    for (int e = nK + t; e < nW; e += G) {
      const int a = (e - nK) / nr, j = (e - nK) % nr;
      X[e] = Xp[(long long)mp[a] * ldr + j];
    }
  }
  group_sync<G>(bar);
  if (m > k) {
    for (int e = t; e < nK; e += G) {
      const int c = e / nr, j = e - c * nr;
      double acc = X[e];
      for (int r = k; r < m; r++) acc -= Lp(r, c) * X[r * nr + j];
      X[e] = acc;
    }
    group_sync<G>(bar);
  }
  for (int c = k - 1; c > 0; c--) {
    const double* Xc = X + c * nr;
    const int n = c * nr;
    for (int e = t; e < n; e += G) {
      const int r = e / nr, j = e - r * nr;
      X[e] -= Lp(c, r) * Xc[j];
    }
    group_sync<G>(bar);
  }
  for (int e = t; e < nK; e += G) {
    const int r = e / nr, j = e - r * nr;
    y[(piv + r) * ldr + col0 + j] = X[e];
  }
  if (!L.is_leaf) {
    double* out = x_out + f * out_rows * ldr + col0;
    for (int e = t; e < nW; e += G) {
      const int r = e / nr, j = e - r * nr;
      out[(long long)r * ldr + j] = X[e];
    }
  }
}

// ------------------------------------------------------------- large fronts
__global__ void solve_gather_fwd(LevelArgs L, LevelArgs C, const double* __restrict__ w_child,
                                 long long child_rows, int child_at0, double* W,
                                 long long out_rows, const double* __restrict__ y, int nrhs) {
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const long long piv = L.piv_off[f];
  const int nW = s.m * nrhs, nK = s.k * nrhs;
  int kc[2] = {0, 0};
  for (int c = 0; c < s.nsrc; c++)  // update rows of a small child's block start at 0
    kc[c] = child_at0 ? 0
                      : C.pat[(size_t)C.pattern_of[2 * (L.front_base + f) + c - C.front_base] *
                                  TF_PAT_WIDTH + TF_PAT_K];
  double* Wf = W + f * out_rows * nrhs;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < nW; e += gridDim.y * blockDim.x) {
    const int r = e / nrhs, j = e - r * nrhs;
    double v = e < nK ? y[piv * nrhs + e] : 0.0;
    for (int c = 0; c < s.nsrc; c++) {
      const int i = L.maps[s.ioff + c * s.m + r];
      if (i >= 0) v += w_child[(2 * (L.front_base + f) + c - C.front_base) * child_rows * nrhs + (long long)(kc[c] + i) * nrhs + j];
    }
    Wf[e] = v;
  }
}

// Block j0: Y_b = M W_b (rows [j0, j0+kb)), y_b = Y_b / d; rows below: W_r -= L_r,b Y_b.
__global__ void __launch_bounds__(256) solve_fwd_block(LevelArgs L, const double* __restrict__ factors,
                                                        double* W, long long out_rows, double* y,
                                                        int nrhs, int j0) {
  extern __shared__ __align__(16) double sm[];
  double* Wb = sm;                 // [SB][nrhs] right-hand block
  double* Yb = sm + SB * nrhs;     // [SB][nrhs] solved block
  double* Ms = Yb + SB * nrhs;     // [SB][SB] diagonal-block inverse
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(j0 + SB, s.k) - j0;
  if (kb <= 0) return;
  const int j1 = j0 + kb;
  const int r0 = j1 + blockIdx.y * RB;
  if (blockIdx.y > 0 && r0 >= s.m) return;
  const double* Lp = factors + f * L.fac_stride;
  const double* M = L.aux + f * L.aux_stride + (long long)(j0 / SB) * SB * SB;
  double* Wf = W + f * out_rows * nrhs;
  const int n = kb * nrhs;
  for (int e = threadIdx.x; e < n; e += blockDim.x) Wb[e] = Wf[(long long)j0 * nrhs + e];
#pragma unroll 4
  for (int e = threadIdx.x; e < SB * SB; e += blockDim.x) Ms[e] = __ldg(M + e);
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int r = e / nrhs, j = e - r * nrhs;
    const double* mr = Ms + r * SB;
    double acc = Wb[e];  // M has a unit diagonal
    for (int q = 0; q < r; q++) acc += mr[q] * Wb[q * nrhs + j];
    Yb[e] = acc;
  }
  __syncthreads();
  if (blockIdx.y == 0) {
    const double* dv = Lp + (long long)s.m * s.kp + j0;
    const long long piv = L.piv_off[f] + j0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) y[piv * nrhs + e] = Yb[e] / dv[e / nrhs];
  }
  const int rows = min(RB, s.m - r0);
  if (nrhs == 1) {
    // warp per row, lanes across the 64 block columns: coalesced panel reads
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int rl = warp; rl < rows; rl += 8) {
      const double* lrow = Lp + (long long)(r0 + rl) * s.kp + j0;
      double acc = 0.0;
      if (lane < kb) acc = lrow[lane] * Yb[lane];
      if (lane + 32 < kb) acc += lrow[lane + 32] * Yb[lane + 32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) Wf[r0 + rl] -= acc;
    }
    return;
  }
  for (int e = threadIdx.x; e < rows * nrhs; e += blockDim.x) {
    const int rl = e / nrhs, j = e - rl * nrhs;
    const long long r = r0 + rl;
    const double* lrow = Lp + r * s.kp + j0;
    double acc = Wf[r * nrhs + j];
    for (int q = 0; q < kb; q++) acc -= lrow[q] * Yb[q * nrhs + j];
    Wf[r * nrhs + j] = acc;
  }
}

__global__ void solve_gather_bwd(LevelArgs L, LevelArgs PA, int has_parent,
                                 const double* __restrict__ x_parent, long long parent_rows,
                                 double* X, long long out_rows, const double* __restrict__ y,
                                 int nrhs) {
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const long long piv = L.piv_off[f];
  const int nW = s.m * nrhs, nK = s.k * nrhs;
  double* Xf = X + f * out_rows * nrhs;
  const int* mp = nullptr;
  const double* Xp = nullptr;
  if (has_parent) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    mp = PA.maps + (((L.front_base + f) & 1) == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    Xp = x_parent + pf * parent_rows * nrhs;
  }
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < nW; e += gridDim.y * blockDim.x) {
    if (e < nK) {
      Xf[e] = y[piv * nrhs + e];
    } else {
      const int a = (e - nK) / nrhs, j = (e - nK) % nrhs;
      Xf[e] = Xp[(long long)mp[a] * nrhs + j];
    }
  }
}

// partial[f][x][c][j] = sum_{r in chunk x of [j1, m)} L[r][j0+c] X[r][j]
__global__ void __launch_bounds__(256) solve_bwd_partial(LevelArgs L, const double* __restrict__ factors,
                                                          const double* __restrict__ X,
                                                          long long out_rows, int nrhs, int j0,
                                                          double* partial, int nchunk) {
  extern __shared__ __align__(16) double sm[];  // Xr [RB][nrhs]
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(j0 + SB, s.k) - j0;
  if (kb <= 0) return;
  const int j1 = j0 + kb;
  const int r0 = j1 + blockIdx.y * RB;
  double* P = partial + ((f * nchunk + blockIdx.y) * SB) * (long long)nrhs;
  const int n = kb * nrhs;
  if (r0 >= s.m) {
    for (int e = threadIdx.x; e < n; e += blockDim.x) P[e] = 0.0;
    return;
  }
  const double* Lp = factors + f * L.fac_stride;
  const double* Xf = X + f * out_rows * nrhs;
  const int rows = min(RB, s.m - r0);
  for (int e = threadIdx.x; e < rows * nrhs; e += blockDim.x) sm[e] = Xf[(long long)r0 * nrhs + e];
  __syncthreads();
  if (nrhs == 1) {
    // 64 columns x 4 row groups, fixed-order reduction of the 4 partial sums
    __shared__ double red[4][SB];
    const int c = threadIdx.x & (SB - 1), g = threadIdx.x >> 6;
    double acc = 0.0;
    if (c < kb) {
      const double* lcol = Lp + (long long)r0 * s.kp + j0 + c;
      for (int q = g; q < rows; q += 4) acc += lcol[(long long)q * s.kp] * sm[q];
    }
    red[g][c] = acc;
    __syncthreads();
    if (g == 0 && c < kb) P[c] = ((red[0][c] + red[1][c]) + red[2][c]) + red[3][c];
    return;
  }
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int j = e / kb, c = e - j * kb;  // c fastest: coalesced panel reads
    const double* lcol = Lp + (long long)r0 * s.kp + j0 + c;
    double acc = 0.0;
    for (int q = 0; q < rows; q++) acc += lcol[(long long)q * s.kp] * sm[q * nrhs + j];
    P[c * nrhs + j] = acc;
  }
}

// X_b = M^T (X_b - sum_x partial[x]); writes X rows [j0, j0+kb) and y.
__global__ void __launch_bounds__(256) solve_bwd_block(LevelArgs L, double* X, long long out_rows,
                                                        double* y, int nrhs, int j0,
                                                        const double* __restrict__ partial,
                                                        int nchunk) {
  extern __shared__ __align__(16) double sm[];  // Rb [SB][nrhs], then M [SB][SB]
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(j0 + SB, s.k) - j0;
  if (kb <= 0) return;
  const int j1 = j0 + kb;
  const int used = s.m > j1 ? (s.m - j1 + RB - 1) / RB : 0;
  const double* M = L.aux + f * L.aux_stride + (long long)(j0 / SB) * SB * SB;
  double* Xf = X + f * out_rows * nrhs;
  const int n = kb * nrhs;
  double* Ms = sm + SB * nrhs;
#pragma unroll 4
  for (int e = threadIdx.x; e < SB * SB; e += blockDim.x) Ms[e] = __ldg(M + e);
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    double v = Xf[(long long)j0 * nrhs + e];
    for (int x = 0; x < used; x++) v -= partial[((f * nchunk + x) * SB) * (long long)nrhs + e];
    sm[e] = v;
  }
  __syncthreads();
  const long long piv = L.piv_off[f] + j0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int c = e / nrhs, j = e - c * nrhs;
    double acc = sm[e];  // (M^T)[c][c] = 1
    for (int q = c + 1; q < kb; q++) acc += Ms[q * SB + c] * sm[q * nrhs + j];
    Xf[(long long)j0 * nrhs + e] = acc;
    y[piv * nrhs + e] = acc;
  }
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
constexpr size_t kSmallSolveSmem = 160 * 1024;

template <int G, int GPC, bool FWD, bool STAGE>
static cudaError_t launch_small_solve(const LevelArgs& L, const LevelArgs& O, int flag,
                                      const double* factors, const double* w_in,
                                      long long in_rows, double* w_out, long long out_rows,
                                      double* y, int nr, int ldr, int col0, cudaStream_t st) {
  const size_t pan = STAGE ? (size_t)L.max_m * L.max_k + L.max_m : 0;
  const int per = (int)(((size_t)L.max_m * nr + pan) * 8 + 15) & ~15;
  const size_t smem = (size_t)per * GPC;
  const unsigned blocks = (unsigned)((L.n_fronts + GPC - 1) / GPC);
  if (FWD) {
    auto kern = solve_fwd_small<G, GPC, STAGE>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    timer_begin(K_SOLVE_SMALL_FWD, st);
    kern<<<blocks, G * GPC, smem, st>>>(L, O, factors, w_in, in_rows, flag, w_out, out_rows, y,
                                        nr, ldr, col0, per);
    timer_end(st);
  } else {
    auto kern = solve_bwd_small<G, GPC, STAGE>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    timer_begin(K_SOLVE_SMALL_BWD, st);
    kern<<<blocks, G * GPC, smem, st>>>(L, O, flag, factors, w_in, in_rows, w_out, out_rows, y,
                                        nr, ldr, col0, per);
    timer_end(st);
  }
  return cudaGetLastError();
}

static int small_cols(const LevelArgs& L, int nrhs) {
  const long long fixed = (long long)L.max_m * L.max_k + L.max_m;
  const int cmax = (int)((kSmallSolveSmem / 8 - fixed) / std::max(L.max_m, 1));
  return std::max(1, std::min(nrhs, cmax));
}

// flag: forward -- 1 if the child level's update rows start at row 0 of its
// blocks (small child level); backward -- has_parent.
template <bool FWD>
static cudaError_t dispatch_small(const LevelArgs& L, const LevelArgs& O, int flag,
                                  const double* factors, const double* w_in, long long in_rows,
                                  double* w_out, long long out_rows, double* y, int nrhs,
                                  cudaStream_t st) {
  const int cw = small_cols(L, nrhs);
  for (int col0 = 0; col0 < nrhs; col0 += cw) {
    const int nr = std::min(cw, nrhs - col0);
    const long long work = (long long)L.max_m * nr;
    cudaError_t e;
    if (nr == 1) {  // vector block only in shared memory
#define TFB_SMALL(G, GPC)                                                                    \
  launch_small_solve<G, GPC, FWD, false>(L, O, flag, factors, w_in, in_rows, w_out, out_rows, \
                                         y, nr, nrhs, col0, st)
      if (work <= 12) e = TFB_SMALL(1, 128);
      else if (work <= 24) e = TFB_SMALL(2, 64);
      else if (work <= 48) e = TFB_SMALL(4, 64);
      else if (work <= 96) e = TFB_SMALL(8, 32);
      else if (work <= 256) e = TFB_SMALL(32, 8);
      else e = TFB_SMALL(128, 2);
#undef TFB_SMALL
    } else {
      const long long bytes = (work + (long long)L.max_m * L.max_k + L.max_m) * 8;
#define TFB_SMALL(G, GPC)                                                                   \
  launch_small_solve<G, GPC, FWD, true>(L, O, flag, factors, w_in, in_rows, w_out, out_rows, \
                                        y, nr, nrhs, col0, st)
      if (work <= 24 && bytes * 64 <= (long long)kSmallSolveSmem) e = TFB_SMALL(2, 64);
      else if (work <= 48 && bytes * 64 <= (long long)kSmallSolveSmem) e = TFB_SMALL(4, 64);
      else if (work <= 96 && bytes * 32 <= (long long)kSmallSolveSmem) e = TFB_SMALL(8, 32);
      else if (work <= 256 && bytes * 8 <= (long long)kSmallSolveSmem) e = TFB_SMALL(32, 8);
      else if (work <= 2048 && bytes * 2 <= (long long)kSmallSolveSmem) e = TFB_SMALL(128, 2);
      else e = TFB_SMALL(256, 1);
#undef TFB_SMALL
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

long long solve_workspace_doubles(const LevelArgs& L, int nrhs) {
  if (!level_is_large(L.is_leaf, L.max_m)) return 0;
  const long long nchunk = (L.max_m + RB - 1) / RB;
  return (long long)L.n_fronts * nchunk * SB * nrhs;
}

cudaError_t launch_solve_fwd(const LevelArgs& L, const LevelArgs& C, const double* factors,
                             const double* w_child, long long child_rows, double* w_out,
                             long long out_rows, double* y, int nrhs, cudaStream_t st) {
  if (!level_is_large(L.is_leaf, L.max_m))
    return dispatch_small<true>(L, C, level_is_large(C.is_leaf, C.max_m) ? 0 : 1, factors, w_child,
                                child_rows, w_out, out_rows, y, nrhs, st);
  const unsigned nf = (unsigned)L.n_fronts;
  const long long nW = (long long)L.max_m * nrhs;
  timer_begin(K_SOLVE_GATHER, st);
  solve_gather_fwd<<<dim3(nf, (unsigned)std::min<long long>((nW + 255) / 256, 1024)), 256, 0,
                     st>>>(L, C, w_child, child_rows, level_is_large(C.is_leaf, C.max_m) ? 0 : 1, w_out, out_rows, y,
                          nrhs);
  timer_end(st);
  const size_t smem = sizeof(double) * (2 * SB * (size_t)nrhs + SB * SB);
  cudaFuncSetAttribute(solve_fwd_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int j0 = 0; j0 < L.max_k; j0 += SB) {
    const int rows = std::max(1, L.max_m - j0 - 1);
    timer_begin(K_SOLVE_FWD_BLOCK, st);
    solve_fwd_block<<<dim3(nf, (unsigned)((rows + RB - 1) / RB)), 256, smem, st>>>(
        L, factors, w_out, out_rows, y, nrhs, j0);
    timer_end(st);
  }
  return cudaGetLastError();
}

cudaError_t launch_solve_bwd(const LevelArgs& L, const LevelArgs& PA, int has_parent,
                             const double* factors, const double* x_parent, long long parent_rows,
                             double* x_out, long long out_rows, double* y, int nrhs,
                             double* work, long long work_doubles, cudaStream_t st) {
  if (!level_is_large(L.is_leaf, L.max_m))
    return dispatch_small<false>(L, PA, has_parent, factors, x_parent, parent_rows, x_out,
                                 out_rows, y, nrhs, st);
  if (!work || work_doubles < solve_workspace_doubles(L, nrhs)) return cudaErrorInvalidValue;
  const unsigned nf = (unsigned)L.n_fronts;
  const long long nW = (long long)L.max_m * nrhs;
  timer_begin(K_SOLVE_GATHER, st);
  solve_gather_bwd<<<dim3(nf, (unsigned)std::min<long long>((nW + 255) / 256, 1024)), 256, 0,
                     st>>>(L, PA, has_parent, x_parent, parent_rows, x_out, out_rows, y, nrhs);
  timer_end(st);
  const int nchunk = (L.max_m + RB - 1) / RB;
  const size_t smp = sizeof(double) * RB * (size_t)nrhs;
  const size_t smb = sizeof(double) * (SB * (size_t)nrhs + SB * SB);
  cudaFuncSetAttribute(solve_bwd_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp);
  cudaFuncSetAttribute(solve_bwd_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
  const int nblk = (L.max_k + SB - 1) / SB;
  for (int b = nblk - 1; b >= 0; b--) {
    const int j0 = b * SB;
    const int rows = std::max(1, L.max_m - j0 - 1);
    const int used = (rows + RB - 1) / RB;
    timer_begin(K_SOLVE_BWD_PARTIAL, st);
    solve_bwd_partial<<<dim3(nf, (unsigned)used), 256, smp, st>>>(L, factors, x_out, out_rows,
                                                                  nrhs, j0, work, nchunk);
    timer_end(st);
    timer_begin(K_SOLVE_BWD_BLOCK, st);
    solve_bwd_block<<<nf, 256, smb, st>>>(L, x_out, out_rows, y, nrhs, j0, work, nchunk);
    timer_end(st);
  }
  return cudaGetLastError();
}

int solve_launches(const LevelArgs& L, int nrhs, bool fwd) {
  if (!level_is_large(L.is_leaf, L.max_m)) return (nrhs + small_cols(L, nrhs) - 1) / small_cols(L, nrhs);
  const int nblk = (L.max_k + SB - 1) / SB;
  return fwd ? 1 + nblk : 1 + 2 * nblk;
}

cudaError_t launch_permute_rows(const int* idx, long long n, const double* in, double* out,
                                int nrhs, int scatter, cudaStream_t st) {
  long long total = n * nrhs;
  unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148 * 16);
  if (blocks == 0) return cudaSuccess;
  timer_begin(K_PERMUTE, st);
  permute_rows_kernel<<<blocks, 256, 0, st>>>(idx, n, in, out, nrhs, scatter);
  timer_end(st);
  return cudaGetLastError();
}

}  // namespace tfb
