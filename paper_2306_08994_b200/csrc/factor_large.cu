// Large-front level path (fronts too big for one SM's shared memory).
//
// Per level, batched over all fronts of the level (one launch per step):
//   1. zero the front panel P (m x k, row-major, in the factor buffer) and the
//      packed Schur block S (in this level's update buffer);
//   2. extend-add child 0 then child 1 (fixed order, no atomics);
//   3. recursive blocked partial LDL^T of the k fully-summed columns:
//      64-wide diagonal blocks in shared memory, row-parallel triangular
//      solves below them, and DMMA (mma.sync m8n8k4 f64) tile updates of
//      the remaining panel columns;
//   4. one DMMA SYRK-style update S -= L21 D L21^T over all k pivots.
// Arithmetic replaced: engine.py:86-105 per pivot (Division, Multiplication,
// Subtraction) and engine.py:537-545 (factorize_nested_loops inner loops).
#include "common.cuh"

namespace tfb {

constexpr int NB = 64;  // diagonal block width
constexpr int TBM = 64, TBN = 64, TBK = 16, TPAD = 4;

__device__ __forceinline__ void front_shape(const LevelArgs& L, long long f, int& m, int& k) {
  const int* P = L.pat + (size_t)L.pattern_of[f] * TF_PAT_WIDTH;
  m = P[TF_PAT_M];
  k = P[TF_PAT_K];
}

__global__ void large_zero_kernel(LevelArgs L, double* factors, double* upd) {
  const long long f = blockIdx.y;
  int m, k;
  front_shape(L, f, m, k);
  const long long nP = (long long)m * k, nS = tri(m - k, 0);
  double* Pf = factors + f * L.fac_stride;
  double* Sf = upd + f * L.upd_stride;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nP + nS;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nP) Pf[e] = 0.0;
    else Sf[e - nP] = 0.0;
  }
}

__global__ void large_scatter_kernel(LevelArgs L, const double* __restrict__ child_upd,
                                     double* factors, double* upd, int c) {
  const long long f = blockIdx.y;
  const int* P = L.pat + (size_t)L.pattern_of[f] * TF_PAT_WIDTH;
  const int m = P[TF_PAT_M], k = P[TF_PAT_K], nsrc = P[TF_PAT_NSRC];
  if (c >= nsrc) return;
  const int len = c == 0 ? P[TF_PAT_LEN0] : P[TF_PAT_LEN1];
  const int* mp = L.maps + (c == 0 ? P[TF_PAT_OFF0] : P[TF_PAT_OFF1]);
  const double* src = child_upd + (2 * f + c) * L.child_upd_stride;
  double* Pf = factors + f * L.fac_stride;
  double* Sf = upd + f * L.upd_stride;
  (void)m;
  const long long n = tri(len, 0);
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= n) return;
  int a = tri_row(e);
  int b = (int)(e - tri(a, 0));
  for (; e < n; e += stride) {
    const int R = mp[a], C = mp[b];
    const int hi = R > C ? R : C, lo = R > C ? C : R;
    const double v = src[e];
    if (lo < k) Pf[(long long)hi * k + lo] += v;
    else Sf[tri(hi - k, lo - k)] += v;
    // advance by stride within the packed triangle
    long long nb = (long long)b + stride;
    while (nb > a) { nb -= a + 1; a++; }
    b = (int)nb;
  }
}

// Factor the diagonal block [a, a+kb) x [a, a+kb) of every front's panel.
__global__ void __launch_bounds__(256) large_diag_kernel(LevelArgs L, double* factors, int a,
                                                          double threshold,
                                                          unsigned long long* err) {
  __shared__ double D[NB][NB + 1];
  __shared__ double lv[NB];
  const long long f = blockIdx.x;
  int m, k;
  front_shape(L, f, m, k);
  const int kb = min(a + NB, k) - a;
  if (kb <= 0) return;
  double* Pf = factors + f * L.fac_stride;
  const int tid = threadIdx.x;
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    int i = e / kb, j = e - i * kb;
    if (j <= i) D[i][j] = Pf[(long long)(a + i) * k + a + j];
  }
  __syncthreads();
  const long long piv0 = L.piv_off[f] + a;
  for (int c = 0; c < kb; c++) {
    const double d = D[c][c];
    if (tid == 0 && fabs(d) <= threshold) record_zero_pivot(err, (unsigned long long)(piv0 + c));
    for (int r = c + 1 + tid; r < kb; r += blockDim.x) lv[r] = D[r][c] / d;
    __syncthreads();
    const int w = kb - c - 1;
    for (int e = tid; e < w * w; e += blockDim.x) {
      int r = c + 1 + e / w, s = c + 1 + e % w;
      if (s <= r) D[r][s] -= lv[s] * D[r][c];
    }
    __syncthreads();
    for (int r = c + 1 + tid; r < kb; r += blockDim.x) D[r][c] = lv[r];
    __syncthreads();
  }
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    int i = e / kb, j = e - i * kb;
    if (j <= i) Pf[(long long)(a + i) * k + a + j] = D[i][j];
  }
}

// Row-parallel triangular solve of the panel rows below the diagonal block:
// row r, columns [a, a+kb): for t: l_rt = a_rt / d_t; a_rc -= l_ct * a_rt.
__global__ void __launch_bounds__(128) large_trsm_kernel(LevelArgs L, double* factors, int a) {
  __shared__ double Lb[NB][NB + 1];
  const long long f = blockIdx.y;
  int m, k;
  front_shape(L, f, m, k);
  const int kb = min(a + NB, k) - a;
  if (kb <= 0) return;
  const int r = a + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (a + kb + (int)(blockIdx.x * blockDim.x) >= m) return;
  double* Pf = factors + f * L.fac_stride;
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    int i = e / kb, j = e - i * kb;
    if (j <= i) Lb[i][j] = Pf[(long long)(a + i) * k + a + j];
  }
  __syncthreads();
  if (r >= m) return;
  double x[NB];
  double* row = Pf + (long long)r * k + a;
#pragma unroll
  for (int t = 0; t < NB; t++) x[t] = t < kb ? row[t] : 0.0;
#pragma unroll
  for (int t = 0; t < NB; t++) {
    if (t < kb) {
      const double v = x[t];
      x[t] = v / Lb[t][t];
#pragma unroll
      for (int c = t + 1; c < NB; c++) x[c] -= Lb[c][t] * v;
    }
  }
#pragma unroll
  for (int t = 0; t < NB; t++)
    if (t < kb) row[t] = x[t];
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// C -= (A diag(d)) B^T on 64x64 tiles with FP64 tensor-core MMA.
// MODE 0 (panel): out P[r][c], r in [row0, m), c in [col0, min(col1, k)), r >= c,
//                 A = P rows r, B = P rows c, K = [t0, min(t1, k)).
// MODE 1 (schur): out S[i][j] packed, i >= j, A = P rows k+i, B = P rows k+j, K = [0, k).
template <int MODE>
__global__ void __launch_bounds__(128) large_update_kernel(LevelArgs L, double* factors,
                                                            double* upd, int row0, int col0,
                                                            int col1, int t0, int t1) {
  __shared__ __align__(16) double As[2][TBM][TBK + TPAD];
  __shared__ __align__(16) double Bs[2][TBN][TBK + TPAD];
  const long long f = blockIdx.z;
  int m, k;
  front_shape(L, f, m, k);
  int aRow0, bRow0, nA, nB, kBeg, kEnd;
  long long tile_r0, tile_c0;
  if (MODE == 0) {
    tile_r0 = row0 + (long long)blockIdx.y * TBM;
    tile_c0 = col0 + (long long)blockIdx.x * TBN;
    const int cLim = min(col1, k);
    if (tile_r0 >= m || tile_c0 >= cLim || tile_r0 + TBM <= tile_c0) return;
    aRow0 = (int)tile_r0;
    bRow0 = (int)tile_c0;
    nA = min(TBM, m - aRow0);
    nB = min(TBN, cLim - bRow0);
    kBeg = t0;
    kEnd = min(t1, k);
  } else {
    // triangular tile index -> (ty, tx), tx <= ty
    const int lin = blockIdx.x;
    int ty = (int)((sqrt(8.0 * lin + 1.0) - 1.0) * 0.5);
    while (ty * (ty + 1) / 2 > lin) ty--;
    while ((ty + 1) * (ty + 2) / 2 <= lin) ty++;
    const int tx = lin - ty * (ty + 1) / 2;
    const int u = m - k;
    tile_r0 = (long long)ty * TBM;
    tile_c0 = (long long)tx * TBN;
    if (tile_r0 >= u) return;
    aRow0 = k + (int)tile_r0;
    bRow0 = k + (int)tile_c0;
    nA = min(TBM, u - (int)tile_r0);
    nB = min(TBN, u - (int)tile_c0);
    kBeg = 0;
    kEnd = k;
  }
  if (kEnd <= kBeg) return;
  const double* Pf = factors + f * L.fac_stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp >> 1, wx = warp & 1;
  // staging: thread loads 8 consecutive K values of one row of A and of B
  const int ld_row = tid >> 1, ld_col = (tid & 1) * 8;
  double ra[8], rb[8];
  auto load_stage = [&](int kt) {
    const int kk0 = kt + ld_col;
    const bool va = ld_row < nA, vb = ld_row < nB;
    const double* pa = Pf + (long long)(aRow0 + ld_row) * k;
    const double* pb = Pf + (long long)(bRow0 + ld_row) * k;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int t = kk0 + j;
      const bool vt = t < kEnd;
      const double dt = vt ? __ldg(Pf + (long long)t * k + t) : 0.0;
      ra[j] = (va && vt) ? pa[t] * dt : 0.0;
      rb[j] = (vb && vt) ? pb[t] : 0.0;
    }
  };
  auto store_stage = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      As[buf][ld_row][ld_col + j] = ra[j];
      Bs[buf][ld_row][ld_col + j] = rb[j];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  load_stage(kBeg);
  store_stage(0);
  __syncthreads();
  int buf = 0;
  for (int kt = kBeg; kt < kEnd; kt += TBK) {
    const bool more = kt + TBK < kEnd;
    if (more) load_stage(kt + TBK);
#pragma unroll
    for (int ks = 0; ks < TBK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; i++) af[i] = As[buf][wy * 32 + i * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; j++) bf[j] = Bs[buf][wx * 32 + j * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma884(acc[i][j], af[i], bf[j]);
    }
    if (more) {
      store_stage(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  // epilogue: C -= acc
  double* out = MODE == 0 ? factors + f * L.fac_stride : upd + f * L.upd_stride;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int rl = wy * 32 + i * 8 + (lane >> 2);
    if (rl >= nA) continue;
    const long long R = tile_r0 + rl;
#pragma unroll
    for (int j = 0; j < 4; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int cl = wx * 32 + j * 8 + 2 * (lane & 3) + h;
        if (cl >= nB) continue;
        const long long C = tile_c0 + cl;
        if (C > R) continue;
        if (MODE == 0) out[R * k + C] -= acc[i][j][h];
        else out[tri(R, C)] -= acc[i][j][h];
      }
    }
  }
}

static cudaError_t panel_factor(const LevelArgs& L, double* factors, double thr,
                                unsigned long long* err, int a, int b, cudaStream_t st) {
  if (b - a <= NB) {
    large_diag_kernel<<<L.n_fronts, 256, 0, st>>>(L, factors, a, thr, err);
    const int rows = L.max_m - a;  // upper bound of rows below the block
    dim3 g((unsigned)((rows + 127) / 128), (unsigned)L.n_fronts);
    large_trsm_kernel<<<g, 128, 0, st>>>(L, factors, a);
    return cudaGetLastError();
  }
  int mid = a + ((b - a) / 2 + NB - 1) / NB * NB;
  if (mid >= b) mid = a + NB;
  cudaError_t e = panel_factor(L, factors, thr, err, a, mid, st);
  if (e != cudaSuccess) return e;
  dim3 g((unsigned)((b - mid + TBN - 1) / TBN), (unsigned)((L.max_m - mid + TBM - 1) / TBM),
         (unsigned)L.n_fronts);
  large_update_kernel<0><<<g, 128, 0, st>>>(L, factors, nullptr, mid, mid, b, a, mid);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return panel_factor(L, factors, thr, err, mid, b, st);
}

cudaError_t launch_factor_large(const LevelArgs& L, const double* child_upd, double* factors,
                                double* upd_out, double thr, unsigned long long* err,
                                cudaStream_t st) {
  if (L.is_leaf) return cudaErrorInvalidValue;  // element fronts are never this large
  {
    long long per = (long long)L.max_m * L.max_k + tri(L.max_upd, 0);
    unsigned gx = (unsigned)std::min<long long>((per + 255) / 256, 1024);
    large_zero_kernel<<<dim3(gx, L.n_fronts), 256, 0, st>>>(L, factors, upd_out);
  }
  // child update sizes are bounded by this level's max_m
  const long long maxsrc = tri(L.max_m, 0);
  unsigned gx = (unsigned)std::min<long long>((maxsrc + 255) / 256, 2048);
  for (int c = 0; c < 2; c++)
    large_scatter_kernel<<<dim3(gx, L.n_fronts), 256, 0, st>>>(L, child_upd, factors, upd_out,
                                                                c);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (L.max_k > 0) {
    e = panel_factor(L, factors, thr, err, 0, L.max_k, st);
    if (e != cudaSuccess) return e;
  }
  if (L.max_upd > 0 && L.max_k > 0) {
    const int T = (L.max_upd + TBM - 1) / TBM;
    large_update_kernel<1><<<dim3((unsigned)(T * (T + 1) / 2), 1, (unsigned)L.n_fronts), 128, 0,
                             st>>>(L, factors, upd_out, 0, 0, 0, 0, 0);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace tfb
