// Large-front level path (fronts too big for one SM's shared memory).
//
// Per level, batched over all fronts of the level (one launch per step):
//   1. zero the factor slot (panel P, m x kp, + diagonal d) and the packed
//      Schur block S in this level's update buffer;
//   2. extend-add child 0 then child 1 (fixed order, no atomics);
//   3. recursive blocked partial LDL^T of the k fully-summed columns:
//      64-wide diagonal blocks factored in shared memory, row-parallel
//      triangular solves below them, DMMA tile updates of the remaining
//      panel columns;
//   4. one DMMA update S -= L21 D L21^T over all k pivots.
// Arithmetic replaced: engine.py:86-105 per pivot (Division, Multiplication,
// Subtraction) and engine.py:537-545 (factorize_nested_loops inner loops).
#include "common.cuh"

namespace tfb {

constexpr int NB = 64;  // diagonal block width

__global__ void large_zero_kernel(LevelArgs L, double* factors, double* upd) {
  const long long f = blockIdx.y;
  const Shape s = front_shape(L, f);
  const long long nP = (long long)s.m * s.kp + s.kp, nS = tri(s.m - s.k, 0);
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
  const Shape s = front_shape(L, f);
  if (c >= s.nsrc) return;
  const int len = c == 0 ? s.len0 : s.len1;
  const int* mp = L.maps + (c == 0 ? s.off0 : s.off1);
  const double* src = child_upd + (2 * f + c) * L.child_upd_stride;
  double* Pf = factors + f * L.fac_stride;
  double* Sf = upd + f * L.upd_stride;
  const long long n = tri(len, 0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int a = tri_row(e), b = (int)(e - tri(a, 0));
    const int R = mp[a], C = mp[b];
    const int hi = R > C ? R : C, lo = R > C ? C : R;
    const double v = src[e];
    if (lo < s.k) Pf[(long long)hi * s.kp + lo] += v;
    else Sf[tri(hi - s.k, lo - s.k)] += v;
  }
}

// Factor the diagonal block [a, a+kb) of every front's panel in shared memory.
__global__ void __launch_bounds__(256) large_diag_kernel(LevelArgs L, double* factors, int a,
                                                          double threshold,
                                                          unsigned long long* err) {
  __shared__ double D[NB][NB + 1];
  __shared__ double lv[NB];
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(a + NB, s.k) - a;
  if (kb <= 0) return;
  double* Pf = factors + f * L.fac_stride;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < kb * NB; e += blockDim.x) {
    const int i = e / NB, j = e - i * NB;
    if (j <= i) D[i][j] = Pf[(long long)(a + i) * s.kp + a + j];
  }
  __syncthreads();
  const long long piv0 = L.piv_off[f] + a;
  for (int c = 0; c < kb; c++) {
    const double d = D[c][c];
    if (tid == 0 && fabs(d) <= threshold) record_zero_pivot(err, (unsigned long long)(piv0 + c));
    for (int r = c + 1 + tid; r < kb; r += blockDim.x) lv[r] = D[r][c] / d;
    __syncthreads();
    for (int r = c + 1 + warp; r < kb; r += 8) {
      const double frc = D[r][c];
      for (int q = c + 1 + lane; q <= r; q += 32) D[r][q] -= lv[q] * frc;
      __syncwarp();
      if (lane == 0) D[r][c] = lv[r];
    }
    __syncthreads();
  }
  for (int e = tid; e < kb * NB; e += blockDim.x) {
    const int i = e / NB, j = e - i * NB;
    if (j <= i) Pf[(long long)(a + i) * s.kp + a + j] = D[i][j];
  }
  double* dv = Pf + (long long)s.m * s.kp + a;
  for (int c = tid; c < kb; c += blockDim.x) dv[c] = D[c][c];
}

// Row-parallel triangular solve below the diagonal block: row r, cols [a, a+kb):
// for t: l_rt = a_rt / d_t; a_rc -= l_ct * a_rt (c > t).
__global__ void __launch_bounds__(128) large_trsm_kernel(LevelArgs L, double* factors, int a) {
  __shared__ double Lb[NB][NB + 1];
  __shared__ double dinv[NB];
  const long long f = blockIdx.y;
  const Shape s = front_shape(L, f);
  const int kb = min(a + NB, s.k) - a;
  if (kb <= 0) return;
  const int row0 = a + kb + blockIdx.x * blockDim.x;
  if (row0 >= s.m) return;
  double* Pf = factors + f * L.fac_stride;
  for (int e = threadIdx.x; e < kb * NB; e += blockDim.x) {
    const int i = e / NB, j = e - i * NB;
    if (j < i) Lb[i][j] = Pf[(long long)(a + i) * s.kp + a + j];
  }
  for (int c = threadIdx.x; c < kb; c += blockDim.x) dinv[c] = 1.0 / Pf[(long long)(a + c) * s.kp + a + c];
  __syncthreads();
  const int r = row0 + threadIdx.x;
  if (r >= s.m) return;
  double x[NB];
  double* row = Pf + (long long)r * s.kp + a;
#pragma unroll
  for (int t = 0; t < NB; t++) x[t] = t < kb ? row[t] : 0.0;
#pragma unroll
  for (int t = 0; t < NB; t++) {
    const double v = x[t];
    x[t] = v * dinv[t];
#pragma unroll
    for (int c = t + 1; c < NB; c++) x[c] -= Lb[c][t] * v;
  }
#pragma unroll
  for (int t = 0; t < NB; t++)
    if (t < kb) row[t] = x[t];
}

// C -= (A diag(d)) B^T with FP64 tensor-core MMA (mma.sync m8n8k4), 128x64
// CTA tiles, 8 warps of 32x32, 3-stage cp.async pipeline over K (BK = 16).
// MODE 0 (panel): out P[r][c], r in [row0, m), c in [col0, min(col1, k)), r >= c,
//                 A = P rows r, B = P rows c, K = [t0, min(t1, k)).
// MODE 1 (schur): out S[i][j] packed, i >= j, A = P rows k+i, B = P rows k+j, K = [0, k).
constexpr int GBM = 128, GBN = 64, GBK = 16, GLD = GBK + 4, GSTAGES = 3;

template <int MODE>
__global__ void __launch_bounds__(256) large_update_kernel(LevelArgs L, double* factors,
                                                            double* upd, int row0, int col0,
                                                            int col1, int t0, int t1) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                                  // [GSTAGES][GBM][GLD]
  double* Bs = As + GSTAGES * GBM * GLD;             // [GSTAGES][GBN][GLD]
  double* Ds = Bs + GSTAGES * GBN * GLD;             // [GSTAGES][GBK]
  const long long f = blockIdx.z;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  int aRow0, bRow0, nA, nB, kBeg, kEnd;
  long long tile_r0, tile_c0;
  if (MODE == 0) {
    tile_r0 = row0 + (long long)blockIdx.y * GBM;
    tile_c0 = col0 + (long long)blockIdx.x * GBN;
    const int cLim = min(col1, k);
    if (tile_r0 >= m || tile_c0 >= cLim || tile_r0 + GBM <= tile_c0) return;
    aRow0 = (int)tile_r0;
    bRow0 = (int)tile_c0;
    nA = min(GBM, m - aRow0);
    nB = min(GBN, cLim - bRow0);
    kBeg = t0;
    kEnd = min(t1, k);
  } else {
    const int u = m - k;
    tile_r0 = (long long)blockIdx.y * GBM;
    tile_c0 = (long long)blockIdx.x * GBN;
    if (tile_r0 >= u || tile_c0 >= u || tile_r0 + GBM <= tile_c0) return;
    aRow0 = k + (int)tile_r0;
    bRow0 = k + (int)tile_c0;
    nA = min(GBM, u - (int)tile_r0);
    nB = min(GBN, u - (int)tile_c0);
    kBeg = 0;
    kEnd = k;
  }
  if (kEnd <= kBeg) return;
  const double* Pf = factors + f * L.fac_stride;
  const double* dvec = Pf + (long long)m * kp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp >> 1, wx = warp & 1;  // 4 x 2 warps of 32x32
  const int nk = (kEnd - kBeg + GBK - 1) / GBK;

  auto issue = [&](int it) {
    const int stage = it % GSTAGES;
    const int kt = kBeg + it * GBK;
    double* as = As + stage * GBM * GLD;
    double* bs = Bs + stage * GBN * GLD;
    // A: 128 rows x 16 doubles = 1024 chunks of 2 doubles, 4 per thread
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int ch = tid + q * 256;
      const int r = ch >> 3, cc = (ch & 7) * 2;
      const int t = kt + cc;
      const bool v = r < nA && t < kEnd;
      const double* src = v ? Pf + (long long)(aRow0 + r) * kp + t : Pf;
      cp_async16(as + r * GLD + cc, src, v);
    }
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int ch = tid + q * 256;
      const int r = ch >> 3, cc = (ch & 7) * 2;
      const int t = kt + cc;
      const bool v = r < nB && t < kEnd;
      const double* src = v ? Pf + (long long)(bRow0 + r) * kp + t : Pf;
      cp_async16(bs + r * GLD + cc, src, v);
    }
    if (tid < GBK / 2) {
      const int t = kt + tid * 2;
      cp_async16(Ds + stage * GBK + tid * 2, t < kEnd ? dvec + t : dvec, t < kEnd);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int it = 0; it < GSTAGES - 1; it++) {
    if (it < nk) issue(it);
    cp_async_commit();
  }
  for (int it = 0; it < nk; it++) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    if (it + GSTAGES - 1 < nk) issue(it + GSTAGES - 1);
    cp_async_commit();
    const int stage = it % GSTAGES;
    const double* as = As + stage * GBM * GLD + (wy * 32 + (lane >> 2)) * GLD + (lane & 3);
    const double* bs = Bs + stage * GBN * GLD + (wx * 32 + (lane >> 2)) * GLD + (lane & 3);
    const double* ds = Ds + stage * GBK + (lane & 3);
    // K tail: entries past kEnd were zero-filled
#pragma unroll
    for (int ks = 0; ks < GBK; ks += 4) {
      const double dk = ds[ks];
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; i++) af[i] = as[i * 8 * GLD + ks] * dk;
#pragma unroll
      for (int j = 0; j < 4; j++) bf[j] = bs[j * 8 * GLD + ks];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma884(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  // epilogue: C -= acc (lower part only)
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
        if (MODE == 0) out[R * kp + C] -= acc[i][j][h];
        else out[tri(R, C)] -= acc[i][j][h];
      }
    }
  }
}

constexpr size_t kGemmSmem = sizeof(double) * (GSTAGES * (GBM + GBN) * GLD + GSTAGES * GBK);

static cudaError_t panel_factor(const LevelArgs& L, double* factors, double thr,
                                unsigned long long* err, int a, int b, cudaStream_t st) {
  if (b - a <= NB) {
    large_diag_kernel<<<L.n_fronts, 256, 0, st>>>(L, factors, a, thr, err);
    const int rows = L.max_m - a;
    dim3 g((unsigned)((rows + 127) / 128), (unsigned)L.n_fronts);
    large_trsm_kernel<<<g, 128, 0, st>>>(L, factors, a);
    return cudaGetLastError();
  }
  int mid = a + ((b - a) / 2 + NB - 1) / NB * NB;
  if (mid >= b) mid = a + NB;
  cudaError_t e = panel_factor(L, factors, thr, err, a, mid, st);
  if (e != cudaSuccess) return e;
  dim3 g((unsigned)((b - mid + GBN - 1) / GBN), (unsigned)((L.max_m - mid + GBM - 1) / GBM),
         (unsigned)L.n_fronts);
  large_update_kernel<0><<<g, 256, kGemmSmem, st>>>(L, factors, nullptr, mid, mid, b, a, mid);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return panel_factor(L, factors, thr, err, mid, b, st);
}

cudaError_t launch_factor_large(const LevelArgs& L, const double* child_upd, double* factors,
                                double* upd_out, double thr, unsigned long long* err,
                                cudaStream_t st) {
  if (L.is_leaf) return cudaErrorInvalidValue;  // element fronts are never this large
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(large_update_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGemmSmem);
    cudaFuncSetAttribute(large_update_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGemmSmem);
    attr = true;
  }
  {
    const long long per = L.fac_stride + tri(L.max_upd, 0);
    const unsigned gx = (unsigned)std::min<long long>((per + 255) / 256, 1024);
    large_zero_kernel<<<dim3(gx, L.n_fronts), 256, 0, st>>>(L, factors, upd_out);
  }
  const long long maxsrc = tri(L.max_m, 0);
  const unsigned gx = (unsigned)std::min<long long>((maxsrc + 255) / 256, 2048);
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
    dim3 g((unsigned)((L.max_upd + GBN - 1) / GBN), (unsigned)((L.max_upd + GBM - 1) / GBM),
           (unsigned)L.n_fronts);
    large_update_kernel<1><<<g, 256, kGemmSmem, st>>>(L, factors, upd_out, 0, 0, 0, 0, 0);
    e = cudaGetLastError();
  }
  return e;
}

int large_panel_launches(int max_k) {
  if (max_k <= 0) return 0;
  if (max_k <= NB) return 2;
  int mid = (max_k / 2 + NB - 1) / NB * NB;
  if (mid >= max_k) mid = NB;
  return large_panel_launches(mid) + 1 + large_panel_launches(max_k - mid);
}

}  // namespace tfb
