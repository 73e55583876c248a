// Large-front level path (fronts too big for one SM's shared memory).
//
// Per level, batched over all fronts of the level (one launch per step):
//   1. gather-form assembly: every entry of the panel P (m x kp), the diagonal
//      vector d and the packed Schur block S is written exactly once, summing
//      its child contributions through the inverse extend-add maps (fixed child
//      order, no atomics, coalesced writes);
//   2. recursive blocked partial LDL^T of the k fully-summed columns:
//      a 64-wide diagonal block is factored in shared memory, which also
//      forms its unit-lower inverse M (kept in `aux` for the solve); the rows
//      below are solved as a DMMA GEMM  P_rb <- (P_rb M^T) D^-1; the remaining
//      panel columns get DMMA rank-64.. updates;
//   3. one DMMA update S -= L21 D L21^T over all k pivots.
// Arithmetic replaced: engine.py:86-105 per pivot (Division, Multiplication,
// Subtraction) and engine.py:537-545 (factorize_nested_loops inner loops).
#include <cstdlib>

#include "common.cuh"

namespace tfb {

constexpr int NB = 64;  // diagonal block width

__global__ void large_assemble_kernel(LevelArgs L, const double* __restrict__ child_upd,
                                      double* __restrict__ factors, double* __restrict__ upd) {
  const long long f = blockIdx.x;  // fronts on x (no 65535 limit), chunks on y
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long nPk = (long long)m * kp, nP = nPk + kp, nS = tri(m - k, 0);
  double* Pf = factors + f * L.fac_stride;
  double* Sf = upd + f * L.upd_stride;
  const int* inv0 = L.maps + s.ioff;
  const int* inv1 = inv0 + m;
  const double* src0 = child_upd + L.child_slot(f, 0) * L.child_upd_stride;
  const double* src1 = child_upd + L.child_slot(f, 1) * L.child_upd_stride;
  const bool two = s.nsrc == 2;
  for (long long e = blockIdx.y * (long long)blockDim.x + threadIdx.x; e < nP + nS;
       e += (long long)gridDim.y * blockDim.x) {
    int r, c;
    double* dst;
    if (e < nPk) {
      r = (int)(e / kp);
      c = (int)(e - (long long)r * kp);
      dst = Pf + e;
      if (c >= k || c > r) { *dst = 0.0; continue; }
    } else if (e < nP) {
      Pf[e] = 0.0;
      continue;
    } else {
      const long long e2 = e - nP;
      const int a = tri_row(e2);
      r = k + a;
      c = k + (int)(e2 - tri(a, 0));
      dst = Sf + e2;
    }
    double v = 0.0;
    {
      const int i = inv0[r], j = inv0[c];
      if (i >= 0 && j >= 0) v += src0[i > j ? tri(i, j) : tri(j, i)];
    }
    if (two) {
      const int i = inv1[r], j = inv1[c];
      if (i >= 0 && j >= 0) v += src1[i > j ? tri(i, j) : tri(j, i)];
    }
    *dst = v;
  }
}

// Factor the diagonal block [a, a+kb) of every front's panel (LDL^T, in shared
// memory), store l (scaled) and d, and the unit-lower inverse M = L_bb^-1 in aux.
// 256 threads: thread t owns row r = t/4, columns [16h, 16h+16) with h = t%4, held
// in registers.  One barrier per pivot: the owners of column c publish it to a
// double-buffered shared vector, every thread applies the rank-1 update to its
// registers.  The inverse is formed the same way, one published row per step.
__global__ void __launch_bounds__(256) large_diag_kernel(LevelArgs L, double* factors, int a,
                                                          double threshold,
                                                          unsigned long long* err) {
  constexpr int Q = 4, W = NB / Q;  // four threads per row, W columns each
  __shared__ double buf[2][NB];
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(a + NB, s.k) - a;
  if (kb <= 0) return;
  double* Pf = factors + f * L.fac_stride;
  const int tid = threadIdx.x, r = tid / Q, h = tid % Q, c0 = h * W;
  const int lane = tid & 31, quad = lane & ~(Q - 1);
  double v[W];
#pragma unroll
  for (int j = 0; j < W; j++) {
    const int col = c0 + j;
    v[j] = (r < kb && col <= r) ? Pf[(long long)(a + r) * s.kp + a + col] : (r == col ? 1.0 : 0.0);
  }
  const long long piv0 = L.piv_off[f] + a;
  // LDL^T: a(r,s) -= (a(s,c)/d) a(r,c); column c becomes l(r,c) = a(r,c)/d.
  // The pivot loop stays rolled (straight-line code executed once per CTA
  // would miss the instruction cache); register slots are selected by
  // compile-time indices inside the unrolled inner loops.
#pragma unroll 1
  for (int c = 0; c < kb; c++) {
    double* cb = buf[c & 1];
    const int cj = c % W;
    const bool own = h == c / W;
    if (own && r >= c) {
      double vc = 0.0;
#pragma unroll
      for (int j = 0; j < W; j++) vc = (j == cj) ? v[j] : vc;
      cb[r] = vc;
    }
    __syncthreads();
    const double d = cb[c];
    if (tid == 0 && fabs(d) <= threshold) record_zero_pivot(err, (unsigned long long)(piv0 + c));
    const double inv = 1.0 / d;
    if (r > c && r < kb) {
      const double arc = cb[r];
#pragma unroll
      for (int j = 0; j < W; j++) {
        const int col = c0 + j;
        if (col > c && col <= r) v[j] -= (cb[col] * inv) * arc;
        if (own && j == cj) v[j] = arc * inv;
      }
    }
  }
  // write l (strict lower) and d back
  if (r < kb) {
#pragma unroll
    for (int j = 0; j < W; j++) {
      const int col = c0 + j;
      if (col <= r) Pf[(long long)(a + r) * s.kp + a + col] = v[j];
      if (col == r) Pf[(long long)s.m * s.kp + a + r] = v[j];
    }
  }
  // unit-lower inverse M = L^-1, right-looking over rows t of M
  double w[W];
#pragma unroll
  for (int j = 0; j < W; j++) w[j] = (c0 + j == r) ? 1.0 : 0.0;
  __syncthreads();
#pragma unroll 1
  for (int t = 0; t < kb - 1; t++) {
    double* rb = buf[t & 1];
    if (r == t) {
#pragma unroll
      for (int j = 0; j < W; j++) rb[c0 + j] = w[j];
    }
    __syncthreads();
    // L[r][t] lives in the quad lane owning column block t / W
    const int tj = t % W;
    double vt = 0.0;
#pragma unroll
    for (int j = 0; j < W; j++) vt = (j == tj) ? v[j] : vt;
    const double lrt = __shfl_sync(0xffffffffu, vt, quad | (t / W));
    if (r > t && r < kb) {
#pragma unroll
      for (int j = 0; j < W; j++)
        if (c0 + j <= t) w[j] -= lrt * rb[c0 + j];
    }
  }
  // aux block: strict lower = M, diagonal = d, strict upper = l transposed
  double* M = L.aux + f * L.aux_stride + (long long)(a / NB) * NB * NB;
#pragma unroll
  for (int j = 0; j < W; j++) {
    const int col = c0 + j;
    if (col < r) {
      M[r * NB + col] = w[j];
      M[col * NB + r] = r < kb ? v[j] : 0.0;
    } else if (col == r) {
      M[r * NB + r] = r < kb ? v[j] : 1.0;
    }
  }
}

// One 64-wide diagonal block of every front's panel, fused with the triangular
// solve of the rows below it.  grid = (fronts, row tiles of 64).  Every CTA
// factors the diagonal block redundantly in shared memory (blocked LDL^T:
// 16-column panels with rank-1 steps, DMMA rank-16 trailing updates), forms
// its unit-lower inverse M (inverted 16x16 diagonal blocks + block
// substitution), then solves its 64-row tile as a DMMA product
// P_rb <- (P_rb M^T) D^-1.  The CTA of row tile 0 also writes l, d and M.
constexpr int TRB = 64;
constexpr int kFusedBlockMaxFronts = 2;
constexpr int DLD = NB + 1, ALD = NB + 4;
constexpr size_t kBlockSmem = sizeof(double) * (2 * NB * DLD + TRB * ALD + 2 * NB);

__global__ void __launch_bounds__(256) large_block_kernel(LevelArgs L, double* factors, int a,
                                                           double threshold,
                                                           unsigned long long* err) {
  extern __shared__ __align__(16) double bsm[];
  double(*D)[DLD] = reinterpret_cast<double(*)[DLD]>(bsm);
  double(*Mi)[DLD] = reinterpret_cast<double(*)[DLD]>(bsm + NB * DLD);
  double(*At)[ALD] = reinterpret_cast<double(*)[ALD]>(bsm + 2 * NB * DLD);
  double* dv = bsm + 2 * NB * DLD + TRB * ALD;
  double* lv = dv + NB;
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(a + NB, s.k) - a;
  if (kb <= 0) return;
  const int row0 = a + kb + blockIdx.y * TRB;
  const bool writer = blockIdx.y == 0;
  if (!writer && row0 >= s.m) return;
  const int rows = min(TRB, s.m - row0);
  double* Pf = factors + f * L.fac_stride;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, tq = lane & 3;

  // 1. diagonal block (identity pad beyond kb) and this CTA's row tile
  for (int e = tid; e < NB * NB; e += 256) {
    const int i = e >> 6, j = e & 63;
    D[i][j] = (i < kb && j <= i) ? Pf[(long long)(a + i) * s.kp + a + j] : (i == j ? 1.0 : 0.0);
    At[i][j] = (i < rows && j < kb) ? Pf[(long long)(row0 + i) * s.kp + a + j] : 0.0;
  }
  __syncthreads();

  // 2. blocked LDL^T of D
  const long long piv0 = L.piv_off[f] + a;
  for (int c0 = 0; c0 < kb; c0 += 16) {
    const int c1 = min(c0 + 16, kb);
    for (int c = c0; c < c1; c++) {
      const double d = D[c][c];
      if (writer && tid == 0 && fabs(d) <= threshold)
        record_zero_pivot(err, (unsigned long long)(piv0 + c));
      if (tid > c && tid < NB) {
        const double l = D[tid][c] / d;
        lv[tid] = l;
        D[tid][c] = l;
      }
      if (tid == c) dv[c] = d;
      __syncthreads();
      const int nc = c1 - c - 1;
      if (nc > 0) {
        const int n = (NB - c - 1) * nc;
        for (int e = tid; e < n; e += 256) {
          const int r = c + 1 + e / nc, q = c + 1 + e % nc;
          if (q <= r) D[r][q] -= lv[q] * (lv[r] * d);
        }
      }
      __syncthreads();
    }
    // rank-(c1-c0) DMMA update of the trailing columns [c0+16, 64)
    const int t0 = c0 + 16;
    if (t0 < NB) {
      const int T = (NB - t0) >> 3, ntile = T * (T + 1) / 2;
      for (int tile = warp; tile < ntile; tile += 8) {
        int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
        while (I * (I + 1) / 2 > tile) I--;
        while ((I + 1) * (I + 2) / 2 <= tile) I++;
        const int J = tile - I * (I + 1) / 2;
        const int ra = t0 + 8 * I + g8, rb = t0 + 8 * J + g8;
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          const int q = c0 + kk + tq;
          const bool v = q < c1;
          dmma884(acc, v ? D[ra][q] * dv[q] : 0.0, v ? D[rb][q] : 0.0);
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int cc = t0 + 8 * J + 2 * tq + h;
          if (cc <= ra) D[ra][cc] -= acc[h];
        }
      }
    }
    __syncthreads();
  }

  // 3. M = L^-1: 16x16 diagonal blocks (warp w < 4, lane c < 16 owns column c) ...
  if (warp < 4 && lane < 16) {
    const int o = warp * 16, c = lane;
    for (int r = 0; r < 16; r++) Mi[o + r][o + c] = r == c ? 1.0 : 0.0;
    for (int r = c + 1; r < 16; r++) {
      double acc = 0.0;
      for (int t = c; t < r; t++) acc -= D[o + r][o + t] * Mi[o + t][o + c];
      Mi[o + r][o + c] = acc;
    }
  }
  __syncthreads();
  // ... then block rows: M_ij = -M_ii * sum_{t=j}^{i-1} L_it M_tj
  for (int bi = 1; bi < 4; bi++) {
    const int oi = 16 * bi;
    // S_ij into lv-free scratch: reuse At? no -- use the upper triangle of Mi as scratch
    for (int e = tid; e < bi * 256; e += 256) {
      const int bj = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const int oj = 16 * bj;
      double acc = 0.0;
      for (int t = oj; t < oi; t++) acc += D[oi + r][t] * Mi[t][oj + c];
      Mi[oj + c][oi + r] = acc;  // scratch: upper part, transposed
    }
    __syncthreads();
    for (int e = tid; e < bi * 256; e += 256) {
      const int bj = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const int oj = 16 * bj;
      double acc = 0.0;
      for (int t = 0; t <= r; t++) acc -= Mi[oi + r][oi + t] * Mi[oj + c][oi + t];
      Mi[oi + r][oj + c] = acc;
    }
    __syncthreads();
  }
  // clear the scratch (upper part) so M is exactly lower-triangular
  for (int e = tid; e < NB * NB; e += 256) {
    const int i = e >> 6, j = e & 63;
    if (j > i) Mi[i][j] = 0.0;
  }
  __syncthreads();

  // 4. write d and the aux block: strict lower = M, diagonal = d, strict upper =
  // l transposed.  The panel's own diagonal block is not rewritten here: other
  // CTAs of this launch may still be reading its assembled values, so
  // large_diag_finalize_kernel copies l, d into it after the level.
  if (writer) {
    for (int c = tid; c < kb; c += 256) Pf[(long long)s.m * s.kp + a + c] = dv[c];
    double* M = L.aux + f * L.aux_stride + (long long)(a / NB) * NB * NB;
    for (int e = tid; e < NB * NB; e += 256) {
      const int i = e >> 6, j = e & 63;
      M[e] = j < i ? Mi[i][j] : (j == i ? (i < kb ? dv[i] : 1.0) : (j < kb ? D[j][i] : 0.0));
    }
  }

  // 5. row tile: X = At M^T, then column c / d_c (DMMA, 8 tiles of 8x8 per warp)
  if (rows > 0) {
    for (int tile = warp; tile < 64; tile += 8) {
      const int I = tile >> 3, J = tile & 7;
      double acc[2] = {0.0, 0.0};
#pragma unroll 4
      for (int kk = 0; kk < NB; kk += 4)
        dmma884(acc, At[8 * I + g8][kk + tq], Mi[8 * J + g8][kk + tq]);
      const int r = 8 * I + g8;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = 8 * J + 2 * tq + h;
        if (r < rows && c < kb) Pf[(long long)(row0 + r) * s.kp + a + c] = acc[h] / dv[c];
      }
    }
  }
}

// Copy every diagonal block's l (aux strict upper, transposed) and d into the
// panel once the level's launches no longer read the assembled values.
__global__ void large_diag_finalize_kernel(LevelArgs L, double* factors) {
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int a = blockIdx.y * NB;
  const int kb = min(a + NB, s.k) - a;
  if (kb <= 0) return;
  double* Pf = factors + f * L.fac_stride;
  const double* M = L.aux + f * L.aux_stride + (long long)blockIdx.y * NB * NB;
  for (int e = threadIdx.x; e < kb * NB; e += blockDim.x) {
    const int i = e >> 6, j = e & 63;
    if (j <= i) Pf[(long long)(a + i) * s.kp + a + j] = M[j * NB + i];
  }
}

// C (+)= op((A diag(d)) B^T) with FP64 tensor-core MMA (mma.sync m8n8k4): BMxBN
// CTA tiles, 8 warps (4 x 2) of (BM/4)x(BN/2), ST-stage cp.async pipeline over K.
// MODE 0 (panel): P[r][c] -= sum_t l_rt d_t l_ct, r in [row0, m), c in [col0, min(col1,k)),
//                 r >= c, t in [t0, min(t1, k)).
// MODE 1 (schur): S[i][j] -= sum_t l_{k+i,t} d_t l_{k+j,t}, i >= j, t in [0, k).
// MODE 2 (trsm) : P[r][t0+c] = (sum_t P[r][t0+t] M[c][t]) / d_{t0+c}, r >= t0+kb,
//                 c < kb (M = unit-lower inverse of the diagonal block at t0).
template <int BM_, int BN_, int BK_, int ST_, int WR_ = 4, int WC_ = 2>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, ST = ST_, LD = BK_ + 4;
  static constexpr int WR = WR_, WC = WC_, NT = 32 * WR_ * WC_;  // warp grid, threads
  static constexpr int WM = BM / WR, WN = BN / WC, MI = WM / 8, NJ = WN / 8;
  static constexpr size_t smem = sizeof(double) * (ST * (BM + BN) * LD + ST * BK);
};

template <int MODE, class G>
__global__ void __launch_bounds__(G::NT) large_update_kernel(LevelArgs L, double* factors,
                                                            double* upd, int row0, int col0,
                                                            int col1, int t0, int t1) {
  constexpr int BM = G::BM, BN = G::BN, BK = G::BK, ST = G::ST, LD = G::LD;
  constexpr int MI = G::MI, NJ = G::NJ;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                       // [ST][BM][LD]
  double* Bs = As + ST * BM * LD;         // [ST][BN][LD]
  double* Ds = Bs + ST * BN * LD;         // [ST][BK]
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  double* Pf = factors + f * L.fac_stride;
  const double* dvec = Pf + (long long)m * kp;
  const double* Bbase = Pf;
  int ldb = kp, aRow0, bRow0, nA, nB, aK0, bK0, kLen;
  long long tile_r0, tile_c0;
  if (MODE == 0) {
    tile_r0 = row0 + (long long)blockIdx.z * BM;
    tile_c0 = col0 + (long long)blockIdx.y * BN;
    const int cLim = min(col1, k);
    if (tile_r0 >= m || tile_c0 >= cLim || tile_r0 + BM <= tile_c0) return;
    aRow0 = (int)tile_r0;
    bRow0 = (int)tile_c0;
    nA = min(BM, m - aRow0);
    nB = min(BN, cLim - bRow0);
    aK0 = bK0 = t0;
    kLen = min(t1, k) - t0;
  } else if (MODE == 1) {
    const int u = m - k;
    tile_r0 = (long long)blockIdx.z * BM;
    tile_c0 = (long long)blockIdx.y * BN;
    if (tile_r0 >= u || tile_c0 >= u || tile_r0 + BM <= tile_c0) return;
    aRow0 = k + (int)tile_r0;
    bRow0 = k + (int)tile_c0;
    nA = min(BM, u - (int)tile_r0);
    nB = min(BN, u - (int)tile_c0);
    aK0 = bK0 = 0;
    kLen = k;
  } else {
    const int kb = min(t0 + NB, k) - t0;
    if (kb <= 0) return;
    tile_r0 = t0 + kb + (long long)blockIdx.z * BM;
    tile_c0 = t0;
    if (tile_r0 >= m) return;
    aRow0 = (int)tile_r0;
    nA = min(BM, m - aRow0);
    Bbase = L.aux + f * L.aux_stride + (long long)(t0 / NB) * NB * NB;
    ldb = NB;
    bRow0 = 0;
    nB = kb;
    aK0 = t0;
    bK0 = 0;
    kLen = kb;
  }
  if (kLen <= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp / G::WC, wx = warp % G::WC;  // WR x WC warps
  const int nk = (kLen + BK - 1) / BK;
  constexpr int CPR = BK / 2;  // 16-byte chunks per tile row

  auto issue = [&](int it) {
    const int stage = it % ST;
    const int kt = it * BK;
    double* as = As + stage * BM * LD;
    double* bs = Bs + stage * BN * LD;
#pragma unroll
    for (int q = 0; q < (BM * CPR + G::NT - 1) / G::NT; q++) {
      const int ch = tid + q * G::NT;
      if (ch >= BM * CPR) break;
      const int r = ch / CPR, cc = (ch % CPR) * 2;
      const int t = kt + cc;
      const bool v = r < nA && t < kLen;
      const double* src = v ? Pf + (long long)(aRow0 + r) * kp + aK0 + t : Pf;
      cp_async16(as + r * LD + cc, src, v);
    }
#pragma unroll
    for (int q = 0; q < (BN * CPR + G::NT - 1) / G::NT; q++) {
      const int ch = tid + q * G::NT;
      if (ch >= BN * CPR) break;
      const int r = ch / CPR, cc = (ch % CPR) * 2;
      const int t = kt + cc;
      const bool v = r < nB && t < kLen;
      const double* src = v ? Bbase + (long long)(bRow0 + r) * ldb + bK0 + t : Bbase;
      cp_async16(bs + r * LD + cc, src, v);
    }
    if (MODE != 2 && tid < CPR) {
      const int t = kt + tid * 2;
      cp_async16(Ds + stage * BK + tid * 2, t < kLen ? dvec + aK0 + t : dvec, t < kLen);
    }
  };

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; i++)
#pragma unroll
    for (int j = 0; j < NJ; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int it = 0; it < ST - 1; it++) {
    if (it < nk) issue(it);
    cp_async_commit();
  }
  for (int it = 0; it < nk; it++) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    if (it + ST - 1 < nk) issue(it + ST - 1);
    cp_async_commit();
    const int stage = it % ST;
    const double* as = As + stage * BM * LD + (wy * G::WM + (lane >> 2)) * LD + (lane & 3);
    const double* bs = Bs + stage * BN * LD + (wx * G::WN + (lane >> 2)) * LD + (lane & 3);
    const double* ds = Ds + stage * BK + (lane & 3);
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[MI], bf[NJ];
      if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < MI; i++) af[i] = as[i * 8 * LD + ks];
      } else {
        const double dk = ds[ks];
#pragma unroll
        for (int i = 0; i < MI; i++) af[i] = as[i * 8 * LD + ks] * dk;
      }
#pragma unroll
      for (int j = 0; j < NJ; j++) bf[j] = bs[j * 8 * LD + ks];
      if (MODE == 2) {  // aux block: use its strict lower part, unit diagonal
        const int tk = it * BK + ks + (lane & 3);
#pragma unroll
        for (int j = 0; j < NJ; j++) {
          const int n = wx * G::WN + j * 8 + (lane >> 2);
          bf[j] = tk < n ? bf[j] : (tk == n ? 1.0 : 0.0);
        }
      }
#pragma unroll
      for (int i = 0; i < MI; i++)
#pragma unroll
        for (int j = 0; j < NJ; j++) dmma884(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  if (MODE == 2) __syncthreads();  // every A tile row is read before it is overwritten
  double* out = MODE == 1 ? upd + f * L.upd_stride : Pf;
#pragma unroll
  for (int i = 0; i < MI; i++) {
    const int rl = wy * G::WM + i * 8 + (lane >> 2);
    if (rl >= nA) continue;
    const long long R = tile_r0 + rl;
#pragma unroll
    for (int j = 0; j < NJ; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int cl = wx * G::WN + j * 8 + 2 * (lane & 3) + h;
        if (cl >= nB) continue;
        const long long C = tile_c0 + cl;
        if (MODE == 2) {
          out[R * kp + C] = acc[i][j][h] / dvec[C];
        } else {
          if (C > R) continue;
          if (MODE == 0) out[R * kp + C] -= acc[i][j][h];
          else out[tri(R, C)] -= acc[i][j][h];
        }
      }
    }
  }
}

// Tile shapes measured on B200 (tools/schur_sweep.sh): 64x64 tiles of 8 warps
// with a 2-stage pipeline keep the most warps resident and win on every level.
using GTrsm = GemmCfg<64, 64, 16, 2>;   // N = 64 = one diagonal block
using GPanel = GemmCfg<64, 64, 16, 2>;
using GSchurA = GemmCfg<64, 64, 16, 2>;        // 8 warps of 16x32
using GSchurB = GemmCfg<64, 64, 8, 4>;
using GSchurC = GemmCfg<64, 64, 16, 3, 2, 2>;  // 4 warps of 32x32
using GSchurD = GemmCfg<64, 32, 16, 3, 4, 1>;  // 4 warps of 16x32
using GSchurE = GemmCfg<128, 64, 16, 3>;

template <int MODE, class G>
static void gemm_attr() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(large_update_kernel<MODE, G>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem);
    done = true;
  }
}

template <class G>
static void launch_schur(const LevelArgs& L, double* factors, double* upd_out, cudaStream_t st) {
  gemm_attr<1, G>();
  dim3 g((unsigned)L.n_fronts, (unsigned)((L.max_upd + G::BN - 1) / G::BN),
         (unsigned)((L.max_upd + G::BM - 1) / G::BM));
  large_update_kernel<1, G><<<g, G::NT, G::smem, st>>>(L, factors, upd_out, 0, 0, 0, 0, 0);
}

static int gemm_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFB_SCHUR_CFG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

static cudaError_t panel_factor(const LevelArgs& L, double* factors, double thr,
                                unsigned long long* err, int a, int b, cudaStream_t st) {
  if (b - a <= NB) {
    const int rows = std::max(1, L.max_m - a - 1);
    if (L.level_fronts <= kFusedBlockMaxFronts) {
      // few fronts: one launch per block (redundant per-CTA diagonal factorization)
      dim3 g((unsigned)L.n_fronts, (unsigned)((rows + TRB - 1) / TRB));
      timer_begin(K_BLOCK, st);
      large_block_kernel<<<g, 256, kBlockSmem, st>>>(L, factors, a, thr, err);
      timer_end(st);
    } else {
      // many fronts: register-tiled diagonal blocks, then the TRSM as a DMMA GEMM
      timer_begin(K_DIAG, st);
      large_diag_kernel<<<L.n_fronts, 256, 0, st>>>(L, factors, a, thr, err);
      timer_end(st);
      dim3 g((unsigned)L.n_fronts, 1, (unsigned)((rows + GTrsm::BM - 1) / GTrsm::BM));
      gemm_attr<2, GTrsm>();
      timer_begin(K_TRSM, st);
      large_update_kernel<2, GTrsm><<<g, GTrsm::NT, GTrsm::smem, st>>>(L, factors, nullptr, 0, 0, 0,
                                                                   a, 0);
      timer_end(st);
    }
    return cudaGetLastError();
  }
  int mid = a + ((b - a) / 2 + NB - 1) / NB * NB;
  if (mid >= b) mid = a + NB;
  cudaError_t e = panel_factor(L, factors, thr, err, a, mid, st);
  if (e != cudaSuccess) return e;
  dim3 g((unsigned)L.n_fronts, (unsigned)((b - mid + GPanel::BN - 1) / GPanel::BN),
         (unsigned)((L.max_m - mid + GPanel::BM - 1) / GPanel::BM));
  gemm_attr<0, GPanel>();
  timer_begin(K_PANEL, st);
  large_update_kernel<0, GPanel><<<g, GPanel::NT, GPanel::smem, st>>>(L, factors, nullptr, mid, mid, b,
                                                                  a, mid);
  timer_end(st);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return panel_factor(L, factors, thr, err, mid, b, st);
}

cudaError_t launch_factor_large(const LevelArgs& L, const double* child_upd, double* factors,
                                double* upd_out, double thr, unsigned long long* err,
                                cudaStream_t st) {
  if (L.is_leaf) return cudaErrorInvalidValue;  // element fronts are never this large
  if (L.max_k > 0 && (!L.aux || L.aux_stride < large_aux_doubles(L.max_k)))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(large_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBlockSmem);
    attr = true;
  }
  {
    const long long per = L.fac_stride + tri(L.max_upd, 0);
    const unsigned gx = (unsigned)std::min<long long>((per + 255) / 256, 1024);
    timer_begin(K_ASSEMBLE, st);
    large_assemble_kernel<<<dim3(L.n_fronts, gx), 256, 0, st>>>(L, child_upd, factors, upd_out);
    timer_end(st);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (L.max_k > 0) {
    e = panel_factor(L, factors, thr, err, 0, L.max_k, st);
    if (e != cudaSuccess) return e;
  }
  if (L.max_upd > 0 && L.max_k > 0) {
    timer_begin(K_SCHUR, st);
    switch (gemm_variant()) {
      case 1: launch_schur<GSchurB>(L, factors, upd_out, st); break;
      case 2: launch_schur<GSchurC>(L, factors, upd_out, st); break;
      case 3: launch_schur<GSchurD>(L, factors, upd_out, st); break;
      case 4: launch_schur<GSchurE>(L, factors, upd_out, st); break;
      default: launch_schur<GSchurA>(L, factors, upd_out, st); break;
    }
    timer_end(st);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (L.max_k > 0) {
    dim3 g((unsigned)L.n_fronts, (unsigned)((L.max_k + NB - 1) / NB));
    timer_begin(K_FINALIZE, st);
    large_diag_finalize_kernel<<<g, 256, 0, st>>>(L, factors);
    timer_end(st);
    e = cudaGetLastError();
  }
  return e;
}

long long large_aux_doubles(int max_k) {
  return (long long)((max_k + NB - 1) / NB) * NB * NB;
}

int large_panel_launches(int max_k, int n_fronts) {
  if (max_k <= 0) return 0;
  if (max_k <= NB) return n_fronts <= kFusedBlockMaxFronts ? 1 : 2;
  int mid = (max_k / 2 + NB - 1) / NB * NB;
  if (mid >= max_k) mid = NB;
  return large_panel_launches(mid, n_fronts) + 1 + large_panel_launches(max_k - mid, n_fronts);
}

}  // namespace tfb
