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
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace tfb {

constexpr int NB = 64;  // diagonal block width
#ifndef TFB_GEMM_MINB
#define TFB_GEMM_MINB 4  // CTAs per SM the DMMA GEMM kernels are compiled for
#endif

// Optional per-phase clock stamps of CTA 0 (tools/diag_bench.cu builds with it).
#ifdef TFB_PHASE_CLOCK
__device__ long long g_phase_clk[32];
#define TFB_PHASE(i)                                                          \
  do {                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_phase_clk[i] = clock64(); \
  } while (0)
#else
#define TFB_PHASE(i) \
  do {               \
  } while (0)
#endif

// Warp per front row (rows dealt round-robin over the CTAs of the front), lanes
// across the row's columns: the panel row P[r][0, kp) and, for r >= k, the
// packed Schur row S[r-k][0, r-k].  The row's child indices are warp-uniform;
// all index math is 32-bit (a front's packed child block is < 2^31 entries).
constexpr int kAsmWarps = 8, kAsmRowsPerWarp = 4;
__device__ __forceinline__ double child_entry(const double* __restrict__ src, int i, int tri_i,
                                              int j) {
  // packed lower-triangular (i, j) of the child block; -1 = not in this child
  if (i < 0 || j < 0) return 0.0;
  return src[i >= j ? tri_i + j : tri32(j, i)];
}
__global__ void __launch_bounds__(32 * kAsmWarps)
    large_assemble_kernel(LevelArgs L, const double* __restrict__ child_upd,
                          double* __restrict__ factors, double* __restrict__ upd, int with_s) {
  const long long f = blockIdx.x;  // fronts on x (no 65535 limit), row groups on y
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  double* Pf = factors + f * L.fac_stride;
  double* Sf = upd + f * L.upd_stride;
  const int* inv0 = L.maps + s.ioff;
  const int* inv1 = inv0 + m;
  const double* src0 = child_upd + L.child_slot(f, 0) * L.child_upd_stride;
  const double* src1 = child_upd + L.child_slot(f, 1) * L.child_upd_stride;
  const bool two = s.nsrc == 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (blockIdx.y == 0 && warp == 0)
    for (int c = lane; c < kp; c += 32) Pf[(long long)m * kp + c] = 0.0;  // d (set by the diag)
  for (int r = blockIdx.y * kAsmWarps + warp; r < m; r += gridDim.y * kAsmWarps) {
    const int i0 = inv0[r], t0 = i0 >= 0 ? tri32(i0, 0) : 0;
    const int i1 = two ? inv1[r] : -1, t1 = i1 >= 0 ? tri32(i1, 0) : 0;
    double* prow = Pf + (long long)r * kp;
    const int pc = min(r + 1, k);
    if (kp <= 32) {  // narrow panels: one column per lane
      double v = 0.0;
      if (lane < pc) v = child_entry(src0, i0, t0, inv0[lane]) + child_entry(src1, i1, t1, two ? inv1[lane] : -1);
      if (lane < kp) prow[lane] = v;
    } else
    for (int c0 = lane; c0 < kp; c0 += 128) {  // 4 columns per lane in flight
      int j0[4], j1[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int c = c0 + 32 * q;
        j0[q] = c < pc ? inv0[c] : -1;
        j1[q] = (two && c < pc) ? inv1[c] : -1;
      }
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; q++)
        v[q] = child_entry(src0, i0, t0, j0[q]) + child_entry(src1, i1, t1, j1[q]);
#pragma unroll
      for (int q = 0; q < 4; q++)
        if (c0 + 32 * q < kp) prow[c0 + 32 * q] = v[q];
    }
    if (with_s && r >= k) {  // else the Schur kernel assembles S in its epilogue
      const int a = r - k;
      double* srow = Sf + tri32(a, 0);
      for (int c = lane; c <= a; c += 32) {
        double v = child_entry(src0, i0, t0, inv0[k + c]);
        if (two) v += child_entry(src1, i1, t1, inv1[k + c]);
        srow[c] = v;
      }
    }
  }
}

// ---------------------------------------------------------------- diagonal blocks
// Warp-level LDL^T of a 32x32 symmetric block held in registers: lane r owns
// row r (v[j] = a(r, j) for j <= r, v[j > r] = 0; padding rows are unit rows).
// Pivot c: d = a(c, c) from lane c, l(r, c) = a(r, c) / d, and the rank-1 update
// a(r, j) -= l(r, c) a(j, c) takes a(j, c) from lane j by shuffle.  On return
// v[j < r] = l(r, j) and v[r] = d_r.  No shared memory, no barriers.
__device__ __forceinline__ void warp_ldl32(double (&v)[32], int lane) {
#pragma unroll
  for (int c = 0; c < 32; c++) {
    const double d = __shfl_sync(0xffffffffu, v[c], c);
    const double l = v[c] * (1.0 / d);
#pragma unroll
    for (int j = c + 1; j < 32; j++) {
      const double ajc = __shfl_sync(0xffffffffu, v[c], j);
      if (lane >= j) v[j] -= l * ajc;
    }
    if (lane > c) v[c] = l;
  }
}

// Row `lane` of M = L^-1 for the unit-lower L in v (warp_ldl32 output):
// w[j] = M(lane, j), j < lane; w[lane] = 1; w[j > lane] = 0.  Right-looking:
// after step t row t is final and rows below subtract l(r, t) M(t, :).
__device__ __forceinline__ void warp_inv32(const double (&v)[32], double (&w)[32], int lane) {
#pragma unroll
  for (int j = 0; j < 32; j++) w[j] = j == lane ? 1.0 : 0.0;
#pragma unroll
  for (int t = 0; t < 31; t++) {
#pragma unroll
    for (int j = 0; j <= t; j++) {
      const double mtj = __shfl_sync(0xffffffffu, w[j], t);
      if (lane > t) w[j] -= v[t] * mtj;
    }
  }
}

__device__ __forceinline__ double reg_pick(const double (&v)[32], int i) {
  double x = 0.0;
#pragma unroll
  for (int j = 0; j < 32; j++) x = j == i ? v[j] : x;
  return x;
}

// One warp per front: diagonal blocks of width kb <= 32 (4 fronts per CTA).
// Writes l (strict lower) and d into the panel, d into the pivot vector and
// the aux block (strict lower = M, diagonal = d, strict upper = l^T).
__global__ void __launch_bounds__(128) large_diag32_kernel(LevelArgs L, double* factors, int a,
                                                            double threshold,
                                                            unsigned long long* err) {
  const int lane = threadIdx.x & 31;
  const long long f = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (f >= L.n_fronts) return;
  const Shape s = front_shape(L, f);
  const int kb = min(a + NB, s.k) - a;
  if (kb <= 0) return;
  double* Pf = factors + f * L.fac_stride;
  double v[32];
  const double* prow = Pf + (long long)(a + lane) * s.kp + a;
#pragma unroll
  for (int j = 0; j < 32; j++)
    v[j] = lane < kb ? (j <= lane ? prow[j] : 0.0) : (j == lane ? 1.0 : 0.0);
  warp_ldl32(v, lane);
  const double dr = reg_pick(v, lane);
  if (lane < kb && fabs(dr) <= threshold)
    record_zero_pivot(err, (unsigned long long)(L.piv_off[f] + a + lane));
  double* M = L.aux + f * L.aux_stride + (long long)(a / NB) * NB * NB;
  if (lane < kb) {
    double* pw = Pf + (long long)(a + lane) * s.kp + a;
#pragma unroll
    for (int j = 0; j < 32; j++)
      if (j <= lane) pw[j] = v[j];
    Pf[(long long)s.m * s.kp + a + lane] = dr;
  }
  double w[32];
  warp_inv32(v, w, lane);
  // aux rows/cols [0, 32) of the 64x64 block; the rest is the identity
#pragma unroll
  for (int j = 0; j < 32; j++) {
    if (j < lane) {
      M[lane * NB + j] = w[j];
      M[j * NB + lane] = lane < kb ? v[j] : 0.0;
    }
  }
  M[lane * NB + lane] = lane < kb ? dr : 1.0;
  for (int e = lane; e < 32 * NB; e += 32) {  // rows 32..63: identity
    const int i = 32 + e / NB, j = e % NB;
    M[i * NB + j] = i == j ? 1.0 : 0.0;
  }
  for (int e = lane; e < 32 * 32; e += 32) M[(e >> 5) * NB + 32 + (e & 31)] = 0.0;
}

// 64x64 diagonal-block LDL^T + inverse in shared memory, few barriers:
//   for each 16-column panel: one warp factors it warp-synchronously (lane
//   owns rows c0+lane and c0+32+lane in registers, pivot columns broadcast by
//   shuffles, fully unrolled so register indices are static), then all warps
//   apply the rank-16 update to the trailing block with DMMA;
//   M = L^-1 from 16x16 diagonal-block inverses (one warp each) and block
//   rows M_ij = -M_ii sum_{t=j}^{i-1} L_it M_tj.
// D (ld DLD): the block with unit rows beyond kb; on return its lower part
// holds l (strict) and d (diagonal), dv = d, Mi = L^-1 (unit diagonal, zero
// upper part).  NT threads; ends with a barrier.
constexpr int DLD = NB + 1;

// 1/d: hardware approximation refined by two Newton steps (full double
// precision for normal d; shorter dependency chain than the IEEE division).
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  return fma(r, fma(-d, r, 1.0), r);
}

__device__ __forceinline__ void panel16_warp(double (*D)[DLD], double* dv, int c0, int lane) {
  const int r0 = c0 + lane, r1 = c0 + 32 + lane;
  const bool h0 = r0 < NB, h1 = r1 < NB;
  double x0[16], x1[16];
#pragma unroll
  for (int j = 0; j < 16; j++) {
    x0[j] = h0 ? D[r0][c0 + j] : 0.0;
    x1[j] = h1 ? D[r1][c0 + j] : 0.0;
  }
#pragma unroll
  for (int cc = 0; cc < 16; cc++) {
    const double d = __shfl_sync(0xffffffffu, x0[cc], cc);
    const double inv = rcp_nr(d);
    const double l0 = x0[cc] * inv, l1 = x1[cc] * inv;
#pragma unroll
    for (int jj = cc + 1; jj < 16; jj++) {
      const double ajc = __shfl_sync(0xffffffffu, x0[cc], jj);  // a(c0+jj, c0+cc)
      x0[jj] -= l0 * ajc;  // (entries right of the diagonal are never read)
      x1[jj] -= l1 * ajc;
    }
    if (lane > cc) x0[cc] = l0;
    x1[cc] = l1;
  }
#pragma unroll
  for (int j = 0; j < 16; j++) {
    if (h0 && j <= lane) D[r0][c0 + j] = x0[j];
    if (h1) D[r1][c0 + j] = x1[j];
  }
  if (lane < 16) {
    double x = 0.0;
#pragma unroll
    for (int j = 0; j < 16; j++) x = j == lane ? x0[j] : x;
    dv[c0 + lane] = x;
  }
}

// Row r of the inverse of the 16x16 unit-lower block of D at (o, o), by the
// half-warp owning it (lane & 15 = r; width-16 shuffles).  Writes the full
// 16x16 block of Mi (unit diagonal, zeros above).
__device__ __forceinline__ void inv16_half(double (*D)[DLD], double (*Mi)[DLD], int o, int r) {
  double l[16], w[16];
#pragma unroll
  for (int j = 0; j < 16; j++) {
    l[j] = j < r ? D[o + r][o + j] : 0.0;
    w[j] = j == r ? 1.0 : 0.0;
  }
#pragma unroll
  for (int t = 0; t < 15; t++) {
#pragma unroll
    for (int j = 0; j <= t; j++) {
      const double mtj = __shfl_sync(0xffffffffu, w[j], t, 16);
      if (r > t) w[j] -= l[t] * mtj;
    }
  }
#pragma unroll
  for (int j = 0; j < 16; j++) Mi[o + r][o + j] = w[j];
}

// C = alpha A B for shared-memory operands on 8x8 DMMA tiles (A(i,k) =
// A[i*lda+k], B(k,n) = B[k*ldb+n]; M, N multiples of 8, K of 4).
template <int NT, int MT>
__device__ __forceinline__ void smem_gemm(double* C, int ldc, const double* A, int lda,
                                          const double* B, int ldb, int M, int N, int K,
                                          double alpha) {
  // MT = tiles per warp (ceil(tiles / warps)), accumulated side by side
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g8 = lane >> 2, tq = lane & 3;
  const int TN = N >> 3, ntile = (M >> 3) * TN;
  double acc[MT][2];
  int I[MT], J[MT];
#pragma unroll
  for (int q = 0; q < MT; q++) {
    const int tile = warp + q * (NT / 32);
    I[q] = tile / TN;
    J[q] = tile - I[q] * TN;
    acc[q][0] = acc[q][1] = 0.0;
  }
  for (int k = 0; k < K; k += 4) {
#pragma unroll
    for (int q = 0; q < MT; q++)
      if (warp + q * (NT / 32) < ntile)
        dmma884(acc[q], A[(8 * I[q] + g8) * lda + k + tq], B[(k + tq) * ldb + 8 * J[q] + g8]);
  }
#pragma unroll
  for (int q = 0; q < MT; q++) {
    if (warp + q * (NT / 32) >= ntile) continue;
    double* c = C + (8 * I[q] + g8) * ldc + 8 * J[q] + 2 * tq;
    c[0] = alpha * acc[q][0];
    c[1] = alpha * acc[q][1];
  }
}

template <int NT>
__device__ void diag64_smem(double (*D)[DLD], double (*Mi)[DLD], double* dv, int kb) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, tq = lane & 3;
  const int npan = (kb + 15) >> 4;
#pragma unroll 1
  for (int p = 0; p < 4; p++) {
    const int c0 = 16 * p;
    if (p < npan) {
      if (warp == 0) panel16_warp(D, dv, c0, lane);
    } else if (tid < 16) {
      dv[c0 + tid] = 1.0;  // unit padding
    }
    __syncthreads();
    TFB_PHASE(2 + 2 * p);
    // rank-16 DMMA update of the trailing lower block [c0+16, 64)
    const int t0 = c0 + 16;
    if (p + 1 < npan) {
      // every warp keeps its (<= MT) tiles' accumulators live so the DMMA
      // chains interleave instead of serialising on one accumulator
      const int T = (NB - t0) >> 3, ntile = T * (T + 1) / 2;
      constexpr int MT = (21 + NT / 32 - 1) / (NT / 32);
      double acc[MT][2];
      int ra[MT], rb[MT];
#pragma unroll
      for (int q = 0; q < MT; q++) {
        const int tile = warp + q * (NT / 32);
        int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
        I -= (I * (I + 1) / 2 > tile);
        I += ((I + 1) * (I + 2) / 2 <= tile);
        const int J = tile - I * (I + 1) / 2;
        ra[q] = t0 + 8 * I + g8;
        rb[q] = t0 + 8 * J + g8;
        acc[q][0] = acc[q][1] = 0.0;
      }
#pragma unroll
      for (int kk = 0; kk < 16; kk += 4) {
        const int qc = c0 + kk + tq;
        const double dq = dv[qc];
#pragma unroll
        for (int q = 0; q < MT; q++)
          if (warp + q * (NT / 32) < ntile) dmma884(acc[q], D[ra[q]][qc] * dq, D[rb[q]][qc]);
      }
#pragma unroll
      for (int q = 0; q < MT; q++) {
        if (warp + q * (NT / 32) >= ntile) continue;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int cc = (rb[q] - g8) + 2 * tq + h;
          if (cc <= ra[q]) D[ra[q]][cc] -= acc[q][h];
        }
      }
      __syncthreads();
      TFB_PHASE(3 + 2 * p);
    }
  }
  // M = L^-1 by recursive doubling: 16x16 diagonal-block inverses (half-warps,
  // registers + width-16 shuffles), then M21 = -M22 (L21 M11) at the 32- and
  // 64-levels as DMMA products (scratch: upper part of Mi, cleared after use).
  if (warp < 2) inv16_half(D, Mi, 16 * (2 * warp + (lane >> 4)), lane & 15);
  __syncthreads();
  TFB_PHASE(10);
  smem_gemm<NT, (4 + NT / 32 - 1) / (NT / 32)>(&Mi[0][16], DLD, &D[16][0], DLD, &Mi[0][0], DLD, 16, 16, 16, 1.0);
  smem_gemm<NT, (4 + NT / 32 - 1) / (NT / 32)>(&Mi[32][48], DLD, &D[48][32], DLD, &Mi[32][32], DLD, 16, 16, 16, 1.0);
  __syncthreads();
  smem_gemm<NT, (4 + NT / 32 - 1) / (NT / 32)>(&Mi[16][0], DLD, &Mi[16][16], DLD, &Mi[0][16], DLD, 16, 16, 16, -1.0);
  smem_gemm<NT, (4 + NT / 32 - 1) / (NT / 32)>(&Mi[48][32], DLD, &Mi[48][48], DLD, &Mi[32][48], DLD, 16, 16, 16, -1.0);
  __syncthreads();
  for (int e = tid; e < 2 * 256; e += NT) {
    const int o = (e >> 8) * 32, r = (e >> 4) & 15, c = e & 15;
    Mi[o + r][o + 16 + c] = 0.0;
  }
  __syncthreads();
  TFB_PHASE(11);
  if (kb > 32) {
    smem_gemm<NT, (16 + NT / 32 - 1) / (NT / 32)>(&Mi[0][32], DLD, &D[32][0], DLD, &Mi[0][0], DLD, 32, 32, 32, 1.0);
    __syncthreads();
    smem_gemm<NT, (16 + NT / 32 - 1) / (NT / 32)>(&Mi[32][0], DLD, &Mi[32][32], DLD, &Mi[0][32], DLD, 32, 32, 32, -1.0);
  } else {
    for (int e = tid; e < 32 * 32; e += NT) Mi[32 + (e >> 5)][e & 31] = 0.0;
  }
  __syncthreads();
  for (int e = tid; e < 32 * 32; e += NT) Mi[e >> 5][32 + (e & 31)] = 0.0;
  __syncthreads();
  TFB_PHASE(12);
}

// aux block: strict lower = M, diagonal = d (1 beyond kb), strict upper = l^T.
template <int NT>
__device__ __forceinline__ void write_aux64(double* M, double (*D)[DLD], double (*Mi)[DLD],
                                            const double* dv, int kb) {
  for (int e = threadIdx.x; e < NB * NB; e += NT) {
    const int i = e >> 6, j = e & 63;
    M[e] = j < i ? Mi[i][j] : (j == i ? (i < kb ? dv[i] : 1.0) : (j < kb ? D[j][i] : 0.0));
  }
}

template <int NT>
__device__ __forceinline__ void load_diag_block(double (*D)[DLD], const double* Pf, int kp, int a,
                                                int kb) {
  // every load of the block in flight before the first shared-memory store
  constexpr int Q = NB * NB / NT;
  double t[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int e = threadIdx.x + q * NT, i = e >> 6, j = e & 63;
    t[q] = (i < kb && j <= i) ? Pf[(long long)(a + i) * kp + a + j] : (i == j ? 1.0 : 0.0);
  }
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int e = threadIdx.x + q * NT;
    D[e >> 6][e & 63] = t[q];
  }
}

constexpr size_t kDiagSmem = sizeof(double) * (2 * NB * DLD + NB);

// One CTA per front: diagonal blocks of width kb in (32, 64].  Writes l and d
// into the panel, d into the pivot vector, and the aux block.
__global__ void __launch_bounds__(256) large_diag64_kernel(LevelArgs L, double* factors, int a,
                                                            double threshold,
                                                            unsigned long long* err) {
  extern __shared__ __align__(16) double dsm[];
  double(*D)[DLD] = reinterpret_cast<double(*)[DLD]>(dsm);
  double(*Mi)[DLD] = reinterpret_cast<double(*)[DLD]>(dsm + NB * DLD);
  double* dv = dsm + 2 * NB * DLD;
  const long long f = blockIdx.x;
  const Shape s = front_shape(L, f);
  const int kb = min(a + NB, s.k) - a;
  if (kb <= 0) return;
  double* Pf = factors + f * L.fac_stride;
  TFB_PHASE(0);
  load_diag_block<256>(D, Pf, s.kp, a, kb);
  __syncthreads();
  TFB_PHASE(1);
  diag64_smem<256>(D, Mi, dv, kb);
  for (int e = threadIdx.x; e < NB * NB; e += 256) {
    const int i = e >> 6, j = e & 63;
    if (i < kb && j <= i) Pf[(long long)(a + i) * s.kp + a + j] = D[i][j];
  }
  for (int c = threadIdx.x; c < kb; c += 256) {
    Pf[(long long)s.m * s.kp + a + c] = dv[c];
    if (fabs(dv[c]) <= threshold) record_zero_pivot(err, (unsigned long long)(L.piv_off[f] + a + c));
  }
  write_aux64<256>(L.aux + f * L.aux_stride + (long long)(a / NB) * NB * NB, D, Mi, dv, kb);
  TFB_PHASE(13);
}

// One 64-wide diagonal block of every front's panel, fused with the triangular
// solve of the rows below it.  grid = (fronts, row tiles of 64).  Every CTA
// factors the diagonal block redundantly (diag64_smem), then solves its 64-row
// tile as a DMMA product P_rb <- (P_rb M^T) D^-1.  The CTA of row tile 0 also
// writes d and the aux block.
constexpr int TRB = 64;
// Measured (cfg5 L23, 64^3 L17): at 2 fronts the redundant per-CTA diagonal
// factorizations steal more SM time from the concurrent Schur stream than the
// separate TRSM launch costs (5.29 -> 4.67 ms); the fused kernel now serves
// single-front levels only (the root when TFB_ROOT_DATAFLOW=0)
constexpr int kFusedBlockMaxFronts = 1;
constexpr int ALD = NB + 4;
constexpr size_t kBlockSmem = sizeof(double) * (2 * NB * DLD + TRB * ALD + NB);

__global__ void __launch_bounds__(256) large_block_kernel(LevelArgs L, double* factors, int a,
                                                           double threshold,
                                                           unsigned long long* err) {
  extern __shared__ __align__(16) double bsm[];
  double(*D)[DLD] = reinterpret_cast<double(*)[DLD]>(bsm);
  double(*Mi)[DLD] = reinterpret_cast<double(*)[DLD]>(bsm + NB * DLD);
  double(*At)[ALD] = reinterpret_cast<double(*)[ALD]>(bsm + 2 * NB * DLD);
  double* dv = bsm + 2 * NB * DLD + TRB * ALD;
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

  // 1. diagonal block (unit rows beyond kb) and this CTA's row tile
  load_diag_block<256>(D, Pf, s.kp, a, kb);
  for (int e = tid; e < TRB * NB; e += 256) {
    const int i = e >> 6, j = e & 63;
    At[i][j] = (i < rows && j < kb) ? Pf[(long long)(row0 + i) * s.kp + a + j] : 0.0;
  }
  __syncthreads();
  // 2. factor + invert the diagonal block
  diag64_smem<256>(D, Mi, dv, kb);
  // 3. the writer CTA stores d and the aux block.  The panel's own diagonal
  // block is not rewritten here: other CTAs of this launch may still be
  // reading its assembled values, so large_diag_finalize_kernel copies l, d
  // into it after the level.
  if (writer) {
    for (int c = tid; c < kb; c += 256) {
      Pf[(long long)s.m * s.kp + a + c] = dv[c];
      if (fabs(dv[c]) <= threshold)
        record_zero_pivot(err, (unsigned long long)(L.piv_off[f] + a + c));
    }
    write_aux64<256>(L.aux + f * L.aux_stride + (long long)(a / NB) * NB * NB, D, Mi, dv, kb);
  }
  // 4. row tile: X = At M^T, then column c / d_c (DMMA, 8 tiles of 8x8 per warp)
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
__global__ void __launch_bounds__(G::NT, TFB_GEMM_MINB) large_update_kernel(LevelArgs L, double* factors,
                                                            double* upd, int row0, int col0,
                                                            int col1, int t0, int t1,
                                                            const double* __restrict__ child_upd,
                                                            int asm_s) {
  constexpr int BM = G::BM, BN = G::BN, BK = G::BK, ST = G::ST, LD = G::LD;
  constexpr int MI = G::MI, NJ = G::NJ;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                       // [ST][BM][LD]
  double* Bs = As + ST * BM * LD;         // [ST][BN][LD]
  double* Ds = Bs + ST * BN * LD;         // [ST][BK]
  // MODE 1: 1-D grid over (front, lower-triangular tile (I, J)) in row-major
  // tile order, so co-resident CTAs share L21 row tiles in L2 (col0 = tiles
  // per dimension); other modes: fronts on x
  long long f = blockIdx.x;
  int tI = 0, tJ = 0;
  if (MODE == 1) {
    const long long ntf = (long long)col0 * (col0 + 1) / 2;
    f = (long long)blockIdx.x / ntf;
    const int t = (int)((long long)blockIdx.x - f * ntf);
    tI = tri_row32(t);
    tJ = t - (int)tri32(tI, 0);
  }
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
    tile_r0 = (long long)tI * BM;
    tile_c0 = (long long)tJ * BN;
    if (tile_r0 >= u) return;
    aRow0 = k + (int)tile_r0;
    bRow0 = k + (int)tile_c0;
    nA = min(BM, u - (int)tile_r0);
    nB = min(BN, u - (int)tile_c0);
    aK0 = bK0 = t1 > t0 ? t0 : 0;  // pivot columns [t0, t1) (lookahead chunks) or all
    kLen = t1 > t0 ? min(t1, k) - t0 : k;
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
  if (kLen <= 0) {
    if (!(MODE == 1 && asm_s)) return;
    kLen = 0;  // no pivots in this front: S is its assembled block
  }
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
  if (MODE == 1 && asm_s) {
    // S = (children's contributions, gathered through the inverse extend-add
    // maps: the assembly of S fused here) - L21 D L21^T; one write per entry
    const int* inv0 = L.maps + s.ioff;
    const int* inv1 = inv0 + m;
    const bool two = s.nsrc == 2;
    const double* src0 = child_upd + L.child_slot(f, 0) * L.child_upd_stride;
    const double* src1 = child_upd + L.child_slot(f, 1) * L.child_upd_stride;
    // column maps once per thread, then per row: all child loads issued
    // before any store (no branches between them)
    int b0[NJ][2], b1[NJ][2];
#pragma unroll
    for (int j = 0; j < NJ; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int cl = wx * G::WN + j * 8 + 2 * (lane & 3) + h;
        const bool ok = cl < nB;
        b0[j][h] = ok ? __ldg(inv0 + k + (int)tile_c0 + cl) : -1;
        b1[j][h] = (ok && two) ? __ldg(inv1 + k + (int)tile_c0 + cl) : -1;
      }
#pragma unroll
    for (int i = 0; i < MI; i++) {
      const int rl = wy * G::WM + i * 8 + (lane >> 2);
      const bool okr = rl < nA;
      const int R = (int)tile_r0 + rl;
      const int a0 = okr ? __ldg(inv0 + k + R) : -1, ta0 = a0 >= 0 ? tri32(a0, 0) : 0;
      const int a1 = (okr && two) ? __ldg(inv1 + k + R) : -1, ta1 = a1 >= 0 ? tri32(a1, 0) : 0;
      double v[NJ][2];
#pragma unroll
      for (int j = 0; j < NJ; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int c0 = b0[j][h], c1 = b1[j][h];
          const double x0 = (a0 >= 0 && c0 >= 0) ? __ldg(src0 + (a0 >= c0 ? ta0 + c0 : tri32(c0, a0))) : 0.0;
          const double x1 = (a1 >= 0 && c1 >= 0) ? __ldg(src1 + (a1 >= c1 ? ta1 + c1 : tri32(c1, a1))) : 0.0;
          v[j][h] = x0 + x1;
        }
      if (!okr) continue;
      double* orow = out + tri32(R, 0);
#pragma unroll
      for (int j = 0; j < NJ; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int cl = wx * G::WN + j * 8 + 2 * (lane & 3) + h;
          const int C = (int)tile_c0 + cl;
          if (cl < nB && C <= R) orow[C] = v[j][h] - acc[i][j][h];
        }
    }
    return;
  }
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

// Tile shapes measured on B200 (A/B builds via TFB_LIB): 64x64 tiles of 8 warps
// with a 2-stage pipeline keep the most warps resident and win on every level.
using GTrsm = GemmCfg<64, 64, 16, 2>;   // N = 64 = one diagonal block
using GTrsm32 = GemmCfg<64, 32, 16, 2, 4, 1>;  // blocks of <= 32 columns: 4 warps of 16x32
using GPanel = GemmCfg<64, 64, 16, 2>;
using GSchurA = GemmCfg<64, 64, 16, 2>;        // 8 warps of 16x32

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
static void launch_schur(const LevelArgs& L, double* factors, double* upd_out, cudaStream_t st,
                         int t0 = 0, int t1 = 0, const double* child_upd = nullptr) {
  // child_upd != nullptr: S is assembled in the epilogue (not by the assembly kernel)
  static_assert(G::BM == G::BN, "square Schur tiles");
  gemm_attr<1, G>();
  const int T = (L.max_upd + G::BM - 1) / G::BM;
  const long long grid = (long long)L.n_fronts * T * (T + 1) / 2;
  large_update_kernel<1, G><<<(unsigned)grid, G::NT, G::smem, st>>>(
      L, factors, upd_out, 0, T, 0, t0, t1, child_upd, child_upd ? 1 : 0);
}

// P[r][c] -= sum_{t in [t0, t1)} l_rt d_t l_ct for c in [c0, c1), r >= c.
static void launch_panel_update(const LevelArgs& L, double* factors, int c0, int c1, int t0,
                                int t1, cudaStream_t st) {
  dim3 g((unsigned)L.n_fronts, (unsigned)((c1 - c0 + GPanel::BN - 1) / GPanel::BN),
         (unsigned)((L.max_m - c0 + GPanel::BM - 1) / GPanel::BM));
  gemm_attr<0, GPanel>();
  timer_begin(K_PANEL, st);
  large_update_kernel<0, GPanel><<<g, GPanel::NT, GPanel::smem, st>>>(L, factors, nullptr, c0, c0,
                                                                      c1, t0, t1, nullptr, 0);
  timer_end(st);
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
      if (std::min(NB, L.max_k - a) <= 32)
        large_diag32_kernel<<<(L.n_fronts + 3) / 4, 128, 0, st>>>(L, factors, a, thr, err);
      else
        large_diag64_kernel<<<L.n_fronts, 256, kDiagSmem, st>>>(L, factors, a, thr, err);
      timer_end(st);
      dim3 g((unsigned)L.n_fronts, 1, (unsigned)((rows + GTrsm::BM - 1) / GTrsm::BM));
      timer_begin(K_TRSM, st);
      if (b - a <= 32) {
        gemm_attr<2, GTrsm32>();
        large_update_kernel<2, GTrsm32><<<g, GTrsm32::NT, GTrsm32::smem, st>>>(
            L, factors, nullptr, 0, 0, 0, a, 0, nullptr, 0);
      } else {
        gemm_attr<2, GTrsm>();
        large_update_kernel<2, GTrsm><<<g, GTrsm::NT, GTrsm::smem, st>>>(L, factors, nullptr, 0, 0,
                                                                     0, a, 0, nullptr, 0);
      }
      timer_end(st);
    }
    return cudaGetLastError();
  }
  int mid = a + ((b - a) / 2 + NB - 1) / NB * NB;
  if (mid >= b) mid = a + NB;
  cudaError_t e = panel_factor(L, factors, thr, err, a, mid, st);
  if (e != cudaSuccess) return e;
  launch_panel_update(L, factors, mid, b, a, mid, st);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return panel_factor(L, factors, thr, err, mid, b, st);
}

// Levels with few, wide fronts: the pivot chain (diagonal blocks, their
// triangular solves, panel updates) is latency-bound, so the Schur update and
// the bulk of the panel updates run concurrently with it, one super-block of
// kLookaheadCols pivot columns at a time (right-looking, lookahead 1):
//   chain  (high priority): factor super-block j; update super-block j+1 by j
//   panel  (high priority): update the panel columns beyond j+1 by j
//   schur  (low priority) : S -= L21_j D_j L21_j^T
// Every entry is updated by the super-blocks in increasing order, as in the
// sequential path, so results are identical run to run.
static int lookahead_cols() {  // super-block width (TFB_LOOKAHEAD_COLS for tuning sweeps)
  static int v = 0;
  if (!v) {
    const char* e = getenv("TFB_LOOKAHEAD_COLS");
    v = e ? std::max(64, atoi(e) / 64 * 64) : 256;
  }
  return v;
}
#define kLookaheadCols lookahead_cols()
// Levels without a Schur block (the root) have only the chain and the panel
// updates: narrower super-blocks shorten the chain (TFB_LOOKAHEAD_ROOT_COLS).
static int lookahead_root_cols() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("TFB_LOOKAHEAD_ROOT_COLS");
    v = e ? std::max(64, atoi(e) / 64 * 64) : 128;  // measured best on the cfg5 root
  }
  return v;
}
static int lookahead_width(int max_upd) { return max_upd > 0 ? lookahead_cols() : lookahead_root_cols(); }
constexpr int kLookaheadMaxFronts = 64;  // measured: 32-64 fronts gain ~1% (cfg5 L18-L19)

struct LookaheadStreams {
  cudaStream_t chain = nullptr, panel = nullptr, schur = nullptr;
  cudaEvent_t start, chain_done, panel_done, schur_done;
};
// One set per device and per slice slot: slices of a level (front ranges,
// front_base > 0) factored concurrently on different streams get their own
// streams and events (slot = which eighth of the level the slice starts in).
static LookaheadStreams& lookahead_streams(const LevelArgs& L) {
  static LookaheadStreams all[64][8];
  int dev = 0;
  cudaGetDevice(&dev);
  const long long lf = std::max<long long>(L.level_fronts, 1);
  const int slot = (int)std::min<long long>(7, std::max<long long>(0, L.front_base * 8 / lf));
  LookaheadStreams& ls = all[dev & 63][slot];
  if (!ls.chain) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&ls.chain, cudaStreamNonBlocking, greatest);
    cudaStreamCreateWithPriority(&ls.panel, cudaStreamNonBlocking, greatest);
    cudaStreamCreateWithPriority(&ls.schur, cudaStreamNonBlocking, least);
    for (cudaEvent_t* ev : {&ls.start, &ls.chain_done, &ls.panel_done, &ls.schur_done})
      cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  }
  return ls;
}

static int schur_group() {  // TFB_SCHUR_GROUP (tuning)
  static int v = 0;
  if (!v) {
    const char* e = getenv("TFB_SCHUR_GROUP");
    v = e ? std::max(1, atoi(e)) : 1;
  }
  return v;
}

static bool chain_dataflow() {  // TFB_CHAIN_DATAFLOW: lookahead chains as dataflow launches
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFB_CHAIN_DATAFLOW");
    v = e ? atoi(e) : 0;
  }
  return v != 0;
}
static cudaError_t launch_dataflow(const LevelArgs& L, double* factors, double thr,
                                   unsigned long long* err, int* ws_flags, int cb0, int TC,
                                   int TR, bool coop, cudaStream_t st);

// Only the redundant-per-CTA diagonal-block kernels (large_block_kernel,
// single-front levels; the dataflow chains) leave the panel's diagonal
// blocks as assembled: the separate diagonal kernels (diag32 / diag64) write
// l and d into the panel themselves, so the finalize copy is skipped for them.
static bool need_finalize(long long level_fronts) {
  return level_fronts <= kFusedBlockMaxFronts || chain_dataflow();
}
static bool diag_blocks_need_finalize(const LevelArgs& L) { return need_finalize(L.level_fronts); }

static cudaError_t factor_lookahead(const LevelArgs& L, const double* child_upd, double* factors,
                                    double* upd_out, double thr, unsigned long long* err,
                                    int* ws_flags, cudaStream_t st) {
  LookaheadStreams& S = lookahead_streams(L);
  cudaEventRecord(S.start, st);  // after the assembly
  cudaStreamWaitEvent(S.chain, S.start, 0);
  cudaStreamWaitEvent(S.panel, S.start, 0);
  cudaStreamWaitEvent(S.schur, S.start, 0);
  const int W = lookahead_width(L.max_upd);
  const int nsb = (L.max_k + W - 1) / W;
  const bool schur = L.max_upd > 0;
  for (int j = 0; j < nsb; j++) {
    const int c0 = j * W, c1 = std::min(c0 + W, L.max_k);
    const int c2 = std::min(c1 + W, L.max_k);
    cudaError_t e;
    if (chain_dataflow() && L.max_upd > 0) {
      // the super-block's whole chain (diagonal blocks, sub-diagonal and row
      // tiles down to m) as one dataflow launch
      const int TC = (c1 - c0 + NB - 1) / NB, TR = (L.max_m - c0 + NB - 1) / NB;
      e = launch_dataflow(L, factors, thr, err, ws_flags, c0, TC, TR, false, S.chain);
    } else {
      e = panel_factor(L, factors, thr, err, c0, c1, S.chain);
    }
    if (e != cudaSuccess) return e;
    if (j + 1 < nsb) {
      // the panel stream's update by j-1 covers columns >= c1: it must land first
      if (j >= 1) cudaStreamWaitEvent(S.chain, S.panel_done, 0);
      launch_panel_update(L, factors, c1, c2, c0, c1, S.chain);
    }
    cudaEventRecord(S.chain_done, S.chain);
    if (j + 2 < nsb) {
      cudaStreamWaitEvent(S.panel, S.chain_done, 0);
      launch_panel_update(L, factors, c2, L.max_k, c0, c1, S.panel);
      cudaEventRecord(S.panel_done, S.panel);
    }
    // Schur chunks cover schur_group() super-blocks (fewer read-modify-write
    // passes over S); the first chunk also assembles S (children gathered in
    // its epilogue)
    if (schur && ((j + 1) % schur_group() == 0 || j + 1 == nsb)) {
      const int g0 = (j / schur_group()) * schur_group() * W;
      cudaStreamWaitEvent(S.schur, S.chain_done, 0);
      timer_begin(K_SCHUR, S.schur);
      launch_schur<GSchurA>(L, factors, upd_out, S.schur, g0, c1, g0 == 0 ? child_upd : nullptr);
      timer_end(S.schur);
    }
  }
  cudaEventRecord(S.chain_done, S.chain);
  cudaEventRecord(S.panel_done, S.panel);
  cudaEventRecord(S.schur_done, S.schur);
  cudaStreamWaitEvent(st, S.chain_done, 0);
  cudaStreamWaitEvent(st, S.panel_done, 0);
  cudaStreamWaitEvent(st, S.schur_done, 0);
  if (diag_blocks_need_finalize(L)) {
    dim3 g((unsigned)L.n_fronts, (unsigned)((L.max_k + NB - 1) / NB));
    timer_begin(K_FINALIZE, st);
    large_diag_finalize_kernel<<<g, 256, 0, st>>>(L, factors);
    timer_end(st);
  }
  return cudaGetLastError();
}

static bool root_dataflow() {  // TFB_ROOT_DATAFLOW=0 selects the lookahead path (A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFB_ROOT_DATAFLOW");
    v = e ? atoi(e) != 0 : 1;
  }
  return v != 0;
}

bool root_dataflow_level(const LevelArgs& L) {
  return L.max_upd == 0 && L.max_k > 0 && root_dataflow();
}

static inline long long flag_ints(long long nf, int TR, int TC) {
  return nf * TR * TC + 2 * nf * (TC + 1) + 1 + nf;
}
// Flag words the level's dataflow launches need (tf_level_factor_workspace).
long long level_factor_ws_ints(const LevelArgs& L) {
  const int T = (L.max_k + NB - 1) / NB;
  if (root_dataflow_level(L)) return flag_ints(L.n_fronts, T, T);
  const int W = lookahead_width(L.max_upd);
  if (chain_dataflow() && L.max_upd > 0 && L.max_k > W &&
      L.level_fronts <= kLookaheadMaxFronts)
    return flag_ints(L.n_fronts, (L.max_m + NB - 1) / NB, (W + NB - 1) / NB);
  return 0;
}

// ------------------------------------------------------------- root fronts
// Fronts without a Schur block (the root, m == k): one persistent launch that
// factors the front as a dataflow over its 64x64 lower tiles (i, l).
//   chain CTA (one per front): for every column l, takes the partial
//     diagonal tile A_ll - sum_{j<l-1}, applies column l-1 itself (it still
//     holds L_{l,l-1} and d_{l-1}), factors it (diag64_smem: l, d, inverse M_l)
//     and publishes it; then solves the sub-diagonal tile
//     L_{l+1,l} = A M_l^T D_l^-1 from its partial sum and publishes it.  The
//     pivot chain therefore never leaves one CTA's shared memory.
//   tile CTAs: the other tiles, dealt in column-major order from an atomic
//     counter (a tile only waits on tiles dealt before it or on the chain, so
//     the schedule cannot deadlock).  Tile (i, l) accumulates
//     sum_j L_ij D_j L_lj^T left-looking as the columns j are published
//     (flags, acquire/release); diagonal and sub-diagonal tiles hand their
//     partial sums (columns j < l-1 resp. j < l) to the chain through the
//     panel, the others solve themselves with the published M_l.
// Sums run in a fixed order: results are deterministic.
using GRoot = GemmCfg<64, 64, 16, 2>;
constexpr size_t kRootSmem = sizeof(double) * (3 * NB * DLD + 2 * NB);
static_assert(GRoot::smem <= kRootSmem, "GEMM staging fits the tile buffers");

__device__ __forceinline__ void root_wait(const int* flag) {
  while (ld_acquire_gpu(flag) == 0) __nanosleep(32);
  tfb_jitter((unsigned)(size_t)flag);
}
__device__ __forceinline__ void root_publish(int* flag) {  // after a CTA barrier
  if (threadIdx.x == 0) {
    __threadfence();
    st_release_gpu(flag, 1);
  }
}
__device__ __forceinline__ long long root_clock() {
  long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  return ns;
}

// acc (4x2 warps of 16x32, DMMA fragments) = sum_t A[r][t] * s_t * B[c][t], t < 64,
// A and B in shared memory with row stride DLD (s == nullptr: s_t = 1)
__device__ __forceinline__ void root_tile_product(double (&acc)[GRoot::MI][GRoot::NJ][2],
                                                  double (*A)[DLD], double (*B)[DLD],
                                                  const double* sc) {
  constexpr int MI = GRoot::MI, NJ = GRoot::NJ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wy = warp / GRoot::WC, wx = warp % GRoot::WC, g8 = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int a = 0; a < MI; a++)
#pragma unroll
    for (int b = 0; b < NJ; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
  for (int ks = 0; ks < NB; ks += 4) {
    const double s = sc ? sc[ks + tq] : 1.0;
    double af[MI], bf[NJ];
#pragma unroll
    for (int a = 0; a < MI; a++) af[a] = A[wy * GRoot::WM + a * 8 + g8][ks + tq] * s;
#pragma unroll
    for (int b = 0; b < NJ; b++) bf[b] = B[wx * GRoot::WN + b * 8 + g8][ks + tq];
#pragma unroll
    for (int a = 0; a < MI; a++)
#pragma unroll
      for (int b = 0; b < NJ; b++) dmma884(acc[a][b], af[a], bf[b]);
  }
}

// D[r][c] -= sum_t S[r][t] s_t S[c][t] for c <= r < kb: the 36 lower 8x8
// tiles dealt to the 8 warps (balanced), DMMA over t < 64.
__device__ __forceinline__ void root_syrk_lower(double (*D)[DLD], double (*S)[DLD],
                                                const double* sc, int kb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g8 = lane >> 2, tq = lane & 3;
  constexpr int Q = 5;  // ceil(36 / 8)
  double acc[Q][2];
  int I[Q], J[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int tile = min(warp + 8 * q, 35);
    I[q] = tri_row32(tile);
    J[q] = tile - tri32(I[q], 0);
    acc[q][0] = acc[q][1] = 0.0;
  }
#pragma unroll 4
  for (int ks = 0; ks < NB; ks += 4) {
    const double s = sc[ks + tq];
#pragma unroll
    for (int q = 0; q < Q; q++)
      if (warp + 8 * q < 36)
        dmma884(acc[q], S[8 * I[q] + g8][ks + tq] * s, S[8 * J[q] + g8][ks + tq]);
  }
#pragma unroll
  for (int q = 0; q < Q; q++) {
    if (warp + 8 * q >= 36) continue;
    const int r = 8 * I[q] + g8;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int c = 8 * J[q] + 2 * tq + h;
      if (r < kb && c <= r) D[r][c] -= acc[q][h];
    }
  }
}

// x = S M^T for unit-lower M (only t <= n contributes to column n): warp w
// owns rows 8w..8w+7 and all eight column blocks (balanced, 72 DMMAs each).
// Fragment x[cb][h] is entry (8w + lane/4, 8cb + 2(lane%4) + h).
__device__ __forceinline__ void root_trsm_rows(double (&x)[8][2], double (*S)[DLD],
                                               double (*M)[DLD]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g8 = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int cb = 0; cb < 8; cb++) x[cb][0] = x[cb][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < NB; ks += 4) {
    const double a = S[8 * warp + g8][ks + tq];
#pragma unroll
    for (int cb = 0; cb < 8; cb++)
      if (ks < 8 * cb + 8) dmma884(x[cb], a, M[8 * cb + g8][ks + tq]);
  }
}

// The pivot chain of front f (one CTA).
__device__ void root_chain(const LevelArgs& L, double* factors, double threshold,
                           unsigned long long* err, long long f, int cb0, int TC, int* done,
                           const int* part_diag, const int* part_sub, long long* trace) {
  extern __shared__ __align__(16) double rsm[];
  __shared__ int s_ready;
  double(*D)[DLD] = reinterpret_cast<double(*)[DLD]>(rsm);
  double(*Mi)[DLD] = reinterpret_cast<double(*)[DLD]>(rsm + NB * DLD);
  double(*S)[DLD] = reinterpret_cast<double(*)[DLD]>(rsm + 2 * NB * DLD);
  double* dv = rsm + 3 * NB * DLD;
  double* dprev = dv + NB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g8 = lane >> 2, tq = lane & 3;
  const Shape s = front_shape(L, f);
  const int k = s.k, kp = s.kp, m = s.m;
  const int kend = min(k, cb0 + TC * NB);  // this launch's pivot columns [cb0, kend)
  double* Pf = factors + f * L.fac_stride;
  double* dvec = Pf + (long long)s.m * kp;
  // rows [row0, row0 + nr) x columns [col0, col0 + nc) of the panel into X
  // (asynchronous, zeros outside)
  auto load_tile = [&](double(*X)[DLD], int row0, int nr, int col0, int nc) {
    for (int e = tid; e < NB * NB; e += 256) {
      const int a = e >> 6, b = e & 63;
      const bool v = a < nr && b < nc;
      cp_async8(&X[a][b], v ? Pf + (long long)(row0 + a) * kp + col0 + b : Pf, v);
    }
    cp_async_commit();
  };
  // non-blocking probe of a flag, broadcast to the CTA (the caller syncs)
  auto probe = [&](const int* flag, bool want) {
    if (tid == 0) s_ready = want ? ld_acquire_gpu(flag) : 0;
  };
  bool d_pref = false;
  for (int l = 0; l < TC; l++) {
    const int c0 = cb0 + l * NB, kb = min(NB, kend - c0);
    if (kb <= 0) break;
    const int r0 = c0 + NB, nA = min(NB, m - r0);  // sub-diagonal tile rows
    const int kn = min(NB, kend - r0);             // next diagonal block (<= 0: none)
    if (!d_pref) {
      if (tid == 0) root_wait(part_diag + l);
      __syncthreads();
      load_tile(D, c0, kb, c0, kb);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (trace && tid == 0) trace[l * 8 + 0] = root_clock();
    for (int e = tid; e < NB * NB; e += 256) {  // unit rows / zeros outside the lower part
      const int a = e >> 6, b = e & 63;
      if (!(a < kb && b <= a)) D[a][b] = a == b ? 1.0 : 0.0;
    }
    __syncthreads();
    if (l > 0) root_syrk_lower(D, S, dprev, kb);  // column l-1: D -= L_{l,l-1} D_{l-1} L^T
    probe(part_sub + l + 1, nA > 0);
    __syncthreads();
    const bool s_pref = s_ready != 0;
    if (s_pref) load_tile(S, r0, nA, c0, kb);  // overlaps the diagonal factorization
    diag64_smem<256>(D, Mi, dv, kb);
    if (trace && tid == 0) trace[l * 8 + 1] = root_clock();
    if (nA > 0) {
      // sub-diagonal tile: L_{l+1,l} = A M_l^T D_l^-1, kept in S for column l+1
      if (!s_pref) {
        if (tid == 0) root_wait(part_sub + l + 1);
        __syncthreads();
        load_tile(S, r0, nA, c0, kb);
      }
      if (tid < NB) dprev[tid] = rcp_nr(dv[tid]);
      cp_async_wait<0>();
      __syncthreads();
      double x[8][2];
      root_trsm_rows(x, S, Mi);
      __syncthreads();  // every read of S precedes its overwrite
      const int rl = 8 * warp + g8;
#pragma unroll
      for (int cb = 0; cb < 8; cb++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int cl = 8 * cb + 2 * tq + h;
          const bool in = rl < nA && cl < kb;
          const double v = in ? x[cb][h] * dprev[cl] : 0.0;  // dprev holds 1/d here
          S[rl][cl] = v;
          if (in) Pf[(long long)(r0 + rl) * kp + c0 + cl] = v;
        }
      __syncthreads();  // every 1/d read
      if (tid < NB) dprev[tid] = dv[tid];
      __syncthreads();
      root_publish(done + (l + 1) * TC + l);
      if (trace && tid == 0) trace[l * 8 + 2] = root_clock();
    }
    // d and the aux block (M_l for the other tiles' solves), then the panel
    write_aux64<256>(L.aux + f * L.aux_stride + (long long)(c0 / NB) * NB * NB, D, Mi, dv, kb);
    for (int c = tid; c < kb; c += 256) {
      dvec[c0 + c] = dv[c];
      if (fabs(dv[c]) <= threshold)
        record_zero_pivot(err, (unsigned long long)(L.piv_off[f] + c0 + c));
    }
    __syncthreads();
    root_publish(done + l * TC + l);
    for (int e = tid; e < NB * NB; e += 256) {
      const int a = e >> 6, b = e & 63;
      if (a < kb && b <= a) Pf[(long long)(c0 + a) * kp + c0 + b] = D[a][b];
    }
    if (trace && tid == 0) trace[l * 8 + 3] = root_clock();
    // prefetch the next partial diagonal tile when it is ready
    probe(part_diag + l + 1, kn > 0);
    __syncthreads();  // also: D fully read
    d_pref = s_ready != 0;
    if (d_pref) load_tile(D, r0, kn, r0, kn);
  }
}

// flags of one launch over column blocks [cb0/64, cb0/64 + TC) and row blocks
// [cb0/64, cb0/64 + TR): done[nf][TR][TC], part_diag[nf][TC+1],
// part_sub[nf][TC+1], counter, chain_sm[nf]
inline long long chain_flag_ints(long long nf, int TR, int TC) {
  return nf * TR * TC + 2 * nf * (TC + 1) + 1 + nf;
}

__global__ void __launch_bounds__(256, 2) large_root_kernel(LevelArgs L, double* factors,
                                                         double threshold,
                                                         unsigned long long* err, int* flags,
                                                         int cb0, int TC, int TR,
                                                         long long* trace) {
  constexpr int BK = GRoot::BK, ST = GRoot::ST, LD = GRoot::LD, MI = GRoot::MI, NJ = GRoot::NJ;
  extern __shared__ __align__(16) double rsm[];
  __shared__ int s_tile;
  const int nf = L.n_fronts;
  int* done = flags;                                     // [nf][TR][TC] final tiles
  int* part_diag = done + (long long)nf * TR * TC;       // [nf][TC+1] partial diagonal tiles
  int* part_sub = part_diag + (long long)nf * (TC + 1);  // [nf][TC+1] partial sub-diagonal
  int* counter = part_sub + (long long)nf * (TC + 1);
  int* chain_sm = counter + 1;  // [nf] SM of each chain CTA, + 1 (0: not yet known)
  if (blockIdx.x < (unsigned)nf) {
    if (threadIdx.x == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      st_release_gpu(chain_sm + blockIdx.x, (int)sm + 1);
    }
    root_chain(L, factors, threshold, err, blockIdx.x, cb0, TC,
               done + (long long)blockIdx.x * TR * TC, part_diag + (long long)blockIdx.x * (TC + 1),
               part_sub + (long long)blockIdx.x * (TC + 1), blockIdx.x == 0 ? trace : nullptr);
    return;
  }
  double* As = rsm;  // GEMM staging [ST][64][LD], [ST][64][LD], [ST][BK]
  double* Bs = As + ST * NB * LD;
  double* Ds = Bs + ST * NB * LD;
  double(*D)[DLD] = reinterpret_cast<double(*)[DLD]>(rsm);             // tile
  double(*Mi)[DLD] = reinterpret_cast<double(*)[DLD]>(rsm + NB * DLD);  // M_l
  double* dv = rsm + 2 * NB * DLD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp / GRoot::WC, wx = warp % GRoot::WC, g8 = lane >> 2, tq = lane & 3;
  const long long ntiles = ((long long)TC * TR - (long long)TC * (TC - 1) / 2) * nf;
  // tile CTAs leave the chain CTAs' SMs to them (the chain is the critical path)
  if (tid == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    int mine = 0;
    for (int c = 0; c < nf; c++) {
      int v;
      while ((v = ld_acquire_gpu(chain_sm + c)) == 0) __nanosleep(32);
      mine |= v == (int)sm + 1;
    }
    s_tile = mine;
  }
  __syncthreads();
  if (s_tile) return;
  for (;;) {
    __syncthreads();  // shared memory is reused tile to tile
    if (tid == 0) s_tile = atomicAdd(counter, 1);
    __syncthreads();
    const long long t = s_tile;
    if (t >= ntiles) return;
    if (tid == 0) tfb_jitter((unsigned)t);
    const long long f = t % nf;
    long long rr = t / nf;
    int l = 0;
    while (rr >= TR - l) rr -= TR - l++;
    const int i = l + (int)rr;
    const Shape s = front_shape(L, f);
    const int k = s.k, kp = s.kp, m = s.m;
    const int kend = min(k, cb0 + TC * NB);
    const int r0 = cb0 + i * NB, c0 = cb0 + l * NB;
    if (r0 >= m || c0 >= kend) continue;  // beyond this front (smaller than the level's largest)
    const int nA = min(NB, m - r0), nB = min(NB, kend - c0);
    double* Pf = factors + f * L.fac_stride;
    const double* dvec = Pf + (long long)s.m * kp;
    int* fl = done + f * TR * TC;
    // the chain applies the last column to the diagonal tile itself
    const int ncols = i == l ? max(l - 1, 0) : l;
    const int nk = ncols * (NB / BK);

    auto issue = [&](int it) {
      const int stage = it % ST, kt = it * BK;
      double* as = As + stage * NB * LD;
      double* bs = Bs + stage * NB * LD;
      constexpr int CPR = BK / 2;
#pragma unroll
      for (int q = 0; q < (NB * CPR) / 256; q++) {
        const int ch = tid + q * 256, r = ch / CPR, cc = (ch % CPR) * 2;
        const bool va = r < nA, vb = r < nB;
        cp_async16(as + r * LD + cc, va ? Pf + (long long)(r0 + r) * kp + cb0 + kt + cc : Pf, va);
        cp_async16(bs + r * LD + cc, vb ? Pf + (long long)(c0 + r) * kp + cb0 + kt + cc : Pf, vb);
      }
      if (tid < CPR) cp_async16(Ds + stage * BK + tid * 2, dvec + cb0 + kt + tid * 2, true);
    };
    // column j of the product is ready once tiles (i, j) and (l, j) are final
    auto wait_col = [&](int it) {
      if (tid == 0 && (it % (NB / BK)) == 0) {
        const int j = it / (NB / BK);
        root_wait(fl + i * TC + j);
        if (i != l) root_wait(fl + l * TC + j);
      }
    };

    double acc[MI][NJ][2];
#pragma unroll
    for (int a = 0; a < MI; a++)
#pragma unroll
      for (int b = 0; b < NJ; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    if (nk > 0) {
      wait_col(0);
      __syncthreads();
      issue(0);
    }
    cp_async_commit();
    for (int it = 0; it < nk; it++) {
      if (it + 1 < nk) wait_col(it + 1);
      cp_async_wait<0>();
      __syncthreads();
      if (it + 1 < nk) issue(it + 1);
      cp_async_commit();
      const int stage = it % ST;
      const double* as = As + stage * NB * LD + (wy * GRoot::WM + g8) * LD + tq;
      const double* bs = Bs + stage * NB * LD + (wx * GRoot::WN + g8) * LD + tq;
      const double* ds = Ds + stage * BK + tq;
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        const double dk = ds[ks];
        double af[MI], bf[NJ];
#pragma unroll
        for (int a = 0; a < MI; a++) af[a] = as[a * 8 * LD + ks] * dk;
#pragma unroll
        for (int b = 0; b < NJ; b++) bf[b] = bs[b * 8 * LD + ks];
#pragma unroll
        for (int a = 0; a < MI; a++)
#pragma unroll
          for (int b = 0; b < NJ; b++) dmma884(acc[a][b], af[a], bf[b]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // staging buffers become D / Mi

    if (i <= l + 1) {
      // partial sum for the chain: A - sum, in place
      if (nk > 0) {
#pragma unroll
        for (int a = 0; a < MI; a++)
#pragma unroll
          for (int b = 0; b < NJ; b++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int rl = wy * GRoot::WM + a * 8 + g8, cl = wx * GRoot::WN + b * 8 + 2 * tq + h;
              if (rl < nA && cl < nB && (i != l || cl <= rl))
                Pf[(long long)(r0 + rl) * kp + c0 + cl] -= acc[a][b][h];
            }
      }
      __syncthreads();
      root_publish(i == l ? part_diag + f * (TC + 1) + l : part_sub + f * (TC + 1) + i);
      continue;
    }
    // A = assembled tile - product, into D
#pragma unroll
    for (int a = 0; a < MI; a++)
#pragma unroll
      for (int b = 0; b < NJ; b++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int rl = wy * GRoot::WM + a * 8 + g8, cl = wx * GRoot::WN + b * 8 + 2 * tq + h;
          D[rl][cl] = (rl < nA && cl < nB) ? Pf[(long long)(r0 + rl) * kp + c0 + cl] - acc[a][b][h]
                                           : 0.0;
        }
    // L_il = A M_l^T D_l^-1 (M_l: strict lower part of the published aux block)
    if (tid == 0) root_wait(fl + l * TC + l);
    __syncthreads();
    const double* M = L.aux + f * L.aux_stride + (long long)(c0 / NB) * NB * NB;
    for (int e = tid; e < NB * NB; e += 256) {
      const int a = e >> 6, b = e & 63;
      Mi[a][b] = b < a ? M[e] : (b == a ? 1.0 : 0.0);
    }
    if (tid < NB) dv[tid] = tid < nB ? rcp_nr(dvec[c0 + tid]) : 1.0;
    __syncthreads();
    double x[MI][NJ][2];
    root_tile_product(x, D, Mi, nullptr);
#pragma unroll
    for (int a = 0; a < MI; a++)
#pragma unroll
      for (int b = 0; b < NJ; b++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int rl = wy * GRoot::WM + a * 8 + g8, cl = wx * GRoot::WN + b * 8 + 2 * tq + h;
          if (rl < nA && cl < nB) Pf[(long long)(r0 + rl) * kp + c0 + cl] = x[a][b][h] * dv[cl];
        }
    __syncthreads();
    root_publish(fl + i * TC + l);
  }
}

static int* root_flags(long long ints) {  // per-device scratch, grown on demand
  static int* buf[64] = {};
  static long long cap[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (cap[dev] < ints) {
    if (buf[dev]) cudaFree(buf[dev]);
    buf[dev] = nullptr;
    cap[dev] = 0;
    if (cudaMalloc(&buf[dev], sizeof(int) * ints) != cudaSuccess) return nullptr;
    cap[dev] = ints;
  }
  return buf[dev];
}

static cudaError_t launch_dataflow(const LevelArgs& L, double* factors, double thr,
                                   unsigned long long* err, int* ws_flags, int cb0, int TC,
                                   int TR, bool coop, cudaStream_t st);

static cudaError_t factor_root(const LevelArgs& L, double* factors, double thr,
                               unsigned long long* err, int* ws_flags, cudaStream_t st) {
  const int T = (L.max_k + NB - 1) / NB;
  return launch_dataflow(L, factors, thr, err, ws_flags, 0, T, T, true, st);
}

// The pivot columns [cb0, cb0 + 64 TC) of every front of a level as one
// dataflow launch (root kernel): one chain CTA per front factors the diagonal
// blocks and their sub-diagonal tiles; tile CTAs take the other panel tiles
// (rows down to m) left-looking over the launch's own columns.  Lookahead
// super-blocks use it with the columns before cb0 already applied.
static cudaError_t launch_dataflow(const LevelArgs& L, double* factors, double thr,
                                   unsigned long long* err, int* ws_flags, int cb0, int TC,
                                   int TR, bool coop, cudaStream_t st) {
  const int T = TC;
  const long long nf = L.n_fronts;
  const long long nflags = chain_flag_ints(nf, TR, TC);
  // the caller's workspace (one per DevicePlan level), else a per-device scratch
  int* flags = ws_flags ? ws_flags : root_flags(nflags);
  if (!flags) return cudaErrorMemoryAllocation;
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * nflags, st);
  if (e != cudaSuccess) return e;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(large_root_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kRootSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, large_root_kernel, 256, kRootSmem);
    occ = std::max(occ, 1);
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // chain CTAs + tile CTAs, all co-resident (tile CTAs wait on the chain)
  const long long ntiles = nf * ((long long)TC * TR - (long long)TC * (TC - 1) / 2);
  const long long cap = (long long)sms * occ;
  // tile CTAs that land next to a chain CTA exit: keep at least one other
  if (nf * occ + 1 > cap) return cudaErrorInvalidConfiguration;
  const unsigned grid = (unsigned)std::min(std::max(ntiles + nf, nf * occ + 1), cap);
  static long long* trace = nullptr;
  if (getenv("TFB_ROOT_TRACE") && !trace) {
    cudaMalloc(&trace, sizeof(long long) * 8 * 4096);
    cudaMemset(trace, 0, sizeof(long long) * 8 * 4096);
  }
  timer_begin(K_ROOT, st);
  if (coop) {
    e = launch_cooperative(large_root_kernel, dim3(grid), dim3(256), kRootSmem, st, L, factors,
                           thr, err, flags, cb0, TC, TR, trace);
  } else {
    // concurrent with the lookahead Schur stream: a cooperative grid would wait
    // for the whole grid's worth of free slots.  Progress without co-residency:
    // the chain CTAs are the lowest block indices (dispatched first) and a tile
    // CTA only waits on the chain or on tiles dealt before it.
    large_root_kernel<<<grid, 256, kRootSmem, st>>>(L, factors, thr, err, flags, cb0, TC, TR,
                                                     trace);
    e = cudaGetLastError();
  }
  timer_end(st);
  if (e != cudaSuccess) return e;
  if (trace && T <= 4096) {
    static std::vector<long long> h;
    h.resize(8 * T);
    cudaMemcpyAsync(h.data(), trace, sizeof(long long) * 8 * T, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const long long t0 = h[0];
    for (int l = 0; l < T; l++)
      fprintf(stderr, "col %3d ready %8.1f diag %8.1f sub pub %8.1f diag pub %8.1f us\n", l,
              (h[8 * l] - t0) * 1e-3, (h[8 * l + 1] - t0) * 1e-3, (h[8 * l + 2] - t0) * 1e-3,
              (h[8 * l + 3] - t0) * 1e-3);
  }
  return cudaGetLastError();
}

cudaError_t launch_factor_large(const LevelArgs& L, const double* child_upd, double* factors,
                                double* upd_out, double thr, unsigned long long* err, int* ws_flags,
                                cudaStream_t st) {
  if (L.is_leaf) return cudaErrorInvalidValue;  // element fronts are never this large
  if (L.max_k > 0 && (!L.aux || L.aux_stride < large_aux_doubles(L.max_k)))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(large_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBlockSmem);
    cudaFuncSetAttribute(large_diag64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kDiagSmem);
    attr = true;
  }
  const bool lookahead =
      L.max_k > lookahead_width(L.max_upd) && L.level_fronts <= kLookaheadMaxFronts;
  // S is assembled by the (first) Schur kernel's epilogue unless the level
  // has no pivots
  const bool fused_s = L.max_k > 0 && L.max_upd > 0;
  {
    // ~kAsmRowsPerWarp rows per warp, but at least ~8 CTAs per SM on levels
    // with few (large) fronts, down to one row per warp
    const long long by_rows = (L.max_m + kAsmWarps * kAsmRowsPerWarp - 1) / (kAsmWarps * kAsmRowsPerWarp);
    const long long by_sms = (148LL * 8 + L.n_fronts - 1) / L.n_fronts;
    const long long cap = (L.max_m + kAsmWarps - 1) / kAsmWarps;
    const unsigned gy = (unsigned)std::max(1LL, std::min(std::max(by_rows, by_sms), cap));
    timer_begin(K_ASSEMBLE, st);
    large_assemble_kernel<<<dim3(L.n_fronts, gy), 32 * kAsmWarps, 0, st>>>(
        L, child_upd, factors, upd_out, fused_s ? 0 : 1);
    timer_end(st);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (L.max_upd == 0 && L.max_k > 0 && root_dataflow())
    return factor_root(L, factors, thr, err, ws_flags, st);
  if (lookahead) return factor_lookahead(L, child_upd, factors, upd_out, thr, err, ws_flags, st);
  if (L.max_k > 0) {
    e = panel_factor(L, factors, thr, err, 0, L.max_k, st);
    if (e != cudaSuccess) return e;
  }
  if (fused_s) {
    timer_begin(K_SCHUR, st);
    launch_schur<GSchurA>(L, factors, upd_out, st, 0, 0, child_upd);
    timer_end(st);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (L.max_k > 0 && diag_blocks_need_finalize(L)) {
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

// Kernel launches of one launch_factor_large call (tf_level_launch_count).
int large_level_launches(int max_k, int max_upd, long long level_fronts) {
  const int fronts = (int)std::min<long long>(level_fronts, 1 << 30);
  if (max_upd == 0 && max_k > 0 && root_dataflow()) return 2;  // assembly, root kernel
  const int W = lookahead_width(max_upd);
  if (max_k > W && level_fronts <= kLookaheadMaxFronts) {
    const int nsb = (max_k + W - 1) / W;
    int n = 1 + (need_finalize(level_fronts) ? 1 : 0);  // assembly, finalize
    for (int j = 0; j < nsb; j++) {
      const int c0 = j * W, c1 = std::min(c0 + W, max_k);
      n += large_panel_launches(c1 - c0, fronts) + (j + 1 < nsb) + (j + 2 < nsb) +
           (max_upd > 0 && ((j + 1) % schur_group() == 0 || j + 1 == nsb));
    }
    return n;
  }
  return 1 + large_panel_launches(max_k, fronts) + (max_k > 0 && max_upd > 0 ? 1 : 0) +
         (max_k > 0 && need_finalize(level_fronts) ? 1 : 0);
}

cudaError_t set_jitter_factor(unsigned seed) { return set_jitter_tu(seed); }

}  // namespace tfb
