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
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "front_small.cuh"

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

// Row/column split of a flat index over nr columns: a shift when nr is a
// power of two (the dispatcher slices columns that way), else a division.
#define TFB_DIV_SETUP(nr_) \
  const bool div_p2 = ((nr_) & ((nr_)-1)) == 0; \
  const int div_lg = 31 - __clz(nr_)
#define TFB_DIV(e_) (div_p2 ? ((e_) >> div_lg) : ((e_) / nr))

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
__device__ __forceinline__ void solve_fwd_small_front(
    long long f, const LevelArgs& L, const LevelArgs& C, const double* __restrict__ factors,
    const double* __restrict__ w_child, long long child_rows, int child_at0,
    double* __restrict__ w_out, long long out_rows, double* __restrict__ y, int nr, int ldr,
    int col0, int smem_per_group, unsigned char* smem_raw) {
  if (!STAGE) nr = 1;  // one-column instantiation: index math folds
  TFB_DIV_SETUP(nr);
  const int gid = threadIdx.x / G, t = threadIdx.x - gid * G, bar = 1 + gid;
  if (L.upd_is_zero(f)) return;  // pivot-free subtree: zero update, not written (parent skips it)
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
    const int r = TFB_DIV(e), j = e - r * nr;
    W[e] = e < nK ? y[(piv + r) * ldr + col0 + j] : 0.0;
  }
  group_sync<G>(bar);
  if (!L.is_leaf) {
    for (int c = 0; c < s.nsrc; c++) {
      const long long ch = 2 * (L.front_base + f) + c - C.front_base;
      const int ck = C.pat[(size_t)C.pattern_of[ch] * TF_PAT_WIDTH + TF_PAT_K];
      if (C.upd_is_zero(ch)) continue;  // pivot-free child subtree: zero update, never written
      const int off = child_at0 ? 0 : ck;
      const int len = c == 0 ? s.len0 : s.len1;
      const int* mp = L.maps + (c == 0 ? s.off0 : s.off1);
      const double* Wc = w_child + (ch * child_rows + off) * ldr + col0;
      const int n = len * nr;
      if (C.upd_implicit(ch)) {
        // the child stored its k unscaled pivot rows w_piv (rows [0, ck)):
        // its update row a is -sum_q l(ck+a, q) w_piv[q], summed here in the
        // child's own order (bitwise what it would have written)
        const int* CP = C.pat + (size_t)C.pattern_of[ch] * TF_PAT_WIDTH;
        const int ckp = CP[TF_PAT_KP];
        const double* Pc = C.factors + ch * C.fac_stride + (long long)ck * ckp;
        const double* Wp = w_child + ch * child_rows * ldr + col0;
        for (int e = t; e < n; e += G) {
          const int a = TFB_DIV(e), j = e - a * nr;
          double acc = 0.0;
          for (int q = 0; q < ck; q++) acc -= __ldg(Pc + (long long)a * ckp + q) * Wp[(long long)q * ldr + j];
          W[__ldg(mp + a) * nr + j] += acc;
        }
        group_sync<G>(bar);
        continue;
      }
      int e = t;
      for (; e + 3 * G < n; e += 4 * G) {  // four entries in flight per thread
        int p[4];
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int eq = e + q * G, a = TFB_DIV(eq), j = eq - a * nr;
          p[q] = __ldg(mp + a) * nr + j;
          v[q] = Wc[(long long)a * ldr + j];
        }
#pragma unroll
        for (int q = 0; q < 4; q++) W[p[q]] += v[q];
      }
      for (; e < n; e += G) {
        const int a = TFB_DIV(e), j = e - a * nr;
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
      const int q = TFB_DIV(e), r = c + 1 + q, j = e - q * nr;
      W[r * nr + j] -= Lp(r, c) * Wc[j];
    }
    group_sync<G>(bar);
  }
  for (int e = t; e < nK; e += G) {
    const int r = TFB_DIV(e), j = e - r * nr;
    y[(piv + r) * ldr + col0 + j] = W[e] / dv[r];
  }
  // update rows: w_r - l_r . w_piv (row-contiguous panel reads), straight out
  double* out = w_out + f * out_rows * ldr + col0;
  if (L.upd_implicit(f)) {  // the parent forms -L21 w_piv itself: store w_piv only
    for (int e = t; e < nK; e += G) {
      const int r = TFB_DIV(e), j = e - r * nr;
      out[(long long)r * ldr + j] = W[e];
    }
    return;
  }
  if (!STAGE && k > 4) {
    // one column, rows wider than a sector: a thread's whole row is requested
    // in bursts of 8 entries (every sector of the row in flight together)
    for (int r = k + t; r < m; r += G) {
      const double* lr = Pg + (long long)r * kp;
      double acc = W[r];
      for (int c0 = 0; c0 < k; c0 += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = c0 + q < k ? __ldg(lr + c0 + q) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; q++) acc -= v[q] * W[min(c0 + q, k - 1)];
      }
      out[r - k] = acc;
    }
    return;
  }
  if (!STAGE) {
    // one column, k <= 4: up to four update rows per thread with all their
    // panel loads issued before any store
    for (int r0 = k + t; r0 < m; r0 += 4 * G) {
      double l[4][4];
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int c = 0; c < 4; c++)
          l[q][c] = (r0 + q * G < m && c < k) ? __ldg(Pg + (long long)(r0 + q * G) * kp + c) : 0.0;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int r = r0 + q * G;
        if (r >= m) break;
        double acc = W[r];
#pragma unroll
        for (int c = 0; c < 4; c++)
          if (c < k) acc -= l[q][c] * W[c];
        out[r - k] = acc;
      }
    }
    return;
  }
  for (int e = nK + t; e < nW; e += G) {
    const int r = TFB_DIV(e), j = e - r * nr;
    double acc = W[e];
    for (int c = 0; c < k; c++) acc -= Lp(r, c) * W[c * nr + j];
    out[(long long)(r - k) * ldr + j] = acc;
  }
}

template <int G, int GPC, bool STAGE>
__device__ __forceinline__ void solve_bwd_small_front(
    long long f, const LevelArgs& L, const LevelArgs& PA, int has_parent,
    const double* __restrict__ factors, const double* __restrict__ x_parent,
    long long parent_rows, double* __restrict__ x_out, long long out_rows,
    double* __restrict__ y, int nr, int ldr, int col0, int smem_per_group,
    unsigned char* smem_raw) {
  if (!STAGE) nr = 1;  // one-column instantiation: index math folds
  TFB_DIV_SETUP(nr);
  const int gid = threadIdx.x / G, t = threadIdx.x - gid * G, bar = 1 + gid;
  if (L.upd_is_zero(f)) return;  // pivot-free subtree: nothing to solve, no children to serve
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
    const int r = TFB_DIV(e), j = e - r * nr;
    X[e] = y[(piv + r) * ldr + col0 + j];
  }
  if (has_parent && m > k) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int c = (int)((L.front_base + f) & 1);
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    const int* mp = PA.maps + (c == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    const double* Xp = x_parent + pf * parent_rows * ldr + col0;
    int e = nK + t;
    for (; e + 3 * G < nW; e += 4 * G) {  // four entries in flight per thread
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int eq = e + q * G - nK, a = TFB_DIV(eq), j = eq - a * nr;
        v[q] = Xp[(long long)__ldg(mp + a) * ldr + j];
      }
#pragma unroll
      for (int q = 0; q < 4; q++) X[e + q * G] = v[q];
    }
    for (; e < nW; e += G) {
      const int a = TFB_DIV(e - nK), j = (e - nK) - a * nr;
      X[e] = Xp[(long long)mp[a] * ldr + j];
    }
  }
  group_sync<G>(bar);
  if (m > k && !STAGE && k > G) {
    // one column: thread t owns columns t + qG, so a row's entries are all
    // requested in the same iteration (each sector fetched once)
    for (int cb = t; cb < k; cb += 4 * G) {
      double acc[4];
#pragma unroll
      for (int q = 0; q < 4; q++) acc[q] = cb + q * G < k ? X[cb + q * G] : 0.0;
      for (int r = k; r < m; r++) {
        const double xr = X[r];
        const double* lr = Pg + (long long)r * kp;
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (cb + q * G < k) acc[q] -= __ldg(lr + cb + q * G) * xr;
      }
#pragma unroll
      for (int q = 0; q < 4; q++)
        if (cb + q * G < k) X[cb + q * G] = acc[q];
    }
    group_sync<G>(bar);
  } else if (m > k) {
    for (int e = t; e < nK; e += G) {
      const int c = TFB_DIV(e), j = e - c * nr;
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
      const int r = TFB_DIV(e), j = e - r * nr;
      X[e] -= Lp(c, r) * Xc[j];
    }
    group_sync<G>(bar);
  }
  for (int e = t; e < nK; e += G) {
    const int r = TFB_DIV(e), j = e - r * nr;
    y[(piv + r) * ldr + col0 + j] = X[e];
  }
  if (!L.is_leaf && !L.children_idle(f)) {  // (children without pivots never read it)
    double* out = x_out + f * out_rows * ldr + col0;
    for (int e = t; e < nW; e += G) {
      const int r = TFB_DIV(e), j = e - r * nr;
      out[(long long)r * ldr + j] = X[e];
    }
  }
}

// Small-front sweep kernels: one thread group per front, grid-stride (leaf
// levels, whose fronts are nearly all pivot-free and return at once, run on
// a few resident waves of CTAs; the group-local syncs never span fronts).
template <int G, int GPC, bool STAGE>
__global__ void __launch_bounds__(G* GPC)
    solve_fwd_small(LevelArgs L, LevelArgs C, const double* __restrict__ factors,
                    const double* __restrict__ w_child, long long child_rows, int child_at0,
                    double* __restrict__ w_out, long long out_rows, double* __restrict__ y,
                    int nr, int ldr, int col0, int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  for (long long f = (long long)blockIdx.x * GPC + threadIdx.x / G; f < L.n_fronts;
       f += (long long)gridDim.x * GPC)
    solve_fwd_small_front<G, GPC, STAGE>(f, L, C, factors, w_child, child_rows, child_at0, w_out,
                                         out_rows, y, nr, ldr, col0, smem_per_group, smem_raw);
}

template <int G, int GPC, bool STAGE>
__global__ void __launch_bounds__(G* GPC)
    solve_bwd_small(LevelArgs L, LevelArgs PA, int has_parent, const double* __restrict__ factors,
                    const double* __restrict__ x_parent, long long parent_rows,
                    double* __restrict__ x_out, long long out_rows, double* __restrict__ y,
                    int nr, int ldr, int col0, int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  for (long long f = (long long)blockIdx.x * GPC + threadIdx.x / G; f < L.n_fronts;
       f += (long long)gridDim.x * GPC)
    solve_bwd_small_front<G, GPC, STAGE>(f, L, PA, has_parent, factors, x_parent, parent_rows,
                                         x_out, out_rows, y, nr, ldr, col0, smem_per_group,
                                         smem_raw);
}

// Many right-hand sides on small levels: one warp per front, lane l owns
// columns col0 + l + 32j (j < CPL), and the front is processed in the GATHER
// form, so no vector block is materialised:
//   pivot rows  w_c = y_c + sum_children child[inv(c)]      (registers, c < k)
//               w_r -= l(r,c) w_c  for c < r < k            (forward elimination)
//               y_c = w_c / d_c
//   update rows u_{r-k} = sum_children child[inv(r)] - sum_c l(r,c) w_c   (streamed)
// Child rows come through the inverse extend-add maps (front row -> child
// update row); pivot-free child subtrees are skipped.  No shared memory, no
// index division, every vector access a coalesced 32*8-byte row segment;
// the update rows are streamed four at a time (all their loads in flight).
constexpr int kColsWarps = 8;
template <int KMAX, int CPL>
__global__ void __launch_bounds__(32 * kColsWarps)
    solve_fwd_cols(LevelArgs L, LevelArgs C, const double* __restrict__ factors,
                   const double* __restrict__ w_child, long long child_rows, int child_at0,
                   double* __restrict__ w_out, long long out_rows, double* __restrict__ y, int nr,
                   int ldr, int col0) {
  const int lane = threadIdx.x & 31;
  const long long f = (long long)blockIdx.x * kColsWarps + (threadIdx.x >> 5);
  if (f >= L.n_fronts || L.upd_is_zero(f)) return;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pg = factors + f * L.fac_stride;
  const int* inv0 = L.maps + s.ioff;
  const int* inv1 = inv0 + m;
  // child blocks (null: no such child or a pivot-free subtree)
  const double* Wc0 = nullptr;
  const double* Wc1 = nullptr;
  // implicit children: their update row a is -sum_q l(k+a, q) w_piv[q]
  const double* Pc0 = nullptr;
  const double* Pc1 = nullptr;
  int ck0 = 0, ck1 = 0, ckp0 = 0, ckp1 = 0;
  if (!L.is_leaf) {
    const long long ch0 = 2 * (L.front_base + f) - C.front_base;
    if (!C.upd_is_zero(ch0)) {
      const int* CP = C.pat + (size_t)C.pattern_of[ch0] * TF_PAT_WIDTH;
      const int ck = CP[TF_PAT_K];
      if (C.upd_implicit(ch0)) {
        Wc0 = w_child + ch0 * child_rows * ldr + col0;
        ck0 = ck;
        ckp0 = CP[TF_PAT_KP];
        Pc0 = C.factors + ch0 * C.fac_stride + (long long)ck * ckp0;
      } else {
        Wc0 = w_child + (ch0 * child_rows + (child_at0 ? 0 : ck)) * ldr + col0;
      }
    }
    if (s.nsrc == 2 && !C.upd_is_zero(ch0 + 1)) {
      const int* CP = C.pat + (size_t)C.pattern_of[ch0 + 1] * TF_PAT_WIDTH;
      const int ck = CP[TF_PAT_K];
      if (C.upd_implicit(ch0 + 1)) {
        Wc1 = w_child + (ch0 + 1) * child_rows * ldr + col0;
        ck1 = ck;
        ckp1 = CP[TF_PAT_KP];
        Pc1 = C.factors + (ch0 + 1) * C.fac_stride + (long long)ck * ckp1;
      } else {
        Wc1 = w_child + ((ch0 + 1) * child_rows + (child_at0 ? 0 : ck)) * ldr + col0;
      }
    }
  }
  bool cok[CPL];
#pragma unroll
  for (int j = 0; j < CPL; j++) cok[j] = lane + 32 * j < nr;
  auto child_sum = [&](int r, double (&v)[CPL]) {
    const int i0 = Wc0 ? __ldg(inv0 + r) : -1;
    const int i1 = Wc1 ? __ldg(inv1 + r) : -1;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const int col = lane + 32 * j;
      double a = 0.0, b = 0.0;
      if (i0 >= 0 && cok[j]) {
        if (Pc0) {
          for (int q = 0; q < ck0; q++)
            a -= __ldg(Pc0 + (long long)i0 * ckp0 + q) * Wc0[(long long)q * ldr + col];
        } else {
          a = Wc0[(long long)i0 * ldr + col];
        }
      }
      if (i1 >= 0 && cok[j]) {
        if (Pc1) {
          for (int q = 0; q < ck1; q++)
            b -= __ldg(Pc1 + (long long)i1 * ckp1 + q) * Wc1[(long long)q * ldr + col];
        } else {
          b = Wc1[(long long)i1 * ldr + col];
        }
      }
      v[j] = a + b;
    }
  };
  // pivot rows
  double w[KMAX][CPL];
#pragma unroll
  for (int c = 0; c < KMAX; c++) {
    if (c < k) {
      double v[CPL];
      child_sum(c, v);
#pragma unroll
      for (int j = 0; j < CPL; j++)
        w[c][j] = v[j] + (cok[j] ? y[(piv + c) * ldr + col0 + lane + 32 * j] : 0.0);
    } else {
#pragma unroll
      for (int j = 0; j < CPL; j++) w[c][j] = 0.0;
    }
  }
#pragma unroll
  for (int c = 0; c < KMAX; c++) {
#pragma unroll
    for (int r = c + 1; r < KMAX; r++) {
      if (r < k) {
        const double lrc = __ldg(Pg + (long long)r * kp + c);
#pragma unroll
        for (int j = 0; j < CPL; j++) w[r][j] -= lrc * w[c][j];
      }
    }
  }
  const double* dv = Pg + (long long)m * kp;
#pragma unroll
  for (int c = 0; c < KMAX; c++) {
    if (c < k) {
      const double dinv = 1.0 / __ldg(dv + c);
#pragma unroll
      for (int j = 0; j < CPL; j++)
        if (cok[j]) y[(piv + c) * ldr + col0 + lane + 32 * j] = w[c][j] * dinv;
    }
  }
  double* out = w_out + f * out_rows * ldr + col0;
  if (L.upd_implicit(f)) {  // the parent forms -L21 w_piv itself: store w_piv only
#pragma unroll
    for (int c = 0; c < KMAX; c++)
      if (c < k) {
#pragma unroll
        for (int j = 0; j < CPL; j++)
          if (cok[j]) out[(long long)c * ldr + lane + 32 * j] = w[c][j];
      }
    return;
  }
  // update rows, four at a time
  for (int r0 = k; r0 < m; r0 += 4) {
    double v[4][CPL];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      if (r0 + q < m) child_sum(r0 + q, v[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int r = r0 + q;
      if (r < m) {
      const double* lr = Pg + (long long)r * kp;
#pragma unroll
      for (int c = 0; c < KMAX; c++) {
        if (c < k) {
          const double l = __ldg(lr + c);
#pragma unroll
          for (int j = 0; j < CPL; j++) v[q][j] -= l * w[c][j];
        }
      }
#pragma unroll
      for (int j = 0; j < CPL; j++)
        if (cok[j]) out[(long long)(r - k) * ldr + lane + 32 * j] = v[q][j];
      }
    }
  }
}

// Backward counterpart, same layout (warp per front, lanes own columns):
//   x_r (r >= k) = parent block rows gathered through the parent's map
//   x_c = y_c - sum_{r>=k} l(r,c) x_r      (streamed over r, four rows at a time)
//   x_c -= l(c',c) x_c' for c' > c        (back substitution in registers)
//   y_c = x_c; the full block (m rows) goes to x_out for the children.
template <int KMAX, int CPL>
__global__ void __launch_bounds__(32 * kColsWarps)
    solve_bwd_cols(LevelArgs L, LevelArgs PA, int has_parent, const double* __restrict__ factors,
                   const double* __restrict__ x_parent, long long parent_rows,
                   double* __restrict__ x_out, long long out_rows, double* __restrict__ y, int nr,
                   int ldr, int col0) {
  const int lane = threadIdx.x & 31;
  const long long f = (long long)blockIdx.x * kColsWarps + (threadIdx.x >> 5);
  if (f >= L.n_fronts || L.upd_is_zero(f)) return;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pg = factors + f * L.fac_stride;
  bool cok[CPL];
#pragma unroll
  for (int j = 0; j < CPL; j++) cok[j] = lane + 32 * j < nr;
  const int* mp = nullptr;
  const double* Xp = nullptr;
  if (has_parent && m > k) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int c = (int)((L.front_base + f) & 1);
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    mp = PA.maps + (c == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    Xp = x_parent + pf * parent_rows * ldr + col0;
  }
  double x[KMAX][CPL];
#pragma unroll
  for (int c = 0; c < KMAX; c++)
#pragma unroll
    for (int j = 0; j < CPL; j++)
      x[c][j] = (c < k && cok[j]) ? y[(piv + c) * ldr + col0 + lane + 32 * j] : 0.0;
  double* out = (L.is_leaf || L.children_idle(f)) ? nullptr : x_out + f * out_rows * ldr + col0;
  if (mp) {
    for (int r0 = k; r0 < m; r0 += 4) {
      double v[4][CPL];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (r0 + q < m) {
          const long long pr = __ldg(mp + (r0 + q - k));
#pragma unroll
          for (int j = 0; j < CPL; j++) v[q][j] = cok[j] ? Xp[pr * ldr + lane + 32 * j] : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int r = r0 + q;
        if (r < m) {
          const double* lr = Pg + (long long)r * kp;
#pragma unroll
          for (int c = 0; c < KMAX; c++) {
            if (c < k) {
              const double l = __ldg(lr + c);
#pragma unroll
              for (int j = 0; j < CPL; j++) x[c][j] -= l * v[q][j];
            }
          }
          if (out) {
#pragma unroll
            for (int j = 0; j < CPL; j++)
              if (cok[j]) out[(long long)r * ldr + lane + 32 * j] = v[q][j];
          }
        }
      }
    }
  }
#pragma unroll
  for (int c = KMAX - 1; c > 0; c--) {
    if (c < k) {
#pragma unroll
      for (int r = 0; r < c; r++) {
        const double l = __ldg(Pg + (long long)c * kp + r);
#pragma unroll
        for (int j = 0; j < CPL; j++) x[r][j] -= l * x[c][j];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < KMAX; c++) {
    if (c < k) {
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        if (!cok[j]) continue;
        y[(piv + c) * ldr + col0 + lane + 32 * j] = x[c][j];
        if (out) out[(long long)c * ldr + lane + 32 * j] = x[c][j];
      }
    }
  }
}

// Selection: many columns on small levels with few pivots per front
// (TFB_COLS_SOLVE=0 disables, for A/B).
static bool cols_solve_fwd(const LevelArgs& L, int nrhs) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFB_COLS_SOLVE");
    v = e ? atoi(e) : 1;
  }
  // measured on cfg3 (64 RHS): faster for fronts of 12..27 rows with <= 4
  // pivots (L3-L5: 1.37 -> 0.94 ms fwd+bwd), slower for tiny fronts (L2) and
  // for k = 8..16 (L6-L9: register-resident pivot rows too long)
  return v != 0 && nrhs >= 16 && L.max_k <= 4 && L.max_m >= 12 &&
         !level_is_large(L.is_leaf, L.max_m);
}

static cudaError_t launch_bwd_cols(const LevelArgs& L, const LevelArgs& PA, int has_parent,
                                   const double* factors, const double* x_parent,
                                   long long parent_rows, double* x_out, long long out_rows,
                                   double* y, int nrhs, cudaStream_t st) {
  const unsigned g = (unsigned)((L.n_fronts + kColsWarps - 1) / kColsWarps);
  timer_begin(K_SOLVE_SMALL_BWD, st);
  for (int col0 = 0; col0 < nrhs; col0 += 64) {
    const int nr = std::min(64, nrhs - col0);
    const bool two = nr > 32;
#define TFB_COLS(K, P)                                                                        \
  solve_bwd_cols<K, P><<<g, 32 * kColsWarps, 0, st>>>(L, PA, has_parent, factors, x_parent,     \
                                                     parent_rows, x_out, out_rows, y, nr, nrhs, \
                                                     col0)
    if (L.max_k <= 4) { if (two) TFB_COLS(4, 2); else TFB_COLS(4, 1); }
    else if (L.max_k <= 8) { if (two) TFB_COLS(8, 2); else TFB_COLS(8, 1); }
    else { if (two) TFB_COLS(16, 2); else TFB_COLS(16, 1); }
#undef TFB_COLS
  }
  timer_end(st);
  return cudaGetLastError();
}

static cudaError_t launch_fwd_cols(const LevelArgs& L, const LevelArgs& O, int flag,
                                   const double* factors, const double* w_in, long long in_rows,
                                   double* w_out, long long out_rows, double* y, int nrhs,
                                   cudaStream_t st) {
  const unsigned g = (unsigned)((L.n_fronts + kColsWarps - 1) / kColsWarps);
  timer_begin(K_SOLVE_SMALL_FWD, st);
  for (int col0 = 0; col0 < nrhs; col0 += 64) {
    const int nr = std::min(64, nrhs - col0);
    const bool two = nr > 32;
#define TFB_COLS(K, P)                                                                         \
  solve_fwd_cols<K, P><<<g, 32 * kColsWarps, 0, st>>>(L, O, factors, w_in, in_rows, flag, w_out, \
                                                      out_rows, y, nr, nrhs, col0)
    if (L.max_k <= 4) { if (two) TFB_COLS(4, 2); else TFB_COLS(4, 1); }
    else if (L.max_k <= 8) { if (two) TFB_COLS(8, 2); else TFB_COLS(8, 1); }
    else { if (two) TFB_COLS(16, 2); else TFB_COLS(16, 1); }
#undef TFB_COLS
  }
  timer_end(st);
  return cudaGetLastError();
}

// ------------------------------------------------------------- large fronts
// Wavefront sweeps: one persistent launch per level and direction.  Work is
// cut into 64x64 tiles of the fronts' panels; the tiles of the level are
// dealt round-robin, in dependency order, to a co-resident grid, and a tile
// waits on flags published by the tiles it depends on (acquire/release;
// flags cleared before the launch).  Every tile's panel block (and M block)
// is copied to shared memory asynchronously before the tile waits, so the
// per-front dependency chain is one 64x64 product from shared memory per
// pivot block.  Summation orders are fixed: results do not depend on timing.
//   forward : tile (f, R) = rows [64R, 64R+64): W = gather(y, children);
//             W -= L[R, b] Y_b for b < R in order; if R is a pivot block:
//             Y_R = M_R W, y = Y_R / d, publish Y_R.
//   backward: for b = nb-1 .. 0: partial tiles (f, R, b), R >= b+2:
//             P = L[R, b]^T X_R (publish); diagonal tile (f, b):
//             z = y_b - (L[b+1, b]^T X_{b+1} + sum_R P_R), X_b = M_b^T z.
constexpr int TB = 64;         // tile rows = pivot block width (= factorization NB)
constexpr int TLD = TB + 4;    // shared tile row stride (conflict-free 4-thread dots)
constexpr int kWaveCols = 64;  // RHS columns per launch (tile_prod covers up to 64)
// At most this many fronts: prefetch-heavy tile buffers (fewer CTAs per SM).
// Measured on cfg5: the forward sweep wants them only up to 8 fronts (from
// 16 fronts up one buffer and more resident CTAs win, 15-25%), the backward
// one up to 64.  TFB_WAVE_FEW overrides both (tuning sweeps).
static int wave_few_fronts(bool fwd) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("TFB_WAVE_FEW");
    v = e ? atoi(e) : -1;
  }
  return v >= 0 ? v : (fwd ? 8 : 64);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wave_wait(const int* flag) {
  if (threadIdx.x == 0) {
    while (ld_acquire(flag) == 0) __nanosleep(20);
    tfb_jitter((unsigned)(size_t)flag);
  }
  __syncthreads();
}
__device__ __forceinline__ void wave_publish(int* flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(flag, 1);
  }
}
// T[i][c] = src[i * ld + c] for i < rows, c < cols (async 16-byte copies; src
// and T rows 16-byte aligned).  Entries outside are left as they are: the tile
// products below bound their sums and callers ignore out-of-range outputs.
__device__ __forceinline__ void tile_fetch(double* T, const double* src, long long ld, int rows,
                                           int cols) {
  const int cpr = (cols + 1) >> 1;  // 16-byte chunks per row
  for (int e = threadIdx.x; e < rows * cpr; e += 256) {
    const int i = e / cpr, c = (e - i * cpr) * 2;
    if (c + 1 < cols) cp_async16(T + i * TLD + c, src + i * ld + c, true);
    else cp_async8(T + i * TLD + c, src + i * ld + c, true);
  }
  cp_async_commit();
}

// out[i] = sum_{c < nc} T[i][c] v[c] (TRANS: T[c][i]); MASK -1: only c < i,
// +1: only c > i.  One column; four threads per output, interleaved columns
// (conflict-free with TLD = 68); the result is valid in all four threads.
template <bool TRANS, int MASK>
__device__ __forceinline__ double tile_dot(const double* T, const double* v, int nc) {
  const int i = threadIdx.x >> 2, p = threadIdx.x & 3;
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 16; q++) {
    const int c = 4 * q + p;
    const bool on = c < nc && (MASK == 0 || (MASK < 0 ? c < i : c > i));
    if (on) s += (TRANS ? T[c * TLD + i] : T[i * TLD + c]) * v[c];
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  return s;
}
// Several columns: s(i, j) = sum_{c < nc} T[i][c] v[c*nr + j] (TRANS: T[c][i]),
// masked like tile_dot, for i < ni and j < nr <= 64; f(i, j, s) is called once
// per output.  Register-blocked: thread (tid >> 4, tid & 15) owns rows
// ig + 16p and columns jg + 16q (p, q < 4), so each shared load feeds four
// FMAs instead of one.  c runs in order: sums are deterministic.
template <bool TRANS, int MASK, class F>
__device__ __forceinline__ void tile_prod(const double* T, const double* v, int nr, int ni, int nc,
                                          F f) {
  const int ig = threadIdx.x >> 4, jg = threadIdx.x & 15;
  double s[4][4];
#pragma unroll
  for (int p = 0; p < 4; p++)
#pragma unroll
    for (int q = 0; q < 4; q++) s[p][q] = 0.0;
  for (int c = 0; c < nc; c++) {
    double tv[4], vv[4];
#pragma unroll
    for (int p = 0; p < 4; p++) {
      const int i = ig + 16 * p;
      const bool on = MASK == 0 || (MASK < 0 ? c < i : c > i);
      tv[p] = on ? (TRANS ? T[c * TLD + i] : T[i * TLD + c]) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int j = jg + 16 * q;
      vv[q] = j < nr ? v[c * nr + j] : 0.0;
    }
#pragma unroll
    for (int p = 0; p < 4; p++)
#pragma unroll
      for (int q = 0; q < 4; q++) s[p][q] = fma(tv[p], vv[q], s[p][q]);
  }
#pragma unroll
  for (int p = 0; p < 4; p++)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int i = ig + 16 * p, j = jg + 16 * q;
      if (i < ni && j < nr) f(i, j, s[p][q]);
    }
}
// General column count: entry (i, j) of the same product, v row stride nr.
template <bool TRANS, int MASK>
__device__ __forceinline__ double tile_dot_col(const double* T, const double* v, int i, int j,
                                               int nr, int nc) {
  double s = 0.0;
  for (int c = 0; c < nc; c++) {
    const bool on = MASK == 0 || (MASK < 0 ? c < i : c > i);
    if (on) s += (TRANS ? T[c * TLD + i] : T[i * TLD + c]) * v[c * nr + j];
  }
  return s;
}

template <bool ONE>
__global__ void __launch_bounds__(256)
    solve_fwd_wave(LevelArgs L, LevelArgs C, int child_at0, const double* __restrict__ factors,
                   const double* __restrict__ w_child, long long child_rows, double* w_out,
                   long long out_rows, double* y, int nr, int ldr, int col0, int* flags,
                   double* yblk, int nb_max, int rt_max, int nbuf) {
  // nbuf = 3: double-buffered panel tiles plus an early-fetched M tile (levels
  // with few fronts: the per-front chain is the critical path); nbuf = 1: one
  // tile buffer, more CTAs per SM (many fronts: throughput)
  extern __shared__ __align__(16) double wsm[];
  double* T0 = wsm;
  double* T1 = nbuf >= 2 ? T0 + TB * TLD : T0;
  double* Mt = T0 + (nbuf - 1) * TB * TLD;
  double* Wt = T0 + nbuf * TB * TLD;  // [TB][nr]
  double* Yb = Wt + TB * nr;          // [TB][nr]
  const int tid = threadIdx.x;
  TFB_DIV_SETUP(nr);
  const long long nf = L.n_fronts, ntiles = (long long)rt_max * nf;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (threadIdx.x == 0) tfb_jitter((unsigned)tile);
    const int R = (int)(tile / nf);
    const long long f = tile - (long long)R * nf;
    const Shape s = front_shape(L, f);
    const int m = s.m, k = s.k, kp = s.kp, nb = (k + TB - 1) / TB;
    const int r0 = R * TB;
    if (r0 >= m) continue;
    const int rows = min(TB, m - r0);
    const long long piv = L.piv_off[f];
    const double* Pf = factors + f * L.fac_stride;
    int* fl = flags + f * nb_max;
    double* yb = yblk + f * nb_max * TB * nr;
    const int bend = min(R, nb);
    // prefetch: first panel block and (pivot tiles) the M block
    if (bend > 0) tile_fetch(T0, Pf + (long long)r0 * kp, kp, rows, min(TB, k));
    if (R < nb && nbuf == 3) {
      const int kbR = min(TB, k - r0);
      tile_fetch(Mt, L.aux + f * L.aux_stride + (long long)R * TB * TB, TB, kbR, kbR);
    }
    // 1. the tile's rows: pivot-order RHS plus the children's update rows
    {
      long long chs[2] = {0, 0};
      int kc[2] = {0, 0};
      for (int c = 0; c < s.nsrc; c++) {
        chs[c] = 2 * (L.front_base + f) + c - C.front_base;
        kc[c] = child_at0 ? 0 : C.pat[(size_t)C.pattern_of[chs[c]] * TF_PAT_WIDTH + TF_PAT_K];
      }
      const int* inv = L.maps + s.ioff;
      for (int e = tid; e < TB * nr; e += 256) {
        const int rl = ONE ? e : TFB_DIV(e), j = ONE ? 0 : e - rl * nr, r = r0 + rl;
        double v = 0.0;
        if (rl < rows) {
          if (r < k) v = y[(piv + r) * ldr + col0 + j];
          for (int c = 0; c < s.nsrc; c++) {
            const int i = inv[c * m + r];
            if (i >= 0) v += w_child[(chs[c] * child_rows + kc[c] + i) * ldr + col0 + j];
          }
        }
        Wt[e] = v;
      }
    }
    // 2. earlier pivot blocks, in order (next block's tile in flight)
    for (int b = 0; b < bend; b++) {
      double* T = (b & 1) ? T1 : T0;
      if (nbuf >= 2 && b + 1 < bend) {
        tile_fetch((b & 1) ? T0 : T1, Pf + (long long)r0 * kp + (b + 1) * TB, kp, rows,
                   min(TB, k - (b + 1) * TB));
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      wave_wait(fl + b);
      const int kb = min(TB, k - b * TB);
      for (int e0 = tid; e0 < TB * nr; e0 += 8 * 256) {  // eight loads in flight
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const int e = e0 + q * 256;
          v[q] = e < kb * nr ? __ldcg(yb + (long long)b * TB * nr + e) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 8; q++)
          if (e0 + q * 256 < TB * nr) Yb[e0 + q * 256] = v[q];
      }
      __syncthreads();
      if (ONE) {
        const double sdot = tile_dot<false, 0>(T, Yb, kb);
        if ((tid & 3) == 0 && (tid >> 2) < rows) Wt[tid >> 2] -= sdot;
      } else {
        tile_prod<false, 0>(T, Yb, nr, rows, kb,
                            [&](int i, int j, double v) { Wt[i * nr + j] -= v; });
      }
      __syncthreads();
      if (nbuf == 1 && b + 1 < bend)
        tile_fetch(T0, Pf + (long long)r0 * kp + (b + 1) * TB, kp, rows, min(TB, k - (b + 1) * TB));
    }
    // 3. pivot tile: Y = M W on its pivot rows (unit diagonal); publish; own update rows
    if (R < nb) {
      const int kb = min(TB, k - r0);
      if (nbuf < 3) tile_fetch(Mt, L.aux + f * L.aux_stride + (long long)R * TB * TB, TB, kb, kb);
      cp_async_wait<0>();
      __syncthreads();
      if (ONE) {
        const double sdot = tile_dot<false, -1>(Mt, Wt, kb);
        const int i = tid >> 2;
        if ((tid & 3) == 0) Yb[i] = i < kb ? Wt[i] + sdot : 0.0;
      } else {
        tile_prod<false, -1>(Mt, Wt, nr, TB, kb, [&](int i, int j, double v) {
          Yb[i * nr + j] = i < kb ? Wt[i * nr + j] + v : 0.0;
        });
      }
      __syncthreads();
      const double* dv = Pf + (long long)m * kp + r0;
      for (int e = tid; e < kb * nr; e += 256) {
        const int c = ONE ? e : TFB_DIV(e), j = ONE ? 0 : e - c * nr;
        yb[(long long)R * TB * nr + e] = Yb[e];
        y[(piv + r0 + c) * ldr + col0 + j] = Yb[e] / dv[c];
      }
      wave_publish(fl + R);
      if (rows > kb) {  // update rows inside the pivot tile: W -= L[rows, own block] Y
        tile_fetch(T0, Pf + (long long)r0 * kp + r0, kp, rows, kb);
        cp_async_wait<0>();
        __syncthreads();
        if (ONE) {
          const double sdot = tile_dot<false, 0>(T0, Yb, kb);
          const int i = tid >> 2;
          if ((tid & 3) == 0 && i >= kb && i < rows) Wt[i] -= sdot;
        } else {
          tile_prod<false, 0>(T0, Yb, nr, rows, kb, [&](int i, int j, double v) {
            if (i >= kb) Wt[i * nr + j] -= v;
          });
        }
        __syncthreads();
      }
    }
    // 4. the tile's update rows, in place
    for (int e = tid; e < rows * nr; e += 256) {
      const int rl = ONE ? e : e / nr, j = ONE ? 0 : e - rl * nr, r = r0 + rl;
      if (r >= k) w_out[(f * out_rows + r) * ldr + col0 + j] = Wt[e];
    }
    __syncthreads();
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

// Load rows [r0, r0 + rows) of a front's x block (columns col0..col0+nr) into Xs
// [TB][nr], zero-padded; produced rows are read through L2 (__ldcg).
template <bool ONE>
__device__ __forceinline__ void load_x_rows(double* Xs, const double* Xf, int r0, int rows,
                                            int nr, int ldr) {
  if (ONE) {  // one column: one load per thread (keeps the one-column kernel's registers low)
    if (threadIdx.x < TB) Xs[threadIdx.x] = threadIdx.x < rows ? __ldcg(Xf + (long long)(r0 + threadIdx.x) * ldr) : 0.0;
    return;
  }
  const int n = TB * nr;
  for (int e0 = threadIdx.x; e0 < n; e0 += 8 * 256) {  // eight loads in flight
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int e = e0 + q * 256, i = e / nr, j = e - i * nr;
      v[q] = (e < n && i < rows) ? __ldcg(Xf + (long long)(r0 + i) * ldr + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; q++)
      if (e0 + q * 256 < n) Xs[e0 + q * 256] = v[q];
  }
}

template <bool ONE>
__global__ void __launch_bounds__(256)
    solve_bwd_wave(LevelArgs L, const double* __restrict__ factors, double* X, long long out_rows,
                   double* y, int nr, int ldr, int col0, int* flags, double* part, int nb_max,
                   int rt_max, int nbuf) {
  extern __shared__ __align__(16) double wsm[];
  double* T = wsm;                             // panel tile
  double* Mt = T + (nbuf - 1) * TB * TLD;      // M tile (aliases T when nbuf == 1)
  double* Xs = T + nbuf * TB * TLD;            // [TB][nr]
  double* Z = Xs + TB * nr;        // [TB][nr]
  double* red = Z + TB * nr;       // [4][TB] (one column)
  const int tid = threadIdx.x;
  const long long nf = L.n_fronts;
  int* flx = flags;                                  // [nf][nb_max]: X_b final
  int* flp = flags + nf * nb_max;                    // [nf][rt_max][nb_max]: partial (R, b)
  // dependency order: for b = nb_max-1 .. 0: partial tiles (f, R >= b+2), then pivot tiles (f, b)
  long long next = blockIdx.x, base = 0;
  for (int b = nb_max - 1; b >= 0; b--) {
    const long long npart = nf * (long long)max(0, rt_max - b - 2), count = npart + nf;
    for (; next < base + count; next += gridDim.x) {
      const long long item = next - base;
      if (threadIdx.x == 0) tfb_jitter((unsigned)next);
      const bool partial = item < npart;
      const long long f = partial ? item % nf : item - npart;
      const int R = partial ? b + 2 + (int)(item / nf) : b + 1;
      const Shape s = front_shape(L, f);
      const int m = s.m, k = s.k, kp = s.kp, nb = (k + TB - 1) / TB;
      const int rt = (m + TB - 1) / TB;
      if (b >= nb || (partial && R >= rt)) continue;
      const int j0 = b * TB, kb = min(TB, k - j0);
      const long long piv = L.piv_off[f];
      const double* Pf = factors + f * L.fac_stride;
      double* Xf = X + f * out_rows * ldr + col0;
      if (partial) {
        // P = L[R, b]^T X_R
        double* pp = part + ((f * rt_max + R) * (long long)nb_max + b) * TB * nr;
        const int r0 = R * TB, rows = min(TB, m - r0);
        tile_fetch(T, Pf + (long long)r0 * kp + j0, kp, rows, kb);
        if (R < nb) wave_wait(flx + f * nb_max + R);
        load_x_rows<ONE>(Xs, Xf, r0, rows, nr, ldr);
        cp_async_wait<0>();
        __syncthreads();
        if (ONE) {
          const double sdot = tile_dot<true, 0>(T, Xs, rows);
          if ((tid & 3) == 0) pp[tid >> 2] = sdot;
        } else {
          tile_prod<true, 0>(T, Xs, nr, kb, rows,
                             [&](int c, int j, double v) { pp[c * nr + j] = v; });
        }
        wave_publish(flp + (f * rt_max + R) * (long long)nb_max + b);
        __syncthreads();
        continue;
      }
      // pivot tile b.  z = y_b - sum over rows r >= j0 + kb of L[r, b]^T x_r:
      //   (a) update rows sharing the block's own row tile (last block, kb < 64),
      //   (b) partial tiles R >= b+2 (published earlier), in order,
      //   (c) row tile b+1 (waits for X_{b+1}): the dependency chain.
      if (nbuf == 2) tile_fetch(Mt, L.aux + f * L.aux_stride + (long long)b * TB * TB, TB, kb, kb);
      for (int e = tid; e < TB * nr; e += 256) Z[e] = 0.0;
      if (kb < TB && j0 + kb < m) {
        const int rows = min(TB, m - j0);
        tile_fetch(T, Pf + (long long)j0 * kp + j0, kp, rows, kb);
        for (int e = tid; e < TB * nr; e += 256) {
          const int i = e / nr, j = e - i * nr;
          Xs[e] = (i >= kb && i < rows) ? __ldcg(Xf + (long long)(j0 + i) * ldr + j) : 0.0;
        }
        cp_async_wait<0>();
        __syncthreads();
        if (ONE) {
          const double sdot = tile_dot<true, 0>(T, Xs, rows);
          if ((tid & 3) == 0) Z[tid >> 2] = sdot;
        } else {
          tile_prod<true, 0>(T, Xs, nr, kb, rows,
                             [&](int c, int j, double v) { Z[c * nr + j] = v; });
        }
        __syncthreads();
      }
      const int R1 = b + 1, rows1 = R1 < rt ? min(TB, m - R1 * TB) : 0;
      if (rows1 > 0) tile_fetch(T, Pf + (long long)R1 * TB * kp + j0, kp, rows1, kb);
      // (b): every partial's flag polled by its own thread, summed in order
      for (int Rq = b + 2 + tid; Rq < rt; Rq += 256)
        while (ld_acquire(flp + (f * rt_max + Rq) * (long long)nb_max + b) == 0) __nanosleep(20);
      __syncthreads();
      if (ONE) {  // four interleaved partial sums per column, combined in fixed order
        const int c = tid & (TB - 1), g = tid >> 6;
        double acc = 0.0;
        if (c < kb)
          for (int Rq = b + 2 + g; Rq < rt; Rq += 4)
            acc += __ldcg(part + ((f * rt_max + Rq) * (long long)nb_max + b) * TB + c);
        red[g * TB + c] = acc;
        __syncthreads();
        if (tid < kb) Z[tid] += ((red[tid] + red[TB + tid]) + red[2 * TB + tid]) + red[3 * TB + tid];
      } else {
        // kb * nr <= 64 * 64: sixteen entries per thread in two halves, the
        // partials of eight entries requested together (same summation order)
        const int ne = kb * nr;
        for (int h = 0; h < TB * kWaveCols; h += 8 * 256) {
          double acc[8];
#pragma unroll
          for (int q = 0; q < 8; q++) {
            const int e = h + tid + q * 256;
            acc[q] = e < ne ? Z[e] : 0.0;
          }
          for (int Rq = b + 2; Rq < rt; Rq++) {
            const double* pr = part + ((f * rt_max + Rq) * (long long)nb_max + b) * TB * nr;
#pragma unroll
            for (int q = 0; q < 8; q++) {
              const int e = h + tid + q * 256;
              if (e < ne) acc[q] += __ldcg(pr + e);
            }
          }
#pragma unroll
          for (int q = 0; q < 8; q++) {
            const int e = h + tid + q * 256;
            if (e < ne) Z[e] = acc[q];
          }
        }
      }
      // (c)
      if (rows1 > 0 && R1 < nb) wave_wait(flx + f * nb_max + R1);
      load_x_rows<ONE>(Xs, Xf, R1 * TB, rows1, nr, ldr);
      cp_async_wait<0>();
      __syncthreads();
      if (rows1 > 0) {
        if (ONE) {
          const double sdot = tile_dot<true, 0>(T, Xs, rows1);
          if ((tid & 3) == 0) Z[tid >> 2] += sdot;
        } else {
          tile_prod<true, 0>(T, Xs, nr, kb, rows1,
                             [&](int c, int j, double v) { Z[c * nr + j] += v; });
        }
      }
      __syncthreads();
      if (nbuf == 1) tile_fetch(Mt, L.aux + f * L.aux_stride + (long long)b * TB * TB, TB, kb, kb);
      for (int e = tid; e < TB * nr; e += 256) {
        const int c = e / nr, j = e - c * nr;
        Z[e] = c < kb ? y[(piv + j0 + c) * ldr + col0 + j] - Z[e] : 0.0;
      }
      cp_async_wait<0>();
      __syncthreads();
      // X_b = M^T z (M: strict lower part, unit diagonal)
      if (ONE) {
        const double sdot = tile_dot<true, 1>(Mt, Z, kb);
        const int c = tid >> 2;
        if ((tid & 3) == 0 && c < kb) {
          const double xv = Z[c] + sdot;
          Xf[(long long)(j0 + c) * ldr] = xv;
          y[(piv + j0 + c) * ldr + col0] = xv;
        }
      } else {
        tile_prod<true, 1>(Mt, Z, nr, kb, kb, [&](int c, int j, double v) {
          const double xv = Z[c * nr + j] + v;
          Xf[(long long)(j0 + c) * ldr + j] = xv;
          y[(piv + j0 + c) * ldr + col0 + j] = xv;
        });
      }
      wave_publish(flx + f * nb_max + b);
      __syncthreads();
    }
    base += count;
  }
}

__global__ void permute_rows_kernel(const int* __restrict__ idx, long long n,
                                    const double* __restrict__ in, double* __restrict__ out,
                                    int nrhs, int scatter) {
  const long long total = n * nrhs;
  if (nrhs == 1) {  // one column: no row / column split (a 64-bit division per entry)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
      const long long g = (long long)__ldg(idx + i) - 1;
      if (scatter) out[g] = in[i];
      else out[i] = in[g];
    }
    return;
  }
  (void)total;
  // several columns: a warp per row, lanes across the row's columns (coalesced)
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = w0; i < n; i += nw) {
    const long long g = (long long)__ldg(idx + i) - 1;
    const double* src = scatter ? in + i * nrhs : in + g * nrhs;
    double* dst = scatter ? out + g * nrhs : out + i * nrhs;
    for (int j = lane; j < nrhs; j += 32) dst[j] = src[j];
  }
}

// ------------------------------------------------- narrow large fronts
// Large levels whose fronts have k <= 64 pivots (one diagonal block), one
// right-hand side: a warp per front, the front's vector block in shared
// memory.  Every panel row (and every row of the inverse block M) is read by
// the warp as one coalesced request, lanes owning columns t = lane + 32q:
//   forward : Y = M W_piv and W_r - L_r Y (row r >= k) are row dot products,
//             reduced 32 rows at a time by a shuffle transpose-reduction;
//   backward: z = y_piv - L21^T X_rows and x = M^T z accumulate per column,
//             no reduction at all.
// Summation orders are fixed (deterministic).
constexpr int kNarrowWarps = 8;

// 32 row dot products of one warp: sum_t A[r][t] v_t for rows r0 + g + 4j
// (group g = lane / 8, j < 8), t < min(k, TRI ? r : k).  Lane (g, c) reads
// columns [c*CW, c*CW + CW) of its group's rows with 16-byte loads, so each
// warp request covers four whole rows; the eight partial sums of a group are
// combined by a transpose-reduction over its lanes (7 shuffles per 8 rows).
// Returns the sum for row r0 + g + 4c (lane (g, c)).
template <int CW, bool TRI>
__device__ __forceinline__ double rows32_dot(const double* __restrict__ A, int lda, int r0,
                                             int rend, int k, const double (&vt)[CW],
                                             int ncol) {  // readable columns of A's rows (even)
  const int lane = threadIdx.x & 31, g = lane >> 3, c = lane & 7, t0 = c * CW;
  // branch-free: every load is issued up front (rows clamped into the block,
  // columns past the limit read in-bounds neighbours and are masked to zero)
  // (in two halves of four rows: 16-32 registers of loads in flight)
  double v[8];
#pragma unroll
  for (int hf = 0; hf < 8; hf += 4) {
    double2 x[4][CW / 2];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int r = min(r0 + g + 4 * (hf + j), rend - 1);
#pragma unroll
      for (int h = 0; h < CW; h += 2)
        x[j][h / 2] = __ldg(reinterpret_cast<const double2*>(A + (long long)r * lda +
                                                              min(t0 + h, ncol - 2)));
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int r = r0 + g + 4 * (hf + j);
      const int lim = r < rend ? (TRI ? min(k, r) : k) : 0;
      double p = 0.0;
#pragma unroll
      for (int h = 0; h < CW; h += 2) {
        p = fma(t0 + h < lim ? x[j][h / 2].x : 0.0, vt[h], p);
        p = fma(t0 + h + 1 < lim ? x[j][h / 2].y : 0.0, vt[h + 1], p);
      }
      v[hf + j] = p;
    }
  }
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < off; j++) {
      const double send = up ? v[j] : v[j + off];
      const double keep = up ? v[j + off] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// CW = panel columns per lane (8 lanes per row): 4 for k <= 32, 8 for k <= 64
template <int CW>
__global__ void __launch_bounds__(32 * kNarrowWarps, 4)
    solve_fwd_narrow(LevelArgs L, LevelArgs C, int child_at0, const double* __restrict__ factors,
                     const double* __restrict__ w_child, long long child_rows, double* w_out,
                     long long out_rows, double* y, int ldr, int col0) {
  extern __shared__ __align__(16) double nsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long f = (long long)blockIdx.x * kNarrowWarps + warp;
  if (f >= L.n_fronts) return;  // warp-level work only (no CTA barriers)
  double* W = nsm + (long long)warp * L.max_m;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pf = factors + f * L.fac_stride;
  // 1. W = pivot-order RHS rows + the children's update rows
  {
    long long chs[2] = {0, 0};
    int kc[2] = {0, 0};
    for (int c = 0; c < s.nsrc; c++) {
      chs[c] = 2 * (L.front_base + f) + c - C.front_base;
      kc[c] = child_at0 ? 0 : C.pat[(size_t)C.pattern_of[chs[c]] * TF_PAT_WIDTH + TF_PAT_K];
    }
    const int* inv = L.maps + s.ioff;
    for (int r = lane; r < m; r += 32) {
      double v = r < k ? y[(piv + r) * ldr + col0] : 0.0;
      for (int c = 0; c < s.nsrc; c++) {
        const int i = __ldg(inv + c * m + r);
        if (i >= 0) v += w_child[(chs[c] * child_rows + kc[c] + i) * ldr + col0];
      }
      W[r] = v;
    }
  }
  __syncwarp();
  const int t0 = (lane & 7) * CW;
  const int gr = (lane >> 3) + 4 * (lane & 7);  // row of the lane's reduced sum, within 32
  // 2. Y = M W on the pivot rows (M: strict lower part of the aux block, unit diagonal)
  double vt[CW];
#pragma unroll
  for (int h = 0; h < CW; h++) vt[h] = t0 + h < k ? W[t0 + h] : 0.0;
  const double* M = L.aux + f * L.aux_stride;
  double yv[2];
#pragma unroll
  for (int b = 0; b < 2; b++) {
    yv[b] = 0.0;
    if (32 * b < k) {
      const double red = rows32_dot<CW, true>(M, TB, 32 * b, k, k, vt, TB);
      const int n = 32 * b + gr;
      if (n < k) yv[b] = W[n] + red;
    }
  }
  __syncwarp();  // every W read above precedes the stores below
#pragma unroll
  for (int b = 0; b < 2; b++) {
    const int n = 32 * b + gr;
    if (n < k) {
      W[n] = yv[b];
      y[(piv + n) * ldr + col0] = yv[b] / Pf[(long long)m * kp + n];
    }
  }
  __syncwarp();
  // 3. update rows: W_r - L_r Y, 32 rows per round, straight out (in place: rows [k, m))
#pragma unroll
  for (int h = 0; h < CW; h++) vt[h] = t0 + h < k ? W[t0 + h] : 0.0;
  double* out = w_out + f * out_rows * ldr + col0;
  for (int r0 = k; r0 < m; r0 += 32) {
    const double red = rows32_dot<CW, false>(Pf, kp, r0, m, k, vt, kp);
    const int r = r0 + gr;
    if (r < m) out[(long long)r * ldr] = W[r] - red;
  }
}

template <int Q>
__global__ void __launch_bounds__(32 * kNarrowWarps)
    solve_bwd_narrow(LevelArgs L, LevelArgs PA, int has_parent, const double* __restrict__ factors,
                     const double* __restrict__ x_parent, long long parent_rows, double* x_out,
                     long long out_rows, double* y, int ldr, int col0) {
  extern __shared__ __align__(16) double nsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long f = (long long)blockIdx.x * kNarrowWarps + warp;
  if (f >= L.n_fronts) return;
  double* X = nsm + (long long)warp * L.max_m;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pf = factors + f * L.fac_stride;
  // 1. X = pivot rows of y, shared rows gathered from the parent's block
  const int* mp = nullptr;
  const double* Xp = nullptr;
  if (has_parent && m > k) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    mp = PA.maps + (((L.front_base + f) & 1) == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    Xp = x_parent + pf * parent_rows * ldr + col0;
  }
  for (int r = lane; r < m; r += 32)
    X[r] = r < k ? y[(piv + r) * ldr + col0] : (mp ? Xp[(long long)__ldg(mp + r - k) * ldr] : 0.0);
  __syncwarp();
  // 2. z_c = y_c - sum_{r >= k} l_rc x_r (column c = lane + 32q)
  double z[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) z[q] = 0.0;
  int r = k;
  for (; r + 3 < m; r += 4) {  // four rows in flight
    double lv[4][Q];
#pragma unroll
    for (int u = 0; u < 4; u++)
#pragma unroll
      for (int q = 0; q < Q; q++) {
        const int t = lane + 32 * q;
        lv[u][q] = t < k ? __ldg(Pf + (long long)(r + u) * kp + t) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const double xr = X[r + u];
#pragma unroll
      for (int q = 0; q < Q; q++) z[q] += lv[u][q] * xr;
    }
  }
  for (; r < m; r++) {
    const double xr = X[r];
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int t = lane + 32 * q;
      if (t < k) z[q] += __ldg(Pf + (long long)r * kp + t) * xr;
    }
  }
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int t = lane + 32 * q;
    z[q] = t < k ? X[t] - z[q] : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < Q; q++)
    if (lane + 32 * q < k) X[lane + 32 * q] = z[q];
  __syncwarp();
  // 3. x = M^T z: x_c = z_c + sum_{n > c} M(n, c) z_n (rows of M coalesced)
  const double* M = L.aux + f * L.aux_stride;
  double x[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) x[q] = z[q];
  for (int n = 1; n < k; n++) {
    const double zn = X[n];
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int t = lane + 32 * q;
      if (t < n) x[q] += __ldg(M + n * TB + t) * zn;
    }
  }
  double* Xo = x_out + f * out_rows * ldr + col0;
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int t = lane + 32 * q;
    if (t < k) {
      y[(piv + t) * ldr + col0] = x[q];
      Xo[(long long)t * ldr] = x[q];
    }
  }
  for (int rr = k + lane; rr < m; rr += 32) Xo[(long long)rr * ldr] = X[rr];
}

// ------------------------------------------------- CTA-per-front sweeps
// Levels with many fronts of k > 64 pivots, one right-hand side: a CTA per
// front, the front's vector block in shared memory, blocked by the 64-wide
// diagonal blocks of the factorization (inverses M_b from aux).  Every panel
// entry is read once, by coalesced warp requests; no flags, no workspace.
//   forward : per block b: Y_b = M_b W_b (two warps, rows32_dot), then
//             W_r -= L[r, b] Y_b for every row below (32-row chunks dealt to
//             the warps, eight lanes per row);
//   backward: per block b (last first): z_b = X_b - L[rows below, b]^T X_rows
//             (warps split the rows, lanes own columns, fixed-order combine),
//             X_b = M_b^T z_b.
__global__ void __launch_bounds__(256)
    solve_fwd_front(LevelArgs L, LevelArgs C, int child_at0, const double* __restrict__ factors,
                    const double* __restrict__ w_child, long long child_rows, double* w_out,
                    long long out_rows, double* y, int ldr, int col0, double* ywork, int kcols) {
  // ywork != nullptr (split mode): pivot rows only; the unscaled Y goes to
  // ywork[f * kcols + t] for solve_fwd_split_rows, which owns the update rows
  extern __shared__ __align__(16) double fsm[];
  double* W = fsm;
  const long long f = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Shape s = front_shape(L, f);
  const int k = s.k, kp = s.kp, nb = (k + TB - 1) / TB;
  const int m = ywork ? k : s.m;  // rows this kernel sweeps
  const int mf = s.m;             // the panel's row count (d follows it)
  const long long piv = L.piv_off[f];
  const double* Pf = factors + f * L.fac_stride;
  {
    long long chs[2] = {0, 0};
    int kc[2] = {0, 0};
    for (int c = 0; c < s.nsrc; c++) {
      chs[c] = 2 * (L.front_base + f) + c - C.front_base;
      kc[c] = child_at0 ? 0 : C.pat[(size_t)C.pattern_of[chs[c]] * TF_PAT_WIDTH + TF_PAT_K];
    }
    const int* inv = L.maps + s.ioff;
    for (int r = tid; r < m; r += 256) {
      double v = r < k ? y[(piv + r) * ldr + col0] : 0.0;
      for (int c = 0; c < s.nsrc; c++) {
        const int i = __ldg(inv + c * mf + r);
        if (i >= 0) v += w_child[(chs[c] * child_rows + kc[c] + i) * ldr + col0];
      }
      W[r] = v;
    }
  }
  __syncthreads();
  const int t0 = (lane & 7) * 8;
  const int gr = (lane >> 3) + 4 * (lane & 7);
  for (int b = 0; b < nb; b++) {
    const int c0 = b * TB, kb = min(TB, k - c0);
    double vt[8];
    double yv = 0.0;
    const int n = 32 * warp + gr;
    if (warp < 2 && 32 * warp < kb) {
#pragma unroll
      for (int h = 0; h < 8; h++) vt[h] = t0 + h < kb ? W[c0 + t0 + h] : 0.0;
      const double* M = L.aux + f * L.aux_stride + (long long)b * TB * TB;
      const double red = rows32_dot<8, true>(M, TB, 32 * warp, kb, kb, vt, TB);
      if (n < kb) yv = W[c0 + n] + red;
    }
    __syncthreads();
    if (warp < 2 && n < kb) {
      W[c0 + n] = yv;
      y[(piv + c0 + n) * ldr + col0] = yv / Pf[(long long)mf * kp + c0 + n];
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 8; h++) vt[h] = t0 + h < kb ? W[c0 + t0 + h] : 0.0;
    for (int rs = c0 + kb + 32 * warp; rs < m; rs += 256) {
      const double red = rows32_dot<8, false>(Pf + c0, kp, rs, m, kb, vt, kp - c0);
      const int r = rs + gr;
      if (r < m) W[r] -= red;
    }
    __syncthreads();
  }
  if (ywork) {
    for (int t = tid; t < k; t += 256) ywork[f * kcols + t] = W[t];
    return;
  }
  double* out = w_out + f * out_rows * ldr + col0;
  for (int r = k + tid; r < m; r += 256) out[(long long)r * ldr] = W[r];
}

// Split forward sweep, update rows: grid (fronts, chunks of kSplitRows rows of
// [k, m)); W_r (children gathered) - sum over the 64-column blocks of
// L[r, b] Y_b, Y from solve_fwd_front's split mode.
constexpr int kSplitRows = 256;
__global__ void __launch_bounds__(256)
    solve_fwd_split_rows(LevelArgs L, LevelArgs C, int child_at0,
                         const double* __restrict__ factors, const double* __restrict__ w_child,
                         long long child_rows, double* w_out, long long out_rows,
                         const double* __restrict__ ywork, int kcols, int ldr, int col0) {
  extern __shared__ __align__(16) double fsm[];
  double* W = fsm;              // [kSplitRows]
  double* Ys = W + kSplitRows;  // [kcols]
  const long long f = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp, nb = (k + TB - 1) / TB;
  const int rs = k + blockIdx.y * kSplitRows;
  if (rs >= m) return;
  const int re = min(m, rs + kSplitRows);
  const double* Pf = factors + f * L.fac_stride;
  {
    long long chs[2] = {0, 0};
    int kc[2] = {0, 0};
    for (int c = 0; c < s.nsrc; c++) {
      chs[c] = 2 * (L.front_base + f) + c - C.front_base;
      kc[c] = child_at0 ? 0 : C.pat[(size_t)C.pattern_of[chs[c]] * TF_PAT_WIDTH + TF_PAT_K];
    }
    const int* inv = L.maps + s.ioff;
    for (int r = rs + tid; r < re; r += 256) {
      double v = 0.0;
      for (int c = 0; c < s.nsrc; c++) {
        const int i = __ldg(inv + c * m + r);
        if (i >= 0) v += w_child[(chs[c] * child_rows + kc[c] + i) * ldr + col0];
      }
      W[r - rs] = v;
    }
  }
  for (int t = tid; t < k; t += 256) Ys[t] = __ldcg(ywork + f * kcols + t);
  __syncthreads();
  const int t0 = (lane & 7) * 8;
  const int gr = (lane >> 3) + 4 * (lane & 7);
  double* out = w_out + f * out_rows * ldr + col0;
  for (int r0 = rs + 32 * warp; r0 < re; r0 += 256) {
    double red = 0.0;
    for (int b = 0; b < nb; b++) {
      const int c0 = b * TB, kb = min(TB, k - c0);
      double vt[8];
#pragma unroll
      for (int h = 0; h < 8; h++) vt[h] = t0 + h < kb ? Ys[c0 + t0 + h] : 0.0;
      red += rows32_dot<8, false>(Pf + c0, kp, r0, re, kb, vt, kp - c0);
    }
    const int r = r0 + gr;
    if (r < re) out[(long long)r * ldr] = W[r - rs] - red;
  }
}

__global__ void __launch_bounds__(256)
    solve_bwd_front(LevelArgs L, LevelArgs PA, int has_parent, const double* __restrict__ factors,
                    const double* __restrict__ x_parent, long long parent_rows, double* x_out,
                    long long out_rows, double* y, int ldr, int col0, const double* part,
                    int nchunk, int kcols) {
  // part != nullptr (split mode): the update rows' contributions were summed
  // per chunk by solve_bwd_split_rows (part[(f * nchunk + chunk) * kcols + c]);
  // this kernel sweeps the pivot rows only
  extern __shared__ __align__(16) double fsm[];
  double* red = fsm;            // [8][TB]
  double* Z = red + 8 * TB;     // [TB]
  double* X = Z + TB;           // [max_m]
  const long long f = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Shape s = front_shape(L, f);
  const int k = s.k, kp = s.kp, nb = (k + TB - 1) / TB;
  const int m = part ? k : s.m;
  const int nch = part ? (s.m - k + kSplitRows - 1) / kSplitRows : 0;
  const long long piv = L.piv_off[f];
  const double* Pf = factors + f * L.fac_stride;
  const int* mp = nullptr;
  const double* Xp = nullptr;
  if (has_parent && m > k) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    mp = PA.maps + (((L.front_base + f) & 1) == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    Xp = x_parent + pf * parent_rows * ldr + col0;
  }
  for (int r = tid; r < m; r += 256)
    X[r] = r < k ? y[(piv + r) * ldr + col0] : (mp ? Xp[(long long)__ldg(mp + r - k) * ldr] : 0.0);
  __syncthreads();
  for (int b = nb - 1; b >= 0; b--) {
    const int c0 = b * TB, kb = min(TB, k - c0);
    // z_b = X_b - sum over the rows below of l_rc x_r
    double acc[2] = {0.0, 0.0};
    const double* Pc = Pf + c0;
    int r = c0 + kb + warp;
    for (; r + 56 < m; r += 64) {  // eight rows of this warp in flight
      double lv[8][2], xr[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        xr[u] = X[r + 8 * u];
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const int c = lane + 32 * q;
          lv[u][q] = c < kb ? __ldg(Pc + (long long)(r + 8 * u) * kp + c) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; u++)
#pragma unroll
        for (int q = 0; q < 2; q++) acc[q] += lv[u][q] * xr[u];
    }
    for (; r < m; r += 8) {
      const double xr = X[r];
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int c = lane + 32 * q;
        if (c < kb) acc[q] += __ldg(Pc + (long long)r * kp + c) * xr;
      }
    }
    red[warp * TB + lane] = acc[0];
    red[warp * TB + lane + 32] = acc[1];
    __syncthreads();
    if (tid < kb) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; w++) t += red[w * TB + tid];
      for (int ch = 0; ch < nch; ch++) t += __ldcg(part + (f * nchunk + ch) * kcols + c0 + tid);
      Z[tid] = X[c0 + tid] - t;
    }
    __syncthreads();
    // X_b = M_b^T z_b: x_c = z_c + sum_{n > c} M(n, c) z_n
    const double* M = L.aux + f * L.aux_stride + (long long)b * TB * TB;
    acc[0] = acc[1] = 0.0;
    for (int n = warp; n < kb; n += 8) {
      const double zn = Z[n];
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int c = lane + 32 * q;
        if (c < n) acc[q] += __ldg(M + n * TB + c) * zn;
      }
    }
    red[warp * TB + lane] = acc[0];
    red[warp * TB + lane + 32] = acc[1];
    __syncthreads();
    if (tid < kb) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; w++) t += red[w * TB + tid];
      const double xv = Z[tid] + t;
      X[c0 + tid] = xv;
      y[(piv + c0 + tid) * ldr + col0] = xv;
    }
    __syncthreads();
  }
  double* Xo = x_out + f * out_rows * ldr + col0;
  for (int rr = tid; rr < m; rr += 256) Xo[(long long)rr * ldr] = X[rr];
}

// Measured on cfg5 (k = 128, 256): the CTA-per-front sweeps beat the
// wavefront kernels from 256 fronts up backward (1.2-2.5x) and from 512 up
// forward (5-15%);
// below that the wavefront's tile parallelism wins
// (TFB_FRONT_SOLVE=0 disables both; TFB_FRONT_MIN_FRONTS overrides the bound).
// ----------------------------------------- small fronts, one RHS, 8 < k <= 16
// A warp per front (non-leaf small levels): the pivot triangle by warp
// substitution (each lane holds its row / column of L11 in registers,
// pivots broadcast by shuffles), the update rows by rows32_dot (eight lanes
// per 128-byte panel row) forward, and by column accumulation over two row
// streams backward.  Block conventions as solve_fwd_small / solve_bwd_small.
constexpr int kSmallWarps = 8;

__global__ void __launch_bounds__(32 * kSmallWarps)
    solve_fwd_warp16(LevelArgs L, LevelArgs C, const double* __restrict__ factors,
                     const double* __restrict__ w_child, long long child_rows, int child_at0,
                     double* w_out, long long out_rows, double* y, int ldr, int col0) {
  extern __shared__ __align__(16) double wsm16[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long f = (long long)blockIdx.x * kSmallWarps + warp;
  if (f >= L.n_fronts) return;
  double* W = wsm16 + (long long)warp * L.max_m;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pf = factors + f * L.fac_stride;
  for (int r = lane; r < m; r += 32) W[r] = r < k ? y[(piv + r) * ldr + col0] : 0.0;
  __syncwarp();
  for (int c = 0; c < s.nsrc; c++) {  // children one after the other (shared rows collide)
    const long long ch = 2 * (L.front_base + f) + c - C.front_base;
    const int off = child_at0 ? 0 : C.pat[(size_t)C.pattern_of[ch] * TF_PAT_WIDTH + TF_PAT_K];
    const int len = c == 0 ? s.len0 : s.len1;
    const int* mp = L.maps + (c == 0 ? s.off0 : s.off1);
    const double* Wc = w_child + (ch * child_rows + off) * ldr + col0;
    for (int a = lane; a < len; a += 32) W[__ldg(mp + a)] += Wc[(long long)a * ldr];
    __syncwarp();
  }
  // pivot triangle: lane r < k holds w_r and row r of L11
  double lr[16];
#pragma unroll
  for (int j = 0; j < 16; j++) lr[j] = (lane < k && j < lane) ? __ldg(Pf + (long long)lane * kp + j) : 0.0;
  double w = lane < k ? W[lane] : 0.0;
#pragma unroll
  for (int c = 0; c < 15; c++) {
    const double yc = __shfl_sync(0xffffffffu, w, c);
    w -= lr[c] * yc;  // lr[c] = 0 unless c < lane < k
  }
  if (lane < k) {
    W[lane] = w;
    y[(piv + lane) * ldr + col0] = w / Pf[(long long)m * kp + lane];
  }
  __syncwarp();
  const int t0 = (lane & 7) * 2;
  const int gr = (lane >> 3) + 4 * (lane & 7);
  double vt[2];
#pragma unroll
  for (int h = 0; h < 2; h++) vt[h] = t0 + h < k ? W[t0 + h] : 0.0;
  double* out = w_out + f * out_rows * ldr + col0;
  for (int r0 = k; r0 < m; r0 += 32) {
    const double red = rows32_dot<2, false>(Pf, kp, r0, m, k, vt, kp);
    const int r = r0 + gr;
    if (r < m) out[(long long)(r - k) * ldr] = W[r] - red;
  }
}

__global__ void __launch_bounds__(32 * kSmallWarps)
    solve_bwd_warp16(LevelArgs L, LevelArgs PA, int has_parent, const double* __restrict__ factors,
                     const double* __restrict__ x_parent, long long parent_rows, double* x_out,
                     long long out_rows, double* y, int ldr, int col0) {
  extern __shared__ __align__(16) double wsm16[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long f = (long long)blockIdx.x * kSmallWarps + warp;
  if (f >= L.n_fronts) return;
  double* X = wsm16 + (long long)warp * L.max_m;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const long long piv = L.piv_off[f];
  const double* Pf = factors + f * L.fac_stride;
  const int* mp = nullptr;
  const double* Xp = nullptr;
  if (has_parent && m > k) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    mp = PA.maps + (((L.front_base + f) & 1) == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    Xp = x_parent + pf * parent_rows * ldr + col0;
  }
  for (int r = lane; r < m; r += 32)
    X[r] = r < k ? y[(piv + r) * ldr + col0] : (mp ? Xp[(long long)__ldg(mp + r - k) * ldr] : 0.0);
  __syncwarp();
  // z_c = y_c - sum_{r >= k} l_rc x_r: lane (half, c) = (lane / 16, lane % 16), rows by parity
  const int c = lane & 15, hr = lane >> 4;
  double acc = 0.0;
  int r = k + hr;
  for (; r + 6 < m; r += 8) {  // four rows of this half in flight
    double lv[4], xr[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      lv[u] = c < k ? __ldg(Pf + (long long)(r + 2 * u) * kp + c) : 0.0;
      xr[u] = X[r + 2 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; u++) acc += lv[u] * xr[u];
  }
  for (; r < m; r += 2) acc += (c < k ? __ldg(Pf + (long long)r * kp + c) : 0.0) * X[r];
  acc += __shfl_xor_sync(0xffffffffu, acc, 16);
  // backward substitution with L11^T: lane c < k holds column c of L11
  double lc[16];
#pragma unroll
  for (int j = 0; j < 16; j++) lc[j] = (lane < k && j > lane && j < k) ? __ldg(Pf + (long long)j * kp + lane) : 0.0;
  double z = lane < k ? X[lane] - acc : 0.0;
#pragma unroll
  for (int j = 15; j > 0; j--) {
    const double xj = __shfl_sync(0xffffffffu, z, j);
    z -= lc[j] * xj;  // lc[j] = 0 unless lane < j < k
  }
  __syncwarp();
  if (lane < k) {
    y[(piv + lane) * ldr + col0] = z;
    X[lane] = z;
  }
  __syncwarp();
  if (L.children_idle(f)) return;  // children without pivots never read the block
  double* Xo = x_out + f * out_rows * ldr + col0;
  for (int rr = lane; rr < m; rr += 32) Xo[(long long)rr * ldr] = X[rr];
}

static bool warp16_solve(const LevelArgs& L, int nrhs) {
  static int v = -1;  // TFB_WARP16_SOLVE=0: group-per-front kernels instead (A/B)
  if (v < 0) {
    const char* e = getenv("TFB_WARP16_SOLVE");
    v = e ? atoi(e) != 0 : 1;
  }
  // measured on cfg5: 2x faster at k = 16 (m = 79, 111), 1.4x slower at k = 8
  return v && nrhs == 1 && !L.is_leaf && L.max_k > 8 && L.max_k <= 16;
}

// Split backward sweep, update rows: grid (fronts, chunks of kSplitRows rows,
// 64-column blocks); partial z of the chunk for the block's columns (warps
// split the rows, lanes own columns, fixed-order combine).  Block 0 of each
// chunk also writes the chunk's rows of the front's X block for the children.
__global__ void __launch_bounds__(256)
    solve_bwd_split_rows(LevelArgs L, LevelArgs PA, int has_parent,
                         const double* __restrict__ factors, const double* __restrict__ x_parent,
                         long long parent_rows, double* x_out, long long out_rows, double* part,
                         int nchunk, int kcols, int ldr, int col0) {
  __shared__ double Xs[kSplitRows];
  __shared__ double red[8][TB];
  const long long f = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Shape s = front_shape(L, f);
  const int m = s.m, k = s.k, kp = s.kp;
  const int rs = k + blockIdx.y * kSplitRows, c0 = blockIdx.z * TB;
  if (rs >= m || (c0 >= k && blockIdx.z > 0)) return;  // block 0 always serves X (k may be 0)
  const int re = min(m, rs + kSplitRows), kb = min(TB, k - c0);
  const double* Pf = factors + f * L.fac_stride;
  if (has_parent) {
    const long long pf = ((L.front_base + f) >> 1) - PA.front_base;
    const int* PP = PA.pat + (size_t)PA.pattern_of[pf] * TF_PAT_WIDTH;
    const int* mp = PA.maps + (((L.front_base + f) & 1) == 0 ? PP[TF_PAT_OFF0] : PP[TF_PAT_OFF1]);
    const double* Xp = x_parent + pf * parent_rows * ldr + col0;
    for (int r = rs + tid; r < re; r += 256) Xs[r - rs] = Xp[(long long)__ldg(mp + r - k) * ldr];
  } else {
    for (int r = rs + tid; r < re; r += 256) Xs[r - rs] = 0.0;
  }
  __syncthreads();
  if (blockIdx.z == 0) {
    double* Xo = x_out + f * out_rows * ldr + col0;
    for (int r = rs + tid; r < re; r += 256) Xo[(long long)r * ldr] = Xs[r - rs];
  }
  if (kb <= 0) return;  // a front without pivots: X rows only
  double acc[2] = {0.0, 0.0};
  const double* Pc = Pf + c0;
  int r = rs + warp;
  for (; r + 56 < re; r += 64) {  // eight rows of this warp in flight
    double lv[8][2], xr[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      xr[u] = Xs[r + 8 * u - rs];
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int c = lane + 32 * q;
        lv[u][q] = c < kb ? __ldg(Pc + (long long)(r + 8 * u) * kp + c) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; u++)
#pragma unroll
      for (int q = 0; q < 2; q++) acc[q] += lv[u][q] * xr[u];
  }
  for (; r < re; r += 8) {
    const double xr = Xs[r - rs];
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int c = lane + 32 * q;
      if (c < kb) acc[q] += __ldg(Pc + (long long)r * kp + c) * xr;
    }
  }
  red[warp][lane] = acc[0];
  red[warp][lane + 32] = acc[1];
  __syncthreads();
  if (tid < kb) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; w++) t += red[w][tid];
    part[(f * nchunk + blockIdx.y) * kcols + c0 + tid] = t;
  }
}

// Levels with fewer fronts (k > 64): split sweeps, the update rows spread
// over (front, row chunk) CTAs.  Measured on cfg5: backward 1.4-2x faster
// than the wavefront from 32 fronts up; forward slower at every level (its
// pivot-row pass is one CTA per front), so it runs only when forced.
// TFB_SPLIT_SOLVE=0: off; 2: both directions on every such level (tests).
static bool split_solve(const LevelArgs& L, int nrhs, bool fwd) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFB_SPLIT_SOLVE");
    v = e ? atoi(e) : 1;
  }
  if (v == 0 || (fwd && v < 2)) return false;
  return nrhs == 1 && L.max_k > 0 && L.level_fronts >= (v >= 2 ? 1 : 32) &&
         (size_t)(L.max_m + 9 * TB) * 8 <= 200 * 1024;
}

static bool front_solve(const LevelArgs& L, int nrhs, bool fwd) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TFB_FRONT_SOLVE");
    v = e ? atoi(e) : 1;
  }
  static long long min_fronts = -1;  // TFB_FRONT_MIN_FRONTS (tests: drive small meshes through it)
  if (min_fronts < 0) {
    const char* e = getenv("TFB_FRONT_MIN_FRONTS");
    min_fronts = e ? atoll(e) : 0;
  }
  if (v == 0) return false;
  const long long need = min_fronts > 0 ? min_fronts : (fwd ? 512 : 256);
  return nrhs == 1 && L.max_k > 0 && L.level_fronts >= need &&
         (size_t)(L.max_m + 9 * TB) * 8 <= 200 * 1024;
}

static bool narrow_solve(const LevelArgs& L, int nrhs) {
  static int v = -1;  // TFB_NARROW_SOLVE=0: wavefront kernels instead (A/B)
  if (v < 0) {
    const char* e = getenv("TFB_NARROW_SOLVE");
    v = e ? atoi(e) != 0 : 1;
  }
  // a warp per front needs many fronts to fill the GPU (cfg5: >= 2048);
  // fewer fronts take the CTA-per-front / split / wavefront sweeps
  return v && nrhs == 1 && L.max_k > 0 && L.max_k <= 2 * 32 && L.level_fronts >= 1024 &&
         (size_t)kNarrowWarps * L.max_m * 8 <= 200 * 1024;
}

template <class K>
static void narrow_attr(K kern, size_t smem) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// ------------------------------------------------------------------ launch
constexpr size_t kSmallSolveSmem = 160 * 1024;

template <int G, int GPC, bool FWD, bool STAGE>
static cudaError_t launch_small_solve(const LevelArgs& L, const LevelArgs& O, int flag,
                                      const double* factors, const double* w_in,
                                      long long in_rows, double* w_out, long long out_rows,
                                      double* y, int nr, int ldr, int col0, cudaStream_t st) {
  const size_t pan = STAGE ? (size_t)L.max_m * L.max_k + L.max_m : 0;
  // per-group stride in doubles = G mod 16 (G < 16): the groups of a warp
  // are staggered over the shared-memory banks (an odd stride for G = 1)
  int per_d = (int)((size_t)L.max_m * nr + pan);
  if (G < 16) {
    while ((per_d & 15) != (G & 15)) per_d++;
  } else {
    per_d = (per_d + 1) & ~1;
  }
  const int per = per_d * 8;
  const size_t smem = (size_t)per * GPC;
  const unsigned full = (unsigned)((L.n_fronts + GPC - 1) / GPC);
  // leaf levels: nearly every front is pivot-free (returns at once): a few
  // resident waves of CTAs stride over the level
  const unsigned blocks = L.is_leaf ? std::min(full, 148u * 16u) : full;
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
  if (nrhs <= cmax) return std::max(1, nrhs);
  int cw = 1;  // sliced anyway: power-of-two slices keep the kernels' index split a shift
  while (cw * 2 <= cmax) cw *= 2;
  return cw;
}

// flag: forward -- 1 if the child level's update rows start at row 0 of its
// blocks (small child level); backward -- has_parent.
template <bool FWD>
static cudaError_t dispatch_small(const LevelArgs& L, const LevelArgs& O, int flag,
                                  const double* factors, const double* w_in, long long in_rows,
                                  double* w_out, long long out_rows, double* y, int nrhs,
                                  cudaStream_t st) {
  if (cols_solve_fwd(L, nrhs)) {
    if (FWD) return launch_fwd_cols(L, O, flag, factors, w_in, in_rows, w_out, out_rows, y, nrhs, st);
    return launch_bwd_cols(L, O, flag, factors, w_in, in_rows, w_out, out_rows, y, nrhs, st);
  }
  if (warp16_solve(L, nrhs)) {
    const size_t smem = (size_t)kSmallWarps * L.max_m * 8;
    const unsigned g = (unsigned)((L.n_fronts + kSmallWarps - 1) / kSmallWarps);
    if (FWD) {
      timer_begin(K_SOLVE_SMALL_FWD, st);
      solve_fwd_warp16<<<g, 32 * kSmallWarps, smem, st>>>(L, O, factors, w_in, in_rows, flag, w_out,
                                                          out_rows, y, nrhs, 0);
    } else {
      timer_begin(K_SOLVE_SMALL_BWD, st);
      solve_bwd_warp16<<<g, 32 * kSmallWarps, smem, st>>>(L, O, flag, factors, w_in, in_rows, w_out,
                                                          out_rows, y, nrhs, 0);
    }
    timer_end(st);
    return cudaGetLastError();
  }
  const int cw = small_cols(L, nrhs);
  for (int col0 = 0; col0 < nrhs; col0 += cw) {
    const int nr = std::min(cw, nrhs - col0);
    const long long work = (long long)L.max_m * nr;
    cudaError_t e;
    if (nr == 1) {  // vector block only in shared memory
#define TFB_SMALL(G, GPC)                                                                    \
  launch_small_solve<G, GPC, FWD, false>(L, O, flag, factors, w_in, in_rows, w_out, out_rows, \
                                         y, nr, nrhs, col0, st)
      // (G, GPC) per class m <= 12, 24, 48, 96, 256, rest; TFB_SOLVE_CFG overrides
      static int cfg[6][2] = {{1, 128}, {2, 64}, {4, 64}, {8, 32}, {32, 8}, {128, 2}};
      static bool parsed = false;
      if (!parsed) {
        parsed = true;
        if (const char* ev = getenv("TFB_SOLVE_CFG")) {
          for (int i = 0; i < 6 && *ev; i++) {
            int g = 0, n = 0;
            if (sscanf(ev, "%d:%d", &g, &n) == 2) { cfg[i][0] = g; cfg[i][1] = n; }
            while (*ev && *ev != ',') ev++;
            if (*ev == ',') ev++;
          }
        }
      }
      const int cls = work <= 12 ? 0 : work <= 24 ? 1 : work <= 48 ? 2 : work <= 96 ? 3
                    : work <= 256 ? 4 : 5;
      const int G = cfg[cls][0], GPC = cfg[cls][1];
      e = cudaErrorInvalidValue;
#define TFB_CASE(g, n) \
  if (G == g && GPC == n) e = TFB_SMALL(g, n);
      TFB_CASE(1, 128) TFB_CASE(1, 256) TFB_CASE(1, 64) TFB_CASE(2, 64) TFB_CASE(2, 128)
      TFB_CASE(4, 64) TFB_CASE(4, 32) TFB_CASE(8, 32) TFB_CASE(8, 16) TFB_CASE(16, 16)
      TFB_CASE(16, 8) TFB_CASE(32, 8) TFB_CASE(32, 4) TFB_CASE(64, 4) TFB_CASE(128, 2)
#undef TFB_CASE
#undef TFB_SMALL
    } else {
      const long long bytes = (work + (long long)L.max_m * L.max_k + L.max_m) * 8;
#define TFB_SMALL(G, GPC)                                                                   \
  launch_small_solve<G, GPC, FWD, true>(L, O, flag, factors, w_in, in_rows, w_out, out_rows, \
                                        y, nr, nrhs, col0, st)
      if (work <= 24 && bytes * 64 <= (long long)kSmallSolveSmem) e = TFB_SMALL(2, 64);
      else if (work <= 48 && bytes * 64 <= (long long)kSmallSolveSmem) e = TFB_SMALL(4, 64);
      else if (work <= 96 && bytes * 32 <= (long long)kSmallSolveSmem) e = TFB_SMALL(8, 32);
      else if (work <= 1024 && bytes * 8 <= (long long)kSmallSolveSmem) e = TFB_SMALL(32, 8);
      else if (work <= 4096 && bytes * 2 <= (long long)kSmallSolveSmem) e = TFB_SMALL(128, 2);
      else e = TFB_SMALL(256, 1);
#undef TFB_SMALL
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Large levels: Y blocks (forward) or partial products (backward), then flags.
static long long wave_blocks_doubles(const LevelArgs& L, int nrhs) {
  const long long nb = (L.max_k + TB - 1) / TB, rt = (L.max_m + TB - 1) / TB;
  return (long long)L.n_fronts * rt * nb * TB * std::min(nrhs, kWaveCols);
}
long long solve_workspace_doubles(const LevelArgs& L, int nrhs) {
  if (!level_is_large(L.is_leaf, L.max_m)) return 0;
  const long long nb = (L.max_k + TB - 1) / TB, rt = (L.max_m + TB - 1) / TB;
  return wave_blocks_doubles(L, nrhs) + ((long long)L.n_fronts * nb * (1 + rt) + 1) / 2 + 1;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 1;
  }
  return n;
}

// Co-resident grid for a persistent wavefront kernel (tiles wait on each other).
template <class K>
static unsigned wave_grid(K kern, size_t smem, long long ntiles) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  const long long cap = (long long)num_sms() * std::max(occ, 1);
  return (unsigned)std::max(1LL, std::min(ntiles, cap));
}

// Zero the update blocks of leaf elements without pivots (the leaf sweep
// skips them) for parent kernels that read every child block.
__global__ void __launch_bounds__(256)
    zero_unpivoted_leaf_blocks(LevelArgs C, double* w, long long per_front) {
  for (long long f = blockIdx.x; f < C.n_fronts; f += gridDim.x) {
    if (!C.upd_is_zero(f)) continue;
    for (long long i = threadIdx.x; i < per_front; i += blockDim.x) w[f * per_front + i] = 0.0;
  }
}

cudaError_t launch_solve_fwd(const LevelArgs& L, const LevelArgs& C, const double* factors,
                             const double* w_child, long long child_rows, double* w_out,
                             long long out_rows, double* y, int nrhs, double* work,
                             long long work_doubles, cudaStream_t st) {
  const int child_at0 = level_is_large(C.is_leaf, C.max_m) ? 0 : 1;
  // Leaf elements without pivots never write their (zero) update blocks; the
  // group kernels skip such children, every other kernel gets them zeroed.
  const bool small = !level_is_large(L.is_leaf, L.max_m);
  if ((C.is_leaf || C.zero_upd) && w_child && C.n_fronts > 0 && (!small || warp16_solve(L, nrhs))) {
    zero_unpivoted_leaf_blocks<<<(unsigned)std::min<long long>(C.n_fronts, 148 * 8), 256, 0, st>>>(
        C, const_cast<double*>(w_child), child_rows * nrhs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (small)
    return dispatch_small<true>(L, C, child_at0, factors, w_child, child_rows, w_out, out_rows, y,
                                nrhs, st);
  if (narrow_solve(L, nrhs)) {
    const size_t smem = (size_t)kNarrowWarps * L.max_m * 8;
    const unsigned g = (unsigned)((L.n_fronts + kNarrowWarps - 1) / kNarrowWarps);
    timer_begin(K_SOLVE_FWD_WAVE, st);
    if (L.max_k <= 32) {
      narrow_attr(solve_fwd_narrow<4>, smem);
      solve_fwd_narrow<4><<<g, 32 * kNarrowWarps, smem, st>>>(L, C, child_at0, factors, w_child,
                                                              child_rows, w_out, out_rows, y, nrhs, 0);
    } else {
      narrow_attr(solve_fwd_narrow<8>, smem);
      solve_fwd_narrow<8><<<g, 32 * kNarrowWarps, smem, st>>>(L, C, child_at0, factors, w_child,
                                                              child_rows, w_out, out_rows, y, nrhs, 0);
    }
    timer_end(st);
    return cudaGetLastError();
  }
  if (front_solve(L, nrhs, true)) {
    const size_t smem = (size_t)L.max_m * 8;
    narrow_attr(solve_fwd_front, smem);
    timer_begin(K_SOLVE_FWD_WAVE, st);
    solve_fwd_front<<<(unsigned)L.n_fronts, 256, smem, st>>>(
        L, C, child_at0, factors, w_child, child_rows, w_out, out_rows, y, nrhs, 0, nullptr, 0);
    timer_end(st);
    return cudaGetLastError();
  }
  if (split_solve(L, nrhs, true)) {
    if (!work || work_doubles < solve_workspace_doubles(L, nrhs)) return cudaErrorInvalidValue;
    const int kcols = (L.max_k + TB - 1) / TB * TB;
    const unsigned nch = (unsigned)std::max(1, (L.max_upd + kSplitRows - 1) / kSplitRows);
    const size_t smem = (size_t)L.max_m * 8;
    narrow_attr(solve_fwd_front, smem);
    timer_begin(K_SOLVE_FWD_WAVE, st);
    solve_fwd_front<<<(unsigned)L.n_fronts, 256, smem, st>>>(
        L, C, child_at0, factors, w_child, child_rows, w_out, out_rows, y, nrhs, 0, work, kcols);
    const size_t smem2 = (size_t)(kSplitRows + kcols) * 8;
    narrow_attr(solve_fwd_split_rows, smem2);
    solve_fwd_split_rows<<<dim3((unsigned)L.n_fronts, nch), 256, smem2, st>>>(
        L, C, child_at0, factors, w_child, child_rows, w_out, out_rows, work, kcols, nrhs, 0);
    timer_end(st);
    return cudaGetLastError();
  }
  if (!work || work_doubles < solve_workspace_doubles(L, nrhs)) return cudaErrorInvalidValue;
  const int nb = (L.max_k + TB - 1) / TB, rt = (L.max_m + TB - 1) / TB;
  const int cw = std::min(nrhs, kWaveCols);
  double* yblk = work;
  int* flags = reinterpret_cast<int*>(work + wave_blocks_doubles(L, nrhs));
  for (int col0 = 0; col0 < nrhs; col0 += cw) {
    const int nr = std::min(cw, nrhs - col0);
    const int nbuf = L.n_fronts <= wave_few_fronts(true) ? 3 : 1;
    const size_t smem = sizeof(double) * (nbuf * TB * TLD + 2 * TB * nr);
    if (nb > 0) cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)L.n_fronts * nb, st);
    timer_begin(K_SOLVE_FWD_WAVE, st);
    cudaError_t e;
    if (nr == 1) {
      const unsigned g = wave_grid(solve_fwd_wave<true>, smem, (long long)rt * L.n_fronts);
      e = launch_cooperative(solve_fwd_wave<true>, dim3(g), dim3(256), smem, st, L, C, child_at0,
                             factors, w_child, child_rows, w_out, out_rows, y, nr, nrhs, col0,
                             flags, yblk, nb, rt, nbuf);
    } else {
      const unsigned g = wave_grid(solve_fwd_wave<false>, smem, (long long)rt * L.n_fronts);
      e = launch_cooperative(solve_fwd_wave<false>, dim3(g), dim3(256), smem, st, L, C, child_at0,
                             factors, w_child, child_rows, w_out, out_rows, y, nr, nrhs, col0,
                             flags, yblk, nb, rt, nbuf);
    }
    timer_end(st);
    if (e != cudaSuccess) return e;
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
  if (narrow_solve(L, nrhs)) {
    const size_t smem = (size_t)kNarrowWarps * L.max_m * 8;
    const unsigned g = (unsigned)((L.n_fronts + kNarrowWarps - 1) / kNarrowWarps);
    timer_begin(K_SOLVE_BWD_WAVE, st);
    if (L.max_k <= 32) {
      narrow_attr(solve_bwd_narrow<1>, smem);
      solve_bwd_narrow<1><<<g, 32 * kNarrowWarps, smem, st>>>(L, PA, has_parent, factors, x_parent,
                                                              parent_rows, x_out, out_rows, y, nrhs, 0);
    } else {
      narrow_attr(solve_bwd_narrow<2>, smem);
      solve_bwd_narrow<2><<<g, 32 * kNarrowWarps, smem, st>>>(L, PA, has_parent, factors, x_parent,
                                                              parent_rows, x_out, out_rows, y, nrhs, 0);
    }
    timer_end(st);
    return cudaGetLastError();
  }
  if (front_solve(L, nrhs, false)) {
    const size_t smem = (size_t)(L.max_m + 9 * TB) * 8;
    narrow_attr(solve_bwd_front, smem);
    timer_begin(K_SOLVE_BWD_WAVE, st);
    solve_bwd_front<<<(unsigned)L.n_fronts, 256, smem, st>>>(
        L, PA, has_parent, factors, x_parent, parent_rows, x_out, out_rows, y, nrhs, 0, nullptr, 0, 0);
    timer_end(st);
    return cudaGetLastError();
  }
  if (split_solve(L, nrhs, false)) {
    if (!work || work_doubles < solve_workspace_doubles(L, nrhs)) return cudaErrorInvalidValue;
    const int kcols = (L.max_k + TB - 1) / TB * TB;
    const int nch = std::max(1, (L.max_upd + kSplitRows - 1) / kSplitRows);
    timer_begin(K_SOLVE_BWD_WAVE, st);
    if (L.max_upd > 0)
      solve_bwd_split_rows<<<dim3((unsigned)L.n_fronts, (unsigned)nch, (unsigned)(kcols / TB)), 256, 0, st>>>(
          L, PA, has_parent, factors, x_parent, parent_rows, x_out, out_rows, work, nch, kcols, nrhs, 0);
    const size_t smem = (size_t)(L.max_m + 9 * TB) * 8;
    narrow_attr(solve_bwd_front, smem);
    solve_bwd_front<<<(unsigned)L.n_fronts, 256, smem, st>>>(
        L, PA, has_parent, factors, x_parent, parent_rows, x_out, out_rows, y, nrhs, 0, work, nch, kcols);
    timer_end(st);
    return cudaGetLastError();
  }
  if (!work || work_doubles < solve_workspace_doubles(L, nrhs)) return cudaErrorInvalidValue;
  const unsigned nf = (unsigned)L.n_fronts;
  const long long nW = (long long)L.max_m * nrhs;
  timer_begin(K_SOLVE_GATHER, st);
  solve_gather_bwd<<<dim3(nf, (unsigned)std::min<long long>((nW + 255) / 256, 1024)), 256, 0,
                     st>>>(L, PA, has_parent, x_parent, parent_rows, x_out, out_rows, y, nrhs);
  timer_end(st);
  const int nb = (L.max_k + TB - 1) / TB, rt = (L.max_m + TB - 1) / TB;
  if (nb == 0) return cudaGetLastError();
  const int cw = std::min(nrhs, kWaveCols);
  double* part = work;
  int* flags = reinterpret_cast<int*>(work + wave_blocks_doubles(L, nrhs));
  long long ntiles = 0;
  for (int b = 0; b < nb; b++) ntiles += (long long)L.n_fronts * (std::max(0, rt - b - 2) + 1);
  for (int col0 = 0; col0 < nrhs; col0 += cw) {
    const int nr = std::min(cw, nrhs - col0);
    const int nbuf = L.n_fronts <= wave_few_fronts(false) ? 2 : 1;
    const size_t smem = sizeof(double) * (nbuf * TB * TLD + 2 * TB * nr + 4 * TB);
    cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)L.n_fronts * nb * (1 + rt), st);
    timer_begin(K_SOLVE_BWD_WAVE, st);
    cudaError_t e;
    if (nr == 1) {
      const unsigned g = wave_grid(solve_bwd_wave<true>, smem, ntiles);
      e = launch_cooperative(solve_bwd_wave<true>, dim3(g), dim3(256), smem, st, L, factors, x_out,
                             out_rows, y, nr, nrhs, col0, flags, part, nb, rt, nbuf);
    } else {
      const unsigned g = wave_grid(solve_bwd_wave<false>, smem, ntiles);
      e = launch_cooperative(solve_bwd_wave<false>, dim3(g), dim3(256), smem, st, L, factors, x_out,
                             out_rows, y, nr, nrhs, col0, flags, part, nb, rt, nbuf);
    }
    timer_end(st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// Whether the level's sweep uses the cooperative wavefront kernels (the
// caller then keeps it off streams that run concurrently with other kernels).
int solve_cooperative(const LevelArgs& L, int nrhs, bool fwd) {
  if (!level_is_large(L.is_leaf, L.max_m)) return 0;
  if (narrow_solve(L, nrhs) || front_solve(L, nrhs, fwd) || split_solve(L, nrhs, fwd)) return 0;
  return L.max_k > 0 ? 1 : 0;
}

int solve_launches(const LevelArgs& L, int nrhs, bool fwd) {
  if (cols_solve_fwd(L, nrhs)) return (nrhs + 63) / 64;
  if (!level_is_large(L.is_leaf, L.max_m))
    return warp16_solve(L, nrhs) ? 1 : (nrhs + small_cols(L, nrhs) - 1) / small_cols(L, nrhs);
  if (narrow_solve(L, nrhs) || front_solve(L, nrhs, fwd)) return 1;
  if (split_solve(L, nrhs, fwd)) return fwd ? 2 : (L.max_upd > 0 ? 2 : 1);
  const int slices = (nrhs + kWaveCols - 1) / kWaveCols;
  if (fwd) return slices;
  return 1 + (L.max_k > 0 ? slices : 0);
}

// ------------------------------------------------------------- tiny trees
// The whole factorization and single-RHS solve of a small tree whose levels
// are all shared-memory levels (1D meshes, small 2D ones) in ONE launch of one
// CTA: there the ~3 launches per level, not the work, are the cost.  Per
// level the CTA's threads stride over its fronts, one thread per front
// (factor_front<1>, solve_*_small_front<1>: the level kernels' per-front code
// with a group of one), a CTA barrier between levels; the permutations to and
// from pivot order are in the same launch.
constexpr int kTreeMaxLevels = 24;
constexpr int kTreeThreads = 1024;  // at most; fewer when the fronts need more scratch
constexpr int kTreeMaxLeaves = 4096;
constexpr size_t kTreeSmemMax = 200 * 1024;
struct TreeArgs {
  LevelArgs lv[kTreeMaxLevels];
  double* fac[kTreeMaxLevels];
  int nlev;
  int fsmem;    // doubles per thread: factor front scratch
  int ssmem;    // doubles per thread: solve vector block
  int threads;  // CTA size
};

__global__ void __launch_bounds__(kTreeThreads)
    tree_small_kernel(TreeArgs A, const double* __restrict__ elem, double* upd0, double* upd1,
                      double thr, unsigned long long* err, const int* __restrict__ perm,
                      long long n_piv, long long n_dof, const double* b, double* x, double* y,
                      double* blk0, double* blk1, int do_factor, int do_solve) {
  extern __shared__ __align__(16) double tsm[];
  const int t = threadIdx.x, nt = blockDim.x;
  if (do_solve) {
    for (long long i = t; i < n_dof; i += nt) x[i] = b[i];  // DOFs outside every front
    for (long long i = t; i < n_piv; i += nt) y[i] = b[perm[i] - 1];
    __syncthreads();
  }
  // one phase per level: factor the level's fronts, then (same thread, same
  // fronts: its factors are its own writes) their forward sweep
  // separate scratch regions: a thread may run a front's forward sweep while
  // another still factors in the same phase
  double* F = tsm + (size_t)t * A.fsmem;
  unsigned char* ssm = reinterpret_cast<unsigned char*>(tsm + (size_t)nt * A.fsmem);
  const int per = A.ssmem * 8;
  for (int L = 0; L < A.nlev; L++) {
    const LevelArgs& lv = A.lv[L];
    if (do_factor) {
      const double* child = (L & 1) ? upd0 : upd1;  // level L-1 wrote upd[(L-1) & 1]
      double* out = (L & 1) ? upd1 : upd0;
      double* lvec = F + small_front_doubles(lv.max_m, lv.max_k) - lv.max_m;
      for (long long f = t; f < lv.n_fronts; f += nt) {
        const Shape S = front_shape(lv, f);
        const double* s0 = lv.is_leaf ? elem + f * lv.elem_stride
                                      : child + lv.child_slot(f, 0) * lv.child_upd_stride;
        const double* s1 =
            lv.is_leaf ? nullptr : child + lv.child_slot(f, 1) * lv.child_upd_stride;
        factor_front<1>(lv, f, S, s0, s1, elem, F, lvec, A.fac[L] + f * lv.fac_stride,
                        out + f * lv.upd_stride, thr, err, 0, 0, 1 << 30);
      }
    }
    if (do_solve) {
      const LevelArgs& C = A.lv[L > 0 ? L - 1 : 0];
      const double* w_child = ((L - 1) & 1) ? blk1 : blk0;
      double* w_out = (L & 1) ? blk1 : blk0;
      for (long long f = t; f < lv.n_fronts; f += nt)
        solve_fwd_small_front<1, kTreeThreads, false>(f, lv, C, A.fac[L], w_child, C.max_m, 1,
                                                     w_out, lv.max_m, y, 1, 1, 0, per, ssm);
    }
    __syncthreads();
  }
  if (!do_solve) return;
  for (int L = A.nlev - 1; L >= 0; L--) {
    const LevelArgs& lv = A.lv[L];
    const bool hp = L + 1 < A.nlev;
    const LevelArgs& PA = A.lv[hp ? L + 1 : L];
    const double* x_parent = ((L + 1) & 1) ? blk1 : blk0;
    double* x_out = (L & 1) ? blk1 : blk0;
    for (long long f = t; f < lv.n_fronts; f += nt)
      solve_bwd_small_front<1, kTreeThreads, false>(f, lv, PA, hp ? 1 : 0, A.fac[L], x_parent,
                                                   PA.max_m, x_out, lv.max_m, y, 1, 1, 0, per,
                                                   ssm);
    __syncthreads();
  }
  for (long long i = t; i < n_piv; i += nt) x[perm[i] - 1] = y[i];
}

// Shared memory of the tiny-tree kernel (0: the tree does not qualify).
size_t tree_small_smem(const LevelArgs* lv, int nlev, TreeArgs* A) {
  if (nlev < 1 || nlev > kTreeMaxLevels || lv[0].n_fronts > kTreeMaxLeaves) return 0;
  int fs = 0, ss = 0;
  for (int L = 0; L < nlev; L++) {
    if (level_is_large(lv[L].is_leaf, lv[L].max_m) || lv[L].front_base != 0 || !lv[L].factors)
      return 0;
    fs = std::max(fs, (small_front_doubles(lv[L].max_m, lv[L].max_k) + 1) & ~1);
    ss = std::max(ss, (lv[L].max_m + 1) & ~1);
  }
  // threads: one per leaf front when the scratch fits (levels have at most as
  // many fronts as the leaves), at least 256
  int nt = kTreeThreads;
  while (nt > 256 && ((size_t)nt * 8 * (fs + ss) > kTreeSmemMax || nt / 2 >= lv[0].n_fronts))
    nt /= 2;
  const size_t smem = (size_t)nt * 8 * (fs + ss);
  if (smem > kTreeSmemMax) return 0;
  if (A) {
    A->threads = nt;
    A->nlev = nlev;
    A->fsmem = fs;
    A->ssmem = ss;
    for (int L = 0; L < nlev; L++) {
      A->lv[L] = lv[L];
      A->fac[L] = const_cast<double*>(lv[L].factors);
    }
  }
  return smem;
}

cudaError_t launch_tree_small(const LevelArgs* lv, int nlev, const double* elem, double* upd0,
                              double* upd1, double thr, unsigned long long* err, const int* perm,
                              long long n_piv, long long n_dof, const double* b, double* x,
                              double* y, double* blk0, double* blk1, int do_factor, int do_solve,
                              cudaStream_t st) {
  TreeArgs A;
  const size_t smem = tree_small_smem(lv, nlev, &A);
  if (!smem) return cudaErrorInvalidValue;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(tree_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  timer_begin(K_SUBTREE, st);
  tree_small_kernel<<<1, A.threads, smem, st>>>(A, elem, upd0, upd1, thr, err, perm, n_piv,
                                                    n_dof, b, x, y, blk0, blk1, do_factor,
                                                    do_solve);
  timer_end(st);
  return cudaGetLastError();
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

cudaError_t set_jitter_solve(unsigned seed) { return set_jitter_tu(seed); }

}  // namespace tfb
