// One small front factored by one thread group in shared memory
// (factor_front): shared by the level kernel (factor_small.cu) and the
// whole-tree kernel for tiny trees (solve.cu).
#pragma once
#include "common.cuh"

namespace tfb {

// Shared-memory front layout (tri(m) + (m-k)(kp+1-k) doubles):
//   rows r < k  : packed lower triangle, F[tri(r) + c]             (pivot block)
//   rows r >= k : rows of odd stride ks = kp+1 (bank-conflict-free column
//                 access), F[tri(k) + (r-k) ks + c]                (L21)
//   Schur block : packed lower tri(m-k) at tri(k) + (m-k) ks  (the update
//                 slot's layout: copies out contiguously)
// The extend-add targets come from the pattern's scatter table
// (symbolic.cpp): entry e of source c lands at F[scat[e]].
__host__ __device__ inline int small_front_doubles(int max_m, int max_k) {
  (void)max_k;
  return (int)tri32(max_m, 0) + 4 * max_m + max_m;  // + pivot/column scratch
}

// Thread t's contiguous chunk [beg, end) of n items split over G threads.
__device__ __forceinline__ void chunk_of(int n, int G, int t, int& beg, int& end) {
  const int c = (n + G - 1) / G;
  beg = min(n, t * c);
  end = min(n, beg + c);
}

// Pivots of leaf child c of level-1 front f (leaf pass-through, leaf_direct).
__device__ __forceinline__ int leaf_child_k(const LevelArgs& L, long long f, int c) {
  const long long ch = L.child_slot(f, c);
  return L.src_pat[(size_t)L.src_pattern_of[ch] * TF_PAT_WIDTH + TF_PAT_K];
}

// One front, one thread group: extend-add of src0/src1 (packed child Schur
// blocks, or the element matrix at the leaves), partial LDL^T, Schur block,
// copy-out of the factor slot and of the packed update to upd_dst.
template <int G>
__device__ __forceinline__ void factor_front(const LevelArgs& L, long long f, const Shape& S,
                                             const double* __restrict__ src0,
                                             const double* __restrict__ src1,
                                             const double* __restrict__ elem, double* F,
                                             double* lv, double* __restrict__ fac_out,
                                             double* __restrict__ upd_dst, double threshold,
                                             unsigned long long* err, int t, int bar,
                                             int fs_k = 16) {
  const int m = S.m, k = S.k, kp = S.kp, u = m - k;
  // leaf pass-through: a leaf without pivots writes nothing; level 1 reads its
  // element matrix instead of its update (tf_level_view.leaf_direct)
  if (L.is_leaf && L.leaf_direct && k == 0) return;
  const int ks = kp + 1, tk = (int)tri32(k, 0), nS = (int)tri32(u, 0), s0 = tk + u * ks;
  double* Sb = F + s0;
  auto rowp = [&](int r) { return r < k ? (int)tri32(r, 0) : tk + (r - k) * ks; };
  {  // zero the front: 16-byte stores (F is 16-byte aligned), odd tail scalar
    const int n2 = (s0 + nS) >> 1;
    double2* F2 = reinterpret_cast<double2*>(F);
    for (int e = t; e < n2; e += G) F2[e] = make_double2(0.0, 0.0);
    if (t == 0 && ((s0 + nS) & 1)) F[s0 + nS - 1] = 0.0;
  }
  group_sync<G>(bar);

  // (1) extend-add through the scatter table: sources in fixed order, no atomics
  const int* sc = L.maps + L.pat[(size_t)L.pattern_of[f] * TF_PAT_WIDTH + TF_PAT_SOFF];
  for (int c = 0; c < S.nsrc; c++) {
    const int len = c == 0 ? S.len0 : S.len1;
    const int n = (int)tri32(len, 0);
    const int* scc = sc + (c == 0 ? 0 : (int)tri32(S.len0, 0));
    if (L.is_leaf) {  // dense len x len element matrix, lower part
      int beg, end;
      chunk_of(n, G, t, beg, end);
      if (beg < end) {
        int a = tri_row32(beg), b = beg - (int)tri32(a, 0);
        for (int e = beg; e < end; e++) {
          F[__ldg(scc + e)] += src0[a * L.elem_ld + b];
          if (++b > a) { a++; b = 0; }
        }
      }
    } else if (L.leaf_direct && leaf_child_k(L, f, c) == 0) {
      // pivot-free leaf child: entry e of its update is the element-matrix
      // entry di[e] (src_maps: per leaf pattern, packed update index ->
      // element index, lower part) -- exactly what the leaf would have written
      const long long ch = L.child_slot(f, c);
      const int* di = L.src_maps + L.src_maps[L.src_pattern_of[ch]];
      const double* E = elem + ch * L.elem_stride;
      int e = t;
      for (; e + 3 * G < n; e += 4 * G) {
        int p[4];
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          p[q] = __ldg(scc + e + q * G);
          v[q] = E[__ldg(di + e + q * G)];
        }
#pragma unroll
        for (int q = 0; q < 4; q++) F[p[q]] += v[q];
      }
      for (; e < n; e += G) F[__ldg(scc + e)] += E[__ldg(di + e)];
    } else {
      const double* src = c == 0 ? src0 : src1;
      int e = t;
      for (; e + 3 * G < n; e += 4 * G) {  // four entries per thread in flight
        int p[4];
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          p[q] = __ldg(scc + e + q * G);
          v[q] = src[e + q * G];
        }
#pragma unroll
        for (int q = 0; q < 4; q++) F[p[q]] += v[q];
      }
      if (e < n) {  // remainder: up to four entries per thread, loads first
        int p[4];
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const bool ok = e + q * G < n;
          p[q] = ok ? __ldg(scc + e + q * G) : -1;
          v[q] = ok ? src[e + q * G] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (p[q] >= 0) F[p[q]] += v[q];
      }
    }
    group_sync<G>(bar);
  }

  // (2) panel.  Wide groups (G >= 32) with k >= fs_k (TFB_SMALL_FSK, measured):
  // (a) the k x k pivot block, right-looking with unscaled columns (one
  // barrier per pivot), scaled to l; (b) every L21 row independently (no
  // barriers): forward substitution against L11, u_rc = a_rc - sum_{q<c}
  // u_rq l(c,q), then l(r,c) = u_rc / d_c.
  if constexpr (G >= 32) {
    if (k >= fs_k) {
      const long long piv0 = L.piv_off[f];
      for (int c = 0; c < k; c++) {
        const double d = F[tri32(c, c)];
        if (t == 0 && fabs(d) <= threshold) record_zero_pivot(err, (unsigned long long)(piv0 + c));
        const double dinv = 1.0 / d;
        for (int r = c + 1 + t; r < k; r += G) {
          double* row = F + tri32(r, 0);
          const double lrc = row[c] * dinv;
          int qc = tri32(c + 1, c);  // F[tri32(q, c)], stepped by q + 1
          for (int q = c + 1; q <= r; qc += ++q) row[q] -= lrc * F[qc];
        }
        group_sync<G>(bar);
      }
      for (int c = t; c < k; c += G) lv[c] = 1.0 / F[tri32(c, c)];
      group_sync<G>(bar);
      for (int r = 1 + t; r < k; r += G) {
        double* row = F + tri32(r, 0);
        for (int c = 0; c < r; c++) row[c] *= lv[c];
      }
      group_sync<G>(bar);
      for (int r = k + t; r < m; r += G) {
        double* row = F + rowp(r);
        for (int c = 1; c < k; c++) {
          const double* lc = F + tri32(c, 0);
          double u = row[c];
          for (int q = 0; q < c; q++) u -= row[q] * lc[q];
          row[c] = u;
        }
        for (int c = 0; c < k; c++) row[c] *= lv[c];
      }
      group_sync<G>(bar);
      goto schur;
    }
  }
  {
  // (2) panel: right-looking over the k pivot columns, updates confined to
  // them, columns kept unscaled during the sweep (a(r,q) -= a(r,c) a(q,c) / d_c
  // reads only finished column-c entries: one barrier per pivot), then scaled.
  const long long piv0 = L.piv_off[f];
  for (int c = 0; c < k; c++) {
    const double d = F[tri32(c, c)];
    if (t == 0 && fabs(d) <= threshold) record_zero_pivot(err, (unsigned long long)(piv0 + c));
    const double dinv = 1.0 / d;
    for (int r = c + 1 + t; r < m; r += G) {
      double* row = F + rowp(r);
      const double lrc = row[c] * dinv;
      const int smax = min(r, k - 1);
      int qc = tri32(c + 1, c);  // F[tri32(q, c)], stepped by q + 1
      for (int q = c + 1; q <= smax; qc += ++q) row[q] -= lrc * F[qc];
    }
    group_sync<G>(bar);
  }
  if (k > 0) {
    for (int c = t; c < k; c += G) lv[c] = 1.0 / F[tri32(c, c)];
    group_sync<G>(bar);
    for (int r = 1 + t; r < m; r += G) {  // l(r, c) = a(r, c) / d_c
      double* row = F + rowp(r);
      const int cm = min(r, k);
      for (int c = 0; c < cm; c++) row[c] *= lv[c];
    }
    group_sync<G>(bar);
  }

  }
schur:
  // (3) Schur block: S[i][j] -= sum_q L21[i][q] d_q L21[j][q], i >= j
  if (k > 0 && u > 0) {
    for (int c = t; c < k; c += G) lv[c] = F[tri32(c, c)];  // pivots
    group_sync<G>(bar);
    const double* P21 = F + tk;
    if constexpr (G >= 32) {
      // a warp takes whole rows I of 8x8 tiles (rows I and T-1-I paired, so
      // every pair has T+1 tiles): the row's A fragments (L21 D, k/4 DMMA
      // steps) are loaded once and reused for its tiles J <= I
      constexpr int KS = 4;  // k <= 16 in register fragments, longer k streamed
      const int warp = t >> 5, lane = t & 31, g8 = lane >> 2, tq = lane & 3;
      const int T = (u + 7) >> 3, nw = G / 32;
      auto tile_row = [&](int I) {
        const int ia = 8 * I + g8;
        const double* arow = P21 + min(ia, u - 1) * ks;
        const bool va = ia < u;
        double af[KS];
#pragma unroll
        for (int s4 = 0; s4 < KS; s4++) {
          const int q = 4 * s4 + tq;
          af[s4] = (va && q < k) ? arow[q] * lv[q] : 0.0;
        }
        for (int J = 0; J <= I; J++) {
          const int ib = 8 * J + g8;
          const double* brow = P21 + min(ib, u - 1) * ks;
          const bool vb = ib < u;
          double acc[2] = {0.0, 0.0};
#pragma unroll
          for (int s4 = 0; s4 < KS; s4++) {
            if (4 * s4 < k) {
              const int q = 4 * s4 + tq;
              dmma884(acc, af[s4], (vb && q < k) ? brow[q] : 0.0);
            }
          }
          for (int kk = 4 * KS; kk < k; kk += 4) {
            const int q = kk + tq;
            const double av = (va && q < k) ? arow[q] * lv[q] : 0.0;
            dmma884(acc, av, (vb && q < k) ? brow[q] : 0.0);
          }
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int jc = 8 * J + 2 * tq + h;
            if (ia < u && jc <= ia) Sb[tri32(ia, jc)] -= acc[h];
          }
        }
      };
      for (int pr = warp; pr < (T + 1) / 2; pr += nw) {
        tile_row(pr);
        if (T - 1 - pr != pr) tile_row(T - 1 - pr);
      }
    } else {
      int beg, end;
      chunk_of(nS, G, t, beg, end);
      if (beg < end) {
        int a = tri_row32(beg), b = beg - (int)tri32(a, 0);
        if (k <= 4) {
          // row a's scaled entries l(a,q) d_q stay in registers while the
          // thread's contiguous chunk walks along the row (same products and
          // summation order as below)
          double wa[4];
          auto load_row = [&](int r) {
            const double* ra = P21 + r * ks;
#pragma unroll
            for (int q = 0; q < 4; q++) wa[q] = q < k ? ra[q] * lv[q] : 0.0;
          };
          load_row(a);
          for (int e = beg; e < end; e++) {
            const double* rb = P21 + b * ks;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < 4; q++)
              if (q < k) acc += wa[q] * rb[q];
            Sb[e] -= acc;
            if (++b > a) {
              a++;
              b = 0;
              if (e + 1 < end) load_row(a);
            }
          }
        } else {
          for (int e = beg; e < end; e++) {
            const double* ra = P21 + a * ks;
            const double* rb = P21 + b * ks;
            double acc = 0.0;
            for (int q = 0; q < k; q++) acc += ra[q] * lv[q] * rb[q];
            Sb[e] -= acc;
            if (++b > a) { a++; b = 0; }
          }
        }
      }
    }
    group_sync<G>(bar);
  }

  // (4) copy-out: factor slot (panel m x kp + pivots) and the packed Schur block
  if (k > 0) {
    for (int e = t; e < k * kp; e += G) {  // pivot block rows: packed -> dense
      const int r = e / kp, c = e - r * kp;
      fac_out[e] = c <= r ? F[tri32(r, c)] : 0.0;
    }
    for (int e = t; e < u * kp; e += G) {  // L21 rows: stride ks -> kp
      const int r = e / kp, c = e - r * kp;
      fac_out[k * kp + e] = F[tk + r * ks + c];
    }
    for (int c = t; c < kp; c += G) fac_out[m * kp + c] = c < k ? F[tri32(c, c)] : 0.0;
  }
  for (int e = t; e < nS; e += G) upd_dst[e] = Sb[e];
}

}  // namespace tfb
