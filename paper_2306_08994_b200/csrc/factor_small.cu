// Small-front level kernel: extend-add + partial LDL^T + Schur complement,
// one thread group per front (G threads, GPC fronts per CTA), the whole front
// resident in shared memory.
//
// Reference semantics replaced (per front, per pivot z in ascending order):
//   Division       q(z,y) = a(z,y) / a(z,z)          engine.py:86-93
//   Multiplication p = q(z,y) * a(x,z)               engine.py:94-100
//   Subtraction    a(x,y) -= p                       engine.py:101-105
//   zero pivot     |a(z,z)| <= 1e-14 * max|A|        engine.py:91-92, 529-530
// on the dense front in [eliminable | shared] order (NodeReorder,
// tasks.py:114-130).  The front is symmetric, so only its lower triangle is
// kept (packed, row-major) and l(x,z) = q(z,x) is stored once.
//
// Output per front: factor slot = panel P (m x kp row-major; P[r][c] = l(r,c)
// for r > c, P[c][c] = d_c) followed by d (kp doubles); update slot = packed
// lower (m-k)^2 Schur complement.
#include "common.cuh"

namespace tfb {

template <int G, int GPC>
__global__ void __launch_bounds__(G* GPC)
    factor_small_kernel(LevelArgs L, const double* __restrict__ child_upd,
                        const double* __restrict__ elem, double* __restrict__ factors,
                        double* __restrict__ upd_out, double threshold,
                        unsigned long long* err, int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / G;
  const int t = threadIdx.x - gid * G;
  const int bar = 1 + gid;
  const long long f = (long long)blockIdx.x * GPC + gid;
  if (f >= L.n_fronts) return;  // whole group exits; syncs are group-local
  unsigned char* my = smem_raw + (size_t)gid * smem_per_group;
  const int mm = L.max_m;
  double* F = reinterpret_cast<double*>(my);
  double* lv = F + tri(mm, 0);
  int* mp = reinterpret_cast<int*>(lv + mm);

  const Shape S = front_shape(L, f);
  const int m = S.m, k = S.k, kp = S.kp;
  const int nF = (int)tri(m, 0);

  for (int e = t; e < nF; e += G) F[e] = 0.0;
  for (int i = t; i < S.len0; i += G) mp[i] = L.maps[S.off0 + i];
  for (int i = t; i < S.len1; i += G) mp[S.len0 + i] = L.maps[S.off1 + i];
  group_sync<G>(bar);

  // extend-add: each source entry read once (coalesced), scattered into F;
  // sources in fixed order, no atomics.
  for (int c = 0; c < S.nsrc; c++) {
    const int len = c == 0 ? S.len0 : S.len1;
    const int* cm = mp + (c == 0 ? 0 : S.len0);
    const int n = (int)tri(len, 0);
    if (L.is_leaf) {
      const double* E = elem + f * L.elem_stride;
      for (int e = t; e < n; e += G) {
        const int a = tri_row(e), b = e - (int)tri(a, 0);
        const int R = cm[a], C = cm[b];
        F[R > C ? tri(R, C) : tri(C, R)] += E[a * L.elem_ld + b];
      }
    } else {
      const double* src = child_upd + (2 * f + c) * L.child_upd_stride;
      for (int e = t; e < n; e += G) {
        const int a = tri_row(e), b = e - (int)tri(a, 0);
        const int R = cm[a], C = cm[b];
        F[R > C ? tri(R, C) : tri(C, R)] += src[e];
      }
    }
    group_sync<G>(bar);
  }

  // partial LDL^T of the k eliminable pivots (right-looking, rank 1 per pivot)
  const long long piv0 = L.piv_off[f];
  for (int c = 0; c < k; c++) {
    const double d = F[tri(c, c)];
    if (t == 0 && fabs(d) <= threshold) record_zero_pivot(err, (unsigned long long)(piv0 + c));
    for (int r = c + 1 + t; r < m; r += G) lv[r] = F[tri(r, c)] / d;
    group_sync<G>(bar);
    if constexpr (G >= 32) {
      const int warp = t >> 5, lane = t & 31;
      for (int r = c + 1 + warp; r < m; r += G / 32) {
        double* row = F + tri(r, 0);
        const double frc = row[c];
        for (int s = c + 1 + lane; s <= r; s += 32) row[s] -= lv[s] * frc;
        __syncwarp();
        if (lane == 0) row[c] = lv[r];
      }
    } else {
      for (int r = c + 1 + t; r < m; r += G) {
        double* row = F + tri(r, 0);
        const double frc = row[c];
        for (int s = c + 1; s <= r; s++) row[s] -= lv[s] * frc;
        row[c] = lv[r];
      }
    }
    group_sync<G>(bar);
  }

  // factor slot: panel rows (lower part) + diagonal vector
  if (k > 0) {
    double* out = factors + f * L.fac_stride;
    const int n = m * k;
    for (int e = t; e < n; e += G) {
      const int r = e / k, c = e - r * k;
      if (c <= r) out[(long long)r * kp + c] = F[tri(r, c)];
    }
    double* dv = out + (long long)m * kp;
    for (int c = t; c < kp; c += G) dv[c] = c < k ? F[tri(c, c)] : 0.0;
  }
  // Schur complement, packed lower (m-k)^2
  const int u = m - k;
  if (u > 0) {
    double* out = upd_out + f * L.upd_stride;
    const int n = (int)tri(u, 0);
    for (int e = t; e < n; e += G) {
      const int a = tri_row(e), b = e - (int)tri(a, 0);
      out[e] = F[tri(k + a, k + b)];
    }
  }
}

int small_smem_per_group(int max_m) {
  size_t bytes = sizeof(double) * ((size_t)max_m * (max_m + 1) / 2 + max_m) +
                 sizeof(int) * 2 * (size_t)max_m;
  bytes = (bytes + 15) & ~(size_t)15;
  return (int)bytes;
}

template <int G, int GPC>
static cudaError_t launch_small_t(const LevelArgs& L, const double* child_upd, const double* elem,
                                  double* factors, double* upd_out, double thr,
                                  unsigned long long* err, cudaStream_t st) {
  const int per = small_smem_per_group(L.max_m);
  // fronts per CTA: GPC, reduced when shared memory would not fit
  int gpc = GPC;
  while (gpc > 1 && (size_t)per * gpc > 200 * 1024) gpc >>= 1;
  if (gpc != GPC) return cudaErrorInvalidConfiguration;
  const size_t smem = (size_t)per * GPC;
  auto kern = factor_small_kernel<G, GPC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long blocks = (L.n_fronts + GPC - 1) / GPC;
  kern<<<(unsigned)blocks, G * GPC, smem, st>>>(L, child_upd, elem, factors, upd_out, thr, err,
                                                per);
  return cudaGetLastError();
}

cudaError_t launch_factor_small(const LevelArgs& L, const double* child_upd, const double* elem,
                                double* factors, double* upd_out, double thr,
                                unsigned long long* err, cudaStream_t st) {
  const int mm = L.max_m;
  if (mm <= 8) return launch_small_t<4, 64>(L, child_upd, elem, factors, upd_out, thr, err, st);
  if (mm <= 16) return launch_small_t<8, 32>(L, child_upd, elem, factors, upd_out, thr, err, st);
  if (mm <= 32) return launch_small_t<16, 8>(L, child_upd, elem, factors, upd_out, thr, err, st);
  if (mm <= 64) return launch_small_t<32, 4>(L, child_upd, elem, factors, upd_out, thr, err, st);
  if (mm <= 128) return launch_small_t<128, 1>(L, child_upd, elem, factors, upd_out, thr, err, st);
  return launch_small_t<256, 1>(L, child_upd, elem, factors, upd_out, thr, err, st);
}

}  // namespace tfb
