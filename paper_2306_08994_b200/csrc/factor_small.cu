// Small-front level kernel: extend-add + partial LDL^T + Schur complement,
// one thread group per front, the whole front resident in shared memory.
//
// Reference semantics replaced (per front, per pivot z in ascending order):
//   Division       q(z,y) = a(z,y) / a(z,z)          engine.py:86-93
//   Multiplication p = q(z,y) * a(x,z)               engine.py:94-100
//   Subtraction    a(x,y) -= p                       engine.py:101-105
//   zero pivot     |a(z,z)| <= 1e-14 * max|A|        engine.py:91-92, 529-530
// on the dense front in [eliminable | shared] order (NodeReorder,
// tasks.py:114-130).  The front is symmetric, so only its lower triangle is
// kept (packed, row-major) and l(x,z) = q(z,x) is stored once.
#include "common.cuh"

namespace tfb {

// Accumulate one source (element matrix or child Schur complement) into the
// packed front F through the source->front position map mp.
template <int G>
__device__ __forceinline__ void extend_add_src(double* F, const int* mp, int len, int ld,
                                               bool full_src, const double* __restrict__ src,
                                               int tid) {
  if (full_src) {  // element matrix, full len x len row-major (leading dim ld), lower triangle
    const int n = len * len;
    for (int e = tid; e < n; e += G) {
      int a = e / len, b = e - a * len;
      if (b > a) continue;
      int R = mp[a], C = mp[b];
      int hi = R > C ? R : C, lo = R > C ? C : R;
      F[tri(hi, lo)] += src[a * ld + b];
    }
  } else {  // packed lower child Schur complement
    const long long n = tri(len, 0);
    if (n == 0) return;
    long long e = tid;
    if (e >= n) return;
    int a = tri_row(e);
    int b = (int)(e - tri(a, 0));
    for (; e < n; e += G) {
      int R = mp[a], C = mp[b];
      int hi = R > C ? R : C, lo = R > C ? C : R;
      F[tri(hi, lo)] += src[e];
      b += G;
      while (b > a) { b -= a + 1; a++; }
    }
  }
}

template <int G, int GPC>
__global__ void __launch_bounds__(G* GPC)
    factor_small_kernel(LevelArgs L, const double* __restrict__ child_upd,
                        const double* __restrict__ elem, double* __restrict__ factors,
                        double* __restrict__ upd_out, double threshold,
                        unsigned long long* err, int smem_per_group) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / G;
  const int tid = threadIdx.x - gid * G;
  const int bar = 1 + gid;
  const long long f = (long long)blockIdx.x * GPC + gid;
  if (f >= L.n_fronts) return;  // whole group exits together
  unsigned char* my = smem_raw + (size_t)gid * smem_per_group;
  const int mm = L.max_m;
  double* F = reinterpret_cast<double*>(my);
  double* lv = F + tri(mm, 0);       // scaled column of the current pivot
  int* mp = reinterpret_cast<int*>(lv + mm);

  const int* P = L.pat + (size_t)L.pattern_of[f] * TF_PAT_WIDTH;
  const int m = P[TF_PAT_M], k = P[TF_PAT_K], nsrc = P[TF_PAT_NSRC];
  const int len0 = P[TF_PAT_LEN0], len1 = P[TF_PAT_LEN1];
  const long long nF = tri(m, 0);

  for (long long e = tid; e < nF; e += G) F[e] = 0.0;
  for (int t = tid; t < len0; t += G) mp[t] = L.maps[P[TF_PAT_OFF0] + t];
  for (int t = tid; t < len1; t += G) mp[len0 + t] = L.maps[P[TF_PAT_OFF1] + t];
  group_sync<G>(bar);
  if (L.is_leaf) {
    extend_add_src<G>(F, mp, len0, L.elem_ld, true, elem + f * L.elem_stride, tid);
  } else {
    extend_add_src<G>(F, mp, len0, 0, false, child_upd + (2 * f) * L.child_upd_stride, tid);
    if (nsrc == 2) {
      group_sync<G>(bar);  // fixed child order, no atomics
      extend_add_src<G>(F, mp + len0, len1, 0, false,
                        child_upd + (2 * f + 1) * L.child_upd_stride, tid);
    }
  }
  group_sync<G>(bar);

  const long long piv0 = L.piv_off[f];
  for (int c = 0; c < k; c++) {
    const double d = F[tri(c, c)];
    if (tid == 0 && fabs(d) <= threshold) record_zero_pivot(err, (unsigned long long)(piv0 + c));
    for (int r = c + 1 + tid; r < m; r += G) lv[r] = F[tri(r, c)] / d;
    group_sync<G>(bar);
    // trailing update of the packed triangle rows/cols (c, m)
    const int w = m - c - 1;
    const long long nT = tri(w, 0);
    if (tid < nT) {
      long long e = tid;
      int a = tri_row(e);
      int b = (int)(e - tri(a, 0));
      for (; e < nT; e += G) {
        const int r = c + 1 + a, s = c + 1 + b;
        F[tri(r, s)] -= lv[s] * F[tri(r, c)];
        b += G;
        while (b > a) { b -= a + 1; a++; }
      }
    }
    group_sync<G>(bar);
    for (int r = c + 1 + tid; r < m; r += G) F[tri(r, c)] = lv[r];
    group_sync<G>(bar);
  }

  // factor panel: row-major m x k, lower part (c <= r)
  if (k > 0) {
    double* out = factors + f * L.fac_stride;
    const long long n = (long long)m * k;
    for (long long e = tid; e < n; e += G) {
      int r = (int)(e / k), c = (int)(e - (long long)r * k);
      if (c <= r) out[e] = F[tri(r, c)];
    }
  }
  // Schur complement, packed lower (m-k)^2
  const int u = m - k;
  if (u > 0) {
    double* out = upd_out + f * L.upd_stride;
    for (int a = 0; a < u; a++) {
      const double* row = F + tri(k + a, k);
      double* orow = out + tri(a, 0);
      for (int b = tid; b <= a; b += G) orow[b] = row[b];
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
  int per = small_smem_per_group(L.max_m);
  size_t smem = (size_t)per * GPC;
  auto kern = factor_small_kernel<G, GPC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  long long blocks = (L.n_fronts + GPC - 1) / GPC;
  kern<<<(unsigned)blocks, G * GPC, smem, st>>>(L, child_upd, elem, factors, upd_out, thr, err,
                                                per);
  return cudaGetLastError();
}

cudaError_t launch_factor_small(const LevelArgs& L, const double* child_upd, const double* elem,
                                double* factors, double* upd_out, double thr,
                                unsigned long long* err, cudaStream_t st) {
  const int mm = L.max_m;
  if (mm <= 8) return launch_small_t<32, 8>(L, child_upd, elem, factors, upd_out, thr, err, st);
  if (mm <= 24) return launch_small_t<32, 4>(L, child_upd, elem, factors, upd_out, thr, err, st);
  if (mm <= 48) return launch_small_t<64, 2>(L, child_upd, elem, factors, upd_out, thr, err, st);
  if (mm <= 96) return launch_small_t<128, 1>(L, child_upd, elem, factors, upd_out, thr, err, st);
  return launch_small_t<256, 1>(L, child_upd, elem, factors, upd_out, thr, err, st);
}

}  // namespace tfb
