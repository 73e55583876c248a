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
// Phases: (1) extend-add of the sources, each thread streaming one contiguous
// chunk of a source's packed triangle; (2) right-looking factorization of the
// k pivot columns only (panel); (3) the Schur block S -= L21 D L21^T in one
// pass -- FP64 tensor-core MMA (mma.sync m8n8k4, 8x8 tiles per warp) when
// the group is at least a warp, FMA otherwise; (4) contiguous copy-out.
//
// Output per front: factor slot = panel P (m x kp row-major; P[r][c] = l(r,c)
// for r > c, P[c][c] = d_c) followed by d (kp doubles); update slot = packed
// lower (m-k)^2 Schur complement.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "front_small.cuh"

namespace tfb {

int small_smem_per_group(int max_m, int max_k) {
  return (int)((sizeof(double) * (size_t)small_front_doubles(max_m, max_k) + 15) & ~(size_t)15);
}

// Per-group stride of the level kernel (bytes): a group of G < 16 threads
// touches G consecutive doubles at a time, so the groups of a warp are
// staggered by G double-banks (stride = G mod 16 doubles) and together cover
// all 16 banks -- with a stride that is a multiple of 16 doubles they would
// pile onto the same G banks (measured: 50% excess shared wavefronts).
static int small_group_stride(int max_m, int max_k, int G) {
  int d = (small_smem_per_group(max_m, max_k) + 7) / 8;  // doubles, even
  if (G < 16)
    while ((d & 15) != (G & 15)) d += 2;
  return d * 8;
}

template <int G, int GPC>
__global__ void __launch_bounds__(G* GPC)
    factor_small_kernel(LevelArgs L, const double* __restrict__ child_upd,
                        const double* __restrict__ elem, double* __restrict__ factors,
                        double* __restrict__ upd_out, double threshold,
                        unsigned long long* err, int smem_per_group, int fs_k) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / G;
  const int t = threadIdx.x - gid * G;
  unsigned char* my = smem_raw + (size_t)gid * smem_per_group;
  double* F = reinterpret_cast<double*>(my);
  double* lv = F + small_front_doubles(L.max_m, L.max_k) - L.max_m;
  // grid-stride over fronts (the grid covers the level except on pass-through
  // leaf levels, where most fronts return at once); syncs are group-local
  for (long long f = (long long)blockIdx.x * GPC + gid; f < L.n_fronts;
       f += (long long)gridDim.x * GPC) {
    const Shape S = front_shape(L, f);
    const double* s0 = L.is_leaf ? elem + f * L.elem_stride
                                 : child_upd + L.child_slot(f, 0) * L.child_upd_stride;
    const double* s1 = L.is_leaf ? nullptr : child_upd + L.child_slot(f, 1) * L.child_upd_stride;
    factor_front<G>(L, f, S, s0, s1, elem, F, lv, factors + f * L.fac_stride,
                    upd_out + f * L.upd_stride, threshold, err, t, 1 + gid, fs_k);
  }
}

template <int G, int GPC>
static cudaError_t launch_small_t(const LevelArgs& L, const double* child_upd, const double* elem,
                                  double* factors, double* upd_out, double thr,
                                  unsigned long long* err, cudaStream_t st) {
  const int per = small_group_stride(L.max_m, L.max_k, G);
  const size_t smem = (size_t)per * GPC;
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  auto kern = factor_small_kernel<G, GPC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long blocks = (L.n_fronts + GPC - 1) / GPC;
  timer_begin(K_SMALL, st);
  static int fs_k = -1;
  if (fs_k < 0) {
    const char* e = getenv("TFB_SMALL_FSK");
    fs_k = e ? atoi(e) : 16;
  }
  // pass-through leaves: nearly every front returns at once, so a few resident
  // waves of CTAs stride over the level instead of one CTA per GPC fronts
  const long long grid = (L.is_leaf && L.leaf_direct) ? std::min(blocks, 148LL * 16) : blocks;
  kern<<<(unsigned)grid, G * GPC, smem, st>>>(L, child_upd, elem, factors, upd_out, thr, err,
                                              per, fs_k);
  timer_end(st);
  return cudaGetLastError();
}

cudaError_t launch_factor_small(const LevelArgs& L, const double* child_upd, const double* elem,
                                double* factors, double* upd_out, double thr,
                                unsigned long long* err, cudaStream_t st) {
  // groups sized so that a CTA's shared memory stays small enough for several
  // CTAs per SM (occupancy hides the shared-memory latency of the pivot loop)
  // (G, GPC) per front-order class m <= 4, 8, 16, 24, 48, 80, 232 (measured
  // on B200, tools/small_sweep.sh); TFB_SMALL_CFG="G:GPC,..." overrides
  static int cfg[7][2] = {{2, 128}, {4, 64}, {8, 16}, {16, 16}, {32, 4}, {128, 1}, {256, 1}};
  static bool parsed = false;
  if (!parsed) {
    parsed = true;
    if (const char* e = getenv("TFB_SMALL_CFG")) {
      for (int i = 0; i < 7 && *e; i++) {
        int g = 0, n = 0;
        if (sscanf(e, "%d:%d", &g, &n) == 2) { cfg[i][0] = g; cfg[i][1] = n; }
        while (*e && *e != ',') e++;
        if (*e == ',') e++;
      }
    }
  }
  const int mm = L.max_m;
  const int cls =
      mm <= 4 ? 0 : mm <= 8 ? 1 : mm <= 16 ? 2 : mm <= 24 ? 3 : mm <= 48 ? 4 : mm <= 80 ? 5 : 6;
  const int G = cfg[cls][0], GPC = cfg[cls][1];
#define TFB_CASE(g, n) \
  if (G == g && GPC == n) return launch_small_t<g, n>(L, child_upd, elem, factors, upd_out, thr, err, st);
  TFB_CASE(2, 128) TFB_CASE(4, 64) TFB_CASE(4, 32) TFB_CASE(8, 32) TFB_CASE(8, 16)
  TFB_CASE(16, 16) TFB_CASE(16, 8) TFB_CASE(32, 8) TFB_CASE(32, 4) TFB_CASE(32, 2)
  TFB_CASE(64, 4) TFB_CASE(64, 2) TFB_CASE(64, 1) TFB_CASE(128, 2) TFB_CASE(128, 1)
  TFB_CASE(256, 1)
#undef TFB_CASE
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- subtrees
// Levels 0..S-1 fused: each thread group (G = 8 threads) owns one subtree,
// rooted at a level-(S-1) front, and factors its fronts level by level; the
// packed updates between the fused levels stay in the group's shared-memory
// arenas, so only the factor slots and the level-(S-1) updates reach HBM.
// 32 groups per CTA keep many independent subtrees in flight per SM.
constexpr int kMaxFuse = 10;
constexpr int kSubG = 8, kSubNG = 32;
struct SubtreeArgs {
  int nlev;
  int arena_doubles[2];  // per group
  int ws_bytes;          // per group
  LevelArgs lv[kMaxFuse];
  double* fac[kMaxFuse];
};

__global__ void __launch_bounds__(kSubG* kSubNG) factor_subtree_kernel(
    SubtreeArgs A, const double* __restrict__ elem, double* __restrict__ upd_out,
    double threshold, unsigned long long* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gid = threadIdx.x / kSubG, t = threadIdx.x - gid * kSubG;
  const int top = A.nlev - 1;
  const long long root = (long long)blockIdx.x * kSubNG + gid;
  if (root >= A.lv[top].n_fronts) return;  // group-local exit
  const size_t per = sizeof(double) * (A.arena_doubles[0] + A.arena_doubles[1]) + A.ws_bytes;
  unsigned char* mine = smem_raw + (size_t)gid * per;
  double* arena[2] = {reinterpret_cast<double*>(mine),
                      reinterpret_cast<double*>(mine) + A.arena_doubles[0]};
  unsigned char* ws = mine + sizeof(double) * (A.arena_doubles[0] + A.arena_doubles[1]);
  for (int L = 0; L < A.nlev; L++) {
    const LevelArgs& lv = A.lv[L];
    double* F = reinterpret_cast<double*>(ws);
    double* lvec = F + small_front_doubles(lv.max_m, lv.max_k) - lv.max_m;
    double* prev = arena[(L + 1) & 1];
    double* cur = arena[L & 1];
    const int cst = L > 0 ? (int)tri32(A.lv[L - 1].max_upd, 0) : 0;
    const int ost = (int)tri32(lv.max_upd, 0);
    const long long base = root << (top - L);
    const long long cnt = min((long long)1 << (top - L), (long long)lv.n_fronts - base);
    for (long long i = 0; i < cnt; i++) {
      const long long f = base + i;
      const Shape S = front_shape(lv, f);
      const double* s0 = lv.is_leaf ? elem + f * lv.elem_stride : prev + (2 * i) * cst;
      const double* s1 = lv.is_leaf ? nullptr : prev + (2 * i + 1) * cst;
      double* dst = L == top ? upd_out + f * lv.upd_stride : cur + i * ost;
      factor_front<kSubG>(lv, f, S, s0, s1, elem, F, lvec, A.fac[L] + f * lv.fac_stride, dst,
                          threshold, err, t, 0);
      group_sync<kSubG>(0);
    }
  }
}

// Shared-memory plan of one subtree group; 0 when the levels cannot be fused.
static size_t subtree_group_bytes(const LevelArgs* lv, int nlev, int arena[2], int* ws) {
  int ws_max = 16;
  arena[0] = arena[1] = 0;
  for (int L = 0; L < nlev; L++) {
    ws_max = std::max(ws_max, small_smem_per_group(lv[L].max_m, lv[L].max_k));
    if (L < nlev - 1) {
      const int nf = 1 << (nlev - 1 - L);
      arena[L & 1] = std::max(arena[L & 1], nf * (int)tri32(lv[L].max_upd, 0));
    }
  }
  arena[0] = (arena[0] + 1) & ~1;
  arena[1] = (arena[1] + 1) & ~1;
  *ws = ws_max;
  return sizeof(double) * (arena[0] + arena[1]) + *ws;
}

int subtree_fusable_levels(const LevelArgs* lv, int n_levels) {
  int best = 0;
  for (int S = 2; S <= std::min(n_levels, kMaxFuse); S++) {
    bool ok = true;
    for (int L = 0; L < S; L++)
      ok = ok && lv[L].max_m <= 16 && !level_is_large(lv[L].is_leaf, lv[L].max_m);
    if (!ok) break;
    int ar[2], ws;
    if (subtree_group_bytes(lv, S, ar, &ws) * kSubNG > 200 * 1024) break;
    best = S;
  }
  return best;
}

cudaError_t launch_factor_subtree(const LevelArgs* lv, int nlev, double* const* fac,
                                  const double* elem, double* upd_out, double thr,
                                  unsigned long long* err, cudaStream_t st) {
  if (nlev < 1 || nlev > kMaxFuse) return cudaErrorInvalidValue;
  SubtreeArgs A;
  A.nlev = nlev;
  for (int L = 0; L < nlev; L++) {
    A.lv[L] = lv[L];
    A.fac[L] = fac[L];
  }
  const size_t per = subtree_group_bytes(lv, nlev, A.arena_doubles, &A.ws_bytes);
  const size_t smem = per * kSubNG;
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(factor_subtree_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long roots = lv[nlev - 1].n_fronts;
  const unsigned blocks = (unsigned)((roots + kSubNG - 1) / kSubNG);
  timer_begin(K_SUBTREE, st);
  factor_subtree_kernel<<<blocks, kSubG * kSubNG, smem, st>>>(A, elem, upd_out, thr, err);
  timer_end(st);
  return cudaGetLastError();
}

}  // namespace tfb
