// Shared device helpers for the level kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>

#include "tracefront_b200.h"

namespace tfb {

// Fronts up to this order are factored entirely in one SM's shared memory.
constexpr int kSmallMaxM = 232;
// Runtime threshold (<= kSmallMaxM) between the shared-memory and the blocked
// large-front paths; lowered by tests to drive the large path on small meshes.
extern int g_small_max_m;
// Per-front doubles of the diagonal-block inverses a large-front level keeps.
long long large_aux_doubles(int max_k);
inline bool level_is_large(int is_leaf, int max_m) { return !is_leaf && max_m > g_small_max_m; }

// Persistent kernels whose CTAs wait on each other (wavefront solves, root
// dataflow) are launched cooperatively: the runtime either makes the whole
// grid co-resident or fails the launch (cudaErrorCooperativeLaunchTooLarge),
// so a spin-wait can never depend on a CTA that is not scheduled (MPS,
// concurrent kernels).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_cooperative(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


// Kernel classes for the optional launch timing (timing.cu).
enum KernelClass {
  K_SMALL = 0, K_SUBTREE, K_ASSEMBLE, K_DIAG, K_BLOCK, K_TRSM, K_PANEL, K_SCHUR, K_FINALIZE,
  K_SOLVE_SMALL_FWD, K_SOLVE_SMALL_BWD, K_SOLVE_GATHER, K_SOLVE_FWD_WAVE, K_SOLVE_BWD_WAVE,
  K_PERMUTE, K_ROOT, K_COUNT
};
void timer_begin(int cls, cudaStream_t st);
void timer_end(cudaStream_t st);

// Kernel-side copy of tf_level_view (passed by value).
struct LevelArgs {
  int n_fronts;
  int is_leaf;
  int elem_ld;
  int max_m;
  int max_k;
  int max_upd;
  long long fac_stride;
  long long upd_stride;
  long long child_upd_stride;
  long long elem_stride;
  const int* __restrict__ pattern_of;
  const long long* __restrict__ piv_off;
  const int* __restrict__ pat;
  const int* __restrict__ maps;
  double* aux;
  long long aux_stride;
  long long front_base;  // tree index of front 0 of this (possibly sliced) view
  long long child_base;  // tree index of slot 0 of the child-level buffer
  long long level_fronts;  // fronts of the whole level (variant choices use this)
  const unsigned char* zero_upd;  // per front (slice-relative): pivot-free subtree, or null
  const unsigned char* implicit_upd;  // per front: forward update left implicit (-L21 w_piv)
  const double* factors;              // this level's factor buffer (implicit updates)
  int leaf_direct;                    // leaf pass-through (tf_level_view.leaf_direct)
  const int* __restrict__ src_pattern_of;  // level 1 with leaf_direct: leaf-level tables
  const int* __restrict__ src_pat;
  const int* __restrict__ src_maps;
  // front f's forward update block is identically zero (never written)
  __device__ __forceinline__ bool upd_is_zero(long long f) const {
    if (zero_upd) return (zero_upd[f] & 1) != 0;
    return is_leaf && pat[(size_t)pattern_of[f] * TF_PAT_WIDTH + TF_PAT_K] == 0;
  }
  // every child of front f has a pivot-free subtree: no child reads the
  // front's backward block
  __device__ __forceinline__ bool children_idle(long long f) const {
    return zero_upd && (zero_upd[f] & 2) != 0;
  }
  __device__ __forceinline__ bool upd_implicit(long long f) const {
    return implicit_upd && implicit_upd[f] != 0;
  }
  // child c of front f (slice-relative) -> slot in the child buffer / view
  __device__ __forceinline__ long long child_slot(long long f, int c) const {
    return 2 * (front_base + f) + c - child_base;
  }
};

inline LevelArgs make_args(const tf_level_view* v) {
  LevelArgs a;
  a.n_fronts = v->n_fronts;
  a.is_leaf = v->is_leaf;
  a.elem_ld = v->elem_ld;
  a.max_m = v->max_m;
  a.max_k = v->max_k;
  a.max_upd = v->max_upd;
  a.fac_stride = v->fac_stride;
  a.upd_stride = v->upd_stride;
  a.child_upd_stride = v->child_upd_stride;
  a.elem_stride = v->elem_stride;
  a.pattern_of = v->pattern_of;
  a.piv_off = reinterpret_cast<const long long*>(v->piv_off);
  a.pat = v->pat;
  a.maps = v->maps;
  a.aux = v->aux;
  a.aux_stride = v->aux_stride;
  a.front_base = v->front_base;
  a.child_base = v->child_base;
  a.level_fronts = v->level_fronts > 0 ? v->level_fronts : v->n_fronts;
  a.zero_upd = v->zero_upd;
  a.implicit_upd = v->implicit_upd;
  a.factors = v->factors;
  a.leaf_direct = v->leaf_direct;
  a.src_pattern_of = v->src_pattern_of;
  a.src_pat = v->src_pat;
  a.src_maps = v->src_maps;
  return a;
}


// Per-front view of the pattern row.
struct Shape {
  int m, k, kp, nsrc, len0, len1, off0, off1, ioff;
};

__device__ __forceinline__ Shape front_shape(const LevelArgs& L, long long f) {
  const int* P = L.pat + (size_t)L.pattern_of[f] * TF_PAT_WIDTH;
  Shape s;
  s.m = P[TF_PAT_M];
  s.k = P[TF_PAT_K];
  s.kp = P[TF_PAT_KP];
  s.nsrc = P[TF_PAT_NSRC];
  s.len0 = P[TF_PAT_LEN0];
  s.len1 = P[TF_PAT_LEN1];
  s.off0 = P[TF_PAT_OFF0];
  s.off1 = P[TF_PAT_OFF1];
  s.ioff = P[TF_PAT_IOFF];
  return s;
}

// Packed lower-triangular row-major offset of (r, c), c <= r.
__host__ __device__ __forceinline__ long long tri(long long r, long long c) {
  return r * (r + 1) / 2 + c;
}

// 32-bit variants for shared-memory fronts (all indices < 2^31).
__host__ __device__ __forceinline__ int tri32(int r, int c) { return ((r * (r + 1)) >> 1) + c; }
__device__ __forceinline__ int tri_row32(int e) {  // exact for e < 2^22
  int r = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  r -= (((r * (r + 1)) >> 1) > e);
  r += ((((r + 1) * (r + 2)) >> 1) <= e);
  return r;
}

// Row of packed index e (exact for any e < 2^50).
__device__ __forceinline__ int tri_row(long long e) {
  int r;
  if (e < (1LL << 22)) {
    r = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  } else {
    r = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
  }
  while ((long long)r * (r + 1) / 2 > e) r--;
  while ((long long)(r + 1) * (r + 2) / 2 <= e) r++;
  return r;
}

// Barrier over a group of G threads: G < 32 lanes of one warp (mask), a
// warp, or a named barrier covering G threads (id >= 1).
template <int G>
__device__ __forceinline__ void group_sync(int bar_id) {
  if constexpr (G < 32) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned base = lane & ~(unsigned)(G - 1);
    const unsigned mask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << base;
    __syncwarp(mask);
  } else if constexpr (G == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(G) : "memory");
  }
}

__device__ __forceinline__ void record_zero_pivot(unsigned long long* err,
                                                  unsigned long long pos) {
  atomicMin(err, pos);
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Scheduling perturbation for race tests (tf_set_jitter): when the seed is
// non-zero, CTAs of the flag-synchronised kernels sleep a pseudo-random time
// at the start of each work item and after each acquire, so producers and
// consumers interleave differently run to run.  A missing wait or an early
// publish then shows up as a result that differs from the unperturbed run.
// One copy per translation unit (set through tf_set_jitter for all of them).
static __device__ unsigned g_jitter_seed;
__device__ __forceinline__ void tfb_jitter(unsigned salt) {
  const unsigned seed = *(volatile unsigned*)&g_jitter_seed;
  if (seed == 0) return;
  unsigned h = (blockIdx.x * 0x9E3779B1u) ^ (salt * 0x85EBCA77u) ^ seed;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
  const unsigned ns = h & 0x3FFF;  // up to ~16 us
  for (unsigned t = 0; t < ns; t += 1000) __nanosleep(1000);
}
inline cudaError_t set_jitter_tu(unsigned seed) {
  return cudaMemcpyToSymbol(g_jitter_seed, &seed, sizeof(seed));
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace tfb
