// Shared device helpers for the level kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tracefront_b200.h"

namespace tfb {

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
  return a;
}

// Packed lower-triangular row-major offset of (r, c), c <= r.
__host__ __device__ __forceinline__ long long tri(long long r, long long c) {
  return r * (r + 1) / 2 + c;
}

// Inverse of tri(): row of packed index e.
__device__ __forceinline__ int tri_row(long long e) {
  int r = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
  while ((long long)r * (r + 1) / 2 > e) r--;
  while ((long long)(r + 1) * (r + 2) / 2 <= e) r++;
  return r;
}

// Barrier over a group of G threads (G = 32: warp; else named barrier id).
template <int G>
__device__ __forceinline__ void group_sync(int bar_id) {
  if constexpr (G == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(G) : "memory");
  }
}

__device__ __forceinline__ void record_zero_pivot(unsigned long long* err,
                                                  unsigned long long pos) {
  atomicMin(err, pos);
}

}  // namespace tfb
