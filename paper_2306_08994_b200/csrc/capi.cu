// extern "C" entry points of libtfb200.so (declared in include/tracefront_b200.h).
#include <cstdio>

#include "common.cuh"

namespace tfb {
cudaError_t launch_factor_small(const LevelArgs& L, const double* child_upd, const double* elem,
                                double* factors, double* upd_out, double thr,
                                unsigned long long* err, cudaStream_t st);
cudaError_t launch_factor_large(const LevelArgs& L, const double* child_upd, double* factors,
                                double* upd_out, double thr, unsigned long long* err,
                                int* ws_flags, cudaStream_t st);
bool root_dataflow_level(const LevelArgs& L);
long long level_factor_ws_ints(const LevelArgs& L);
cudaError_t launch_solve_fwd(const LevelArgs& L, const LevelArgs& C, const double* factors,
                             const double* w_child, long long child_rows, double* w_out,
                             long long out_rows, double* y, int nrhs, double* work,
                             long long work_doubles, cudaStream_t st);
cudaError_t launch_solve_bwd(const LevelArgs& L, const LevelArgs& PA, int has_parent,
                             const double* factors, const double* x_parent, long long parent_rows,
                             double* x_out, long long out_rows, double* y, int nrhs,
                             double* work, long long work_doubles, cudaStream_t st);
cudaError_t launch_permute_rows(const int* idx, long long n, const double* in, double* out,
                                int nrhs, int scatter, cudaStream_t st);
long long solve_workspace_doubles(const LevelArgs& L, int nrhs);
int subtree_fusable_levels(const LevelArgs* lv, int n_levels);
cudaError_t launch_factor_subtree(const LevelArgs* lv, int nlev, double* const* fac,
                                  const double* elem, double* upd_out, double thr,
                                  unsigned long long* err, cudaStream_t st);
struct TreeArgs;
size_t tree_small_smem(const LevelArgs* lv, int nlev, TreeArgs* A);
cudaError_t launch_tree_small(const LevelArgs* lv, int nlev, const double* elem, double* upd0,
                              double* upd1, double thr, unsigned long long* err, const int* perm,
                              long long n_piv, long long n_dof, const double* b, double* x,
                              double* y, double* blk0, double* blk1, int do_factor, int do_solve,
                              cudaStream_t st);
int large_level_launches(int max_k, int max_upd, long long level_fronts);
int solve_launches(const LevelArgs& L, int nrhs, bool fwd);
int solve_cooperative(const LevelArgs& L, int nrhs, bool fwd);
cudaError_t set_jitter_solve(unsigned seed);
cudaError_t set_jitter_factor(unsigned seed);
int g_small_max_m = 112;  // measured best split on B200 (tools/sweep.sh)
}  // namespace tfb

using namespace tfb;

static int status(cudaError_t e) {
  if (e == cudaSuccess) return TF_OK;
  fprintf(stderr, "tfb200: CUDA error %s\n", cudaGetErrorString(e));
  return TF_ERR_CUDA;
}

extern "C" int64_t tf_level_aux_doubles(const tf_level_view* lv) {
  if (!lv || !level_is_large(lv->is_leaf, lv->max_m) || lv->max_k <= 0) return 0;
  return large_aux_doubles(lv->max_k);
}

extern "C" int64_t tf_level_factor_workspace(const tf_level_view* lv) {
  // the dataflow kernels' acquire/release flags (root; lookahead chains): one
  // set per caller-owned workspace, so concurrent factorizations never share them
  if (!lv || lv->n_fronts == 0 || !level_is_large(lv->is_leaf, lv->max_m)) return 0;
  const LevelArgs L = make_args(lv);
  return (int64_t)sizeof(int) * level_factor_ws_ints(L);
}

extern "C" int64_t tf_level_solve_workspace(const tf_level_view* lv, int32_t nrhs) {
  if (!lv || nrhs < 1) return 0;
  return 8 * solve_workspace_doubles(make_args(lv), nrhs);
}

extern "C" int tf_level_factor(const tf_level_view* lv, const double* child_upd,
                               const double* elem, double* factors, double* upd_out,
                               double threshold, unsigned long long* err, void* workspace,
                               int64_t workspace_bytes, void* stream) {
  if (!lv || !err) return TF_ERR_INVALID;
  if (lv->n_fronts == 0) return TF_OK;
  if (lv->is_leaf && !elem) return TF_ERR_INVALID;
  if (!lv->is_leaf && !child_upd) return TF_ERR_INVALID;
  LevelArgs L = make_args(lv);
  cudaStream_t st = (cudaStream_t)stream;
  if (lv->leaf_direct && !lv->is_leaf && (!elem || !lv->src_pattern_of || !lv->src_pat ||
                                          !lv->src_maps || lv->front_base != 0))
    return TF_ERR_INVALID;
  if (!level_is_large(lv->is_leaf, lv->max_m))
    return status(launch_factor_small(L, child_upd, elem, factors, upd_out, threshold, err, st));
  if (lv->leaf_direct) return TF_ERR_INVALID;  // pass-through leaves need the shared-memory path
  if (lv->max_k > 0 && (!lv->aux || lv->aux_stride < large_aux_doubles(lv->max_k)))
    return TF_ERR_INVALID;
  int* flags = nullptr;
  if (workspace) {
    if (workspace_bytes < tf_level_factor_workspace(lv)) return TF_ERR_INVALID;
    flags = static_cast<int*>(workspace);
  }
  return status(launch_factor_large(L, child_upd, factors, upd_out, threshold, err, flags, st));
}

extern "C" int32_t tf_subtree_fusable(const tf_level_view* views, int32_t n_levels) {
  if (!views || n_levels < 1) return 0;
  LevelArgs lv[16];
  const int n = n_levels < 16 ? n_levels : 16;
  for (int L = 0; L < n; L++) lv[L] = make_args(&views[L]);
  return subtree_fusable_levels(lv, n);
}

extern "C" int tf_subtree_factor(const tf_level_view* views, int32_t nlev,
                                 double* const* factors, const double* elem, double* upd_out,
                                 double threshold, unsigned long long* err, void* stream) {
  if (!views || !factors || !elem || !err || nlev < 1 || nlev > 10) return TF_ERR_INVALID;
  LevelArgs lv[10];
  for (int L = 0; L < nlev; L++) {
    lv[L] = make_args(&views[L]);
    lv[L].leaf_direct = 0;  // the subtree kernel keeps every update in shared memory
    if (level_is_large(lv[L].is_leaf, lv[L].max_m) || lv[L].front_base != 0) return TF_ERR_INVALID;
  }
  return status(launch_factor_subtree(lv, nlev, factors, elem, upd_out, threshold, err,
                                      (cudaStream_t)stream));
}

extern "C" int tf_level_solve_fwd(const tf_level_view* lv, const tf_level_view* child,
                                  const double* factors, const double* w_child,
                                  int64_t child_rows, double* w_out, int64_t out_rows, double* y,
                                  int32_t nrhs, void* workspace, int64_t workspace_bytes,
                                  void* stream) {
  if (!lv || nrhs < 1 || out_rows < lv->max_m) return TF_ERR_INVALID;
  if (lv->n_fronts == 0) return TF_OK;
  if (!lv->is_leaf && (!child || !w_child)) return TF_ERR_INVALID;
  LevelArgs L = make_args(lv);
  LevelArgs C = child ? make_args(child) : L;
  if (workspace_bytes < 8 * solve_workspace_doubles(L, nrhs)) return TF_ERR_INVALID;
  return status(launch_solve_fwd(L, C, factors, w_child, child_rows, w_out, out_rows, y, nrhs,
                                 (double*)workspace, workspace_bytes / 8, (cudaStream_t)stream));
}

extern "C" int tf_level_solve_bwd(const tf_level_view* lv, const tf_level_view* parent,
                                  const double* factors, const double* x_parent,
                                  int64_t parent_rows, double* x_out, int64_t out_rows,
                                  double* y, int32_t nrhs, void* workspace,
                                  int64_t workspace_bytes, void* stream) {
  if (!lv || nrhs < 1 || out_rows < lv->max_m || !x_out) return TF_ERR_INVALID;
  if (lv->n_fronts == 0) return TF_OK;
  if (parent && !x_parent) return TF_ERR_INVALID;
  LevelArgs L = make_args(lv);
  LevelArgs PA = parent ? make_args(parent) : L;
  if (workspace_bytes < 8 * solve_workspace_doubles(L, nrhs)) return TF_ERR_INVALID;
  return status(launch_solve_bwd(L, PA, parent ? 1 : 0, factors, x_parent, parent_rows, x_out,
                                 out_rows, y, nrhs, (double*)workspace, workspace_bytes / 8,
                                 (cudaStream_t)stream));
}

extern "C" int32_t tf_tree_small_ok(const tf_level_view* views, int32_t n_levels) {
  if (!views || n_levels < 1 || n_levels > 24) return 0;
  LevelArgs lv[24];
  for (int L = 0; L < n_levels; L++) lv[L] = make_args(&views[L]);
  return tree_small_smem(lv, n_levels, nullptr) > 0 ? 1 : 0;
}

extern "C" int tf_tree_factor_solve(const tf_level_view* views, int32_t n_levels,
                                    const double* elem, double* upd0, double* upd1,
                                    double threshold, unsigned long long* err, const int32_t* perm,
                                    int64_t n_pivots, int64_t n_dof, const double* b, double* x,
                                    double* y, double* blk0, double* blk1, int32_t do_factor,
                                    int32_t do_solve, void* stream) {
  if (!views || n_levels < 1 || n_levels > 24) return TF_ERR_INVALID;
  if (do_factor && (!elem || !upd0 || !upd1 || !err)) return TF_ERR_INVALID;
  if (do_solve && (!perm || !b || !x || !y || !blk0 || !blk1)) return TF_ERR_INVALID;
  LevelArgs lv[24];
  for (int L = 0; L < n_levels; L++) lv[L] = make_args(&views[L]);
  if (tree_small_smem(lv, n_levels, nullptr) == 0) return TF_ERR_INVALID;
  return status(launch_tree_small(lv, n_levels, elem, upd0, upd1, threshold, err, perm, n_pivots,
                                  n_dof, b, x, y, blk0, blk1, do_factor, do_solve,
                                  (cudaStream_t)stream));
}

extern "C" int tf_permute_rows(const int32_t* idx, int64_t n, const double* in, double* out,
                               int32_t nrhs, int32_t scatter, void* stream) {
  if (!idx || !in || !out || nrhs < 1) return TF_ERR_INVALID;
  return status(launch_permute_rows(idx, n, in, out, nrhs, scatter, (cudaStream_t)stream));
}

extern "C" int32_t tf_level_launch_count(const tf_level_view* lv, int32_t nrhs, int32_t phase) {
  if (!lv || lv->n_fronts == 0) return 0;
  LevelArgs L = make_args(lv);
  if (phase == 0) {
    if (!level_is_large(lv->is_leaf, lv->max_m)) return 1;
    return large_level_launches(lv->max_k, lv->max_upd, L.level_fronts);
  }
  return solve_launches(L, nrhs, phase == 1);
}

extern "C" int32_t tf_set_small_max_m(int32_t m) {
  const int old = g_small_max_m;
  if (m >= 1 && m <= kSmallMaxM) g_small_max_m = m;
  return old;
}

extern "C" const char* tf_build_info(void) {
  return "tfb200 sm_100a fp64 (DMMA m8n8k4 via mma.sync; cp.async staging); "
         "shared-memory fronts <= 232, blocked large fronts";
}

extern "C" int tf_set_jitter(uint32_t seed) {
  cudaError_t e = set_jitter_factor(seed);
  if (e == cudaSuccess) e = set_jitter_solve(seed);
  return status(e);
}

extern "C" int32_t tf_level_solve_cooperative(const tf_level_view* lv, int32_t nrhs, int32_t fwd) {
  if (!lv || lv->n_fronts == 0 || nrhs < 1) return 0;
  return solve_cooperative(make_args(lv), nrhs, fwd != 0);
}
