/*
 * tracefront_b200.h — C ABI of the B200-native multifrontal factor/solve path.
 *
 * This is the drop-in boundary for the reference package `tracefront`
 * (/root/reference/pkg/src/tracefront).  The reference is pure Python and
 * has no FFI; each entry point below names the reference function whose
 * semantics it replaces (file:line).  All pointers are plain host or CUDA
 * device pointers, sizes are int64, streams are `cudaStream_t` passed as
 * `void*`.  No torch types cross this boundary.  The library owns only the
 * host-side symbolic plan (`tf_plan`); every device buffer is allocated by
 * the caller.
 *
 * Status codes: TF_OK (0), TF_ZERO_PIVOT (2, mirrors ZeroPivotError /
 * cli.py exit code 2), negative values for invalid input or CUDA errors.
 */
#ifndef TRACEFRONT_B200_H
#define TRACEFRONT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_OK 0
#define TF_ZERO_PIVOT 2
#define TF_ERR_INVALID (-1)
#define TF_ERR_CUDA (-2)
#define TF_ERR_STRAY (-3) /* pivot couples outside its front (tasks.py:136-140) */

/* Pattern table row layout (int32 x TF_PAT_WIDTH per pattern). */
#define TF_PAT_WIDTH 12
#define TF_PAT_M 0      /* front order (non-eliminated indices) */
#define TF_PAT_K 1      /* pivots eliminated in this front */
#define TF_PAT_NSRC 2   /* 1 (element or carry child) or 2 children */
#define TF_PAT_LEN0 3   /* length of source 0 (element size, or child m-k) */
#define TF_PAT_LEN1 4
#define TF_PAT_OFF0 5   /* offset of source-0 map in the maps array */
#define TF_PAT_OFF1 6
#define TF_PAT_LEAF 7   /* 1 when source 0 is an element matrix */
#define TF_PAT_IOFF 8   /* inverse maps: front position -> source position (-1 if none);
                           source 0 at maps[IOFF, IOFF+m), source 1 at [IOFF+m, IOFF+2m) */
#define TF_PAT_KP 9     /* panel leading dimension: k rounded up to a multiple of 4 */
#define TF_PAT_FAC 10   /* doubles of the front's factor slot: m*kp (panel) + kp (diag) */
#define TF_PAT_SOFF 11  /* offset in the maps array of the extend-add scatter table
                           (fronts of order <= 232; -1 otherwise): entry e of source c
                           (packed lower order, source 1 after tri(len0) entries of
                           source 0) -> position in the shared-memory front layout
                           [pivot rows packed | L21 rows of stride kp+1 | Schur block packed] */

/* ------------------------------------------------------------------ mesh */

/* Tensor-product Q_p mesh on the unit box, DOFs numbered by the Morton index
 * of their owning element; elements returned in Morton
 * order, element-local DOF order x fastest.  For dim == 1 this equals
 * fem.py:59-80 (Mesh.element_dofs).  Pass elem_dofs == NULL to query
 * n_dof / n_elem only.  elem_dofs: n_elem * (p+1)^dim int32 (1-based). */
int tf_mesh_tensor(int32_t dim, const int64_t* ns, int32_t degree, int64_t* n_dof,
                   int64_t* n_elem, int32_t* elem_dofs);

/* tf_mesh_tensor on the GPU (same tables, bitwise): Morton keys, a radix sort,
 * an exclusive scan of owned-point counts and one thread per (element, local
 * point).  elem_dofs: device, n_elem * (p+1)^dim int32; order_out (optional,
 * device, n_elem int64): the x-fastest linear index of each Morton-ordered
 * element.  workspace: tf_mesh_tensor_device_workspace() bytes of device
 * memory.  Replaces the element loop of fem.py:59-80 / generate_fronts
 * (fem.py:235-259) for tensor meshes. */
int64_t tf_mesh_tensor_device_workspace(int32_t dim, const int64_t* ns, int32_t degree);
int tf_mesh_tensor_device(int32_t dim, const int64_t* ns, int32_t degree, int32_t* elem_dofs,
                          int64_t* order_out, void* workspace, int64_t workspace_bytes,
                          void* stream);

/* Element matrices of a graded / weighted tensor mesh on the GPU, Morton
 * order: values[e] = (prod_a width_a(e)) * density[e] * ref (ref = kron of the
 * reference 1D mass matrices of unit width, fem.py:108-114).  nodes: device,
 * concatenated per-axis element boundaries (n_a + 1 each) or NULL (uniform);
 * density: device, per Morton element, or NULL. */
int tf_mesh_element_values_device(int32_t dim, const int64_t* ns, int32_t degree,
                                  const int64_t* order, const double* nodes,
                                  const double* density, const double* ref, double* values,
                                  void* stream);

/* -------------------------------------------------------------- symbolic */

typedef struct tf_plan tf_plan;

typedef struct {
  int64_t n_dof;
  int64_t n_leaves;
  int64_t n_nodes;
  int64_t n_pivots;
  int32_t n_levels;
  int32_t max_m;
  int32_t max_k;
  int32_t keep_lists;
} tf_plan_summary;

/* Host-side per-level tables (owned by the plan; valid until destroy). */
typedef struct {
  int32_t level;
  int32_t n_fronts;
  int32_t n_patterns;
  int32_t max_m;
  int32_t max_k;
  int32_t max_upd; /* max (m-k) */
  int64_t node_base;   /* reference node id of front 0 (tree.py:133,153) */
  int64_t piv_base;    /* first pivot-order position of this level */
  int64_t n_pivots;    /* pivots eliminated at this level */
  int64_t maps_len;
  const int32_t* pattern_of; /* [n_fronts] */
  const int64_t* piv_off;    /* [n_fronts] absolute pivot-order offset */
  const int32_t* pat;        /* [n_patterns * TF_PAT_WIDTH] */
  const int32_t* maps;       /* [maps_len] source position -> front position */
} tf_level_host;

/* Replaces sort_fronts + build_elimination_tree + symbolic_eliminate
 * (tree.py:44-48, 106-160; tasks.py:88-159) for fronts given in sorted
 * (leaf) order.  elem_ptr may be NULL when every element has nloc DOFs.
 * keep_lists != 0 keeps the per-node [eliminable | shared] index lists
 * (NodeReorder, tasks.py:62-70) for parity queries. */
int tf_plan_create(int64_t n_dof, int64_t n_elem, const int64_t* elem_ptr, int32_t nloc,
                   const int32_t* elem_dofs, int32_t keep_lists, tf_plan** out);
void tf_plan_destroy(tf_plan* plan);
int tf_plan_summary_get(const tf_plan* plan, tf_plan_summary* out);
int tf_plan_level(const tf_plan* plan, int32_t level, tf_level_host* out);
/* EliminationPlan.pivot_order (tasks.py:83-85): n_pivots 1-based DOFs. */
int tf_plan_pivot_order(const tf_plan* plan, int32_t* out);
/* Per-node front lists of one level: ptr[n_fronts+1], k[n_fronts], idx[ptr[n]]
 * ([eliminable ascending | shared ascending], tasks.py:114-122). */
int tf_plan_node_lists(const tf_plan* plan, int32_t level, int64_t* ptr, int32_t* k,
                       int32_t* idx);
/* Total length of the node lists of one level. */
int64_t tf_plan_node_lists_len(const tf_plan* plan, int32_t level);

/* Statistics of the canonical atomic Foata normal form. */
typedef struct {
  int64_t n_tasks;   /* |alphabet| = cells + sum_steps (a + 2a^2)   (tasks.py:162-182) */
  int64_t n_edges;   /* J1-J4 edges, counted like DependencyGraph.n_edges (tasks.py:207-252) */
  int64_t n_cells;   /* stored positions incl. fill = number of Assertions */
  int64_t max_width; /* widest Foata class */
  int32_t n_classes;
  int32_t singular;  /* pivot with no diagonal entry when TF_ERR_STRAY is returned */
  int64_t n_divisions;       /* sum_steps a   (Subtractions: same count as Multiplications) */
  int64_t n_multiplications; /* sum_steps a^2 */
} tf_fnf_stats;

/* Replaces build_task_graph + compute_fnf (tasks.py:360, schedule.py:60-82) for
 * schedule statistics: streams the Diekert graph in elimination order without
 * materialising it.  widths[c] = tasks in class c+1, kinds[c] = bitmask of
 * TaskKinds (bit kind-1: 1 division, 2 multiplication, 3 subtraction,
 * 4 assertion).  Pass widths = kinds = NULL to size the arrays from
 * st->n_classes; cap is their capacity.  Needs a plan built with keep_lists. */
int tf_atomic_fnf(const tf_plan* plan, tf_fnf_stats* st, int64_t* widths, int32_t* kinds,
                  int32_t cap);

/* ---------------------------------------------------------------- device */

/* Device view of one level: the tf_level_host arrays copied to the GPU. */
typedef struct {
  int32_t level;
  int32_t n_fronts;
  int32_t n_patterns;
  int32_t max_m;
  int32_t max_k;
  int32_t max_upd;
  int32_t is_leaf;
  int32_t elem_ld;          /* leading dimension of element matrices (leaf level) */
  int64_t fac_stride;       /* doubles per front slot in the factor buffer (>= m*k) */
  int64_t upd_stride;       /* doubles per front slot in this level's update buffer */
  int64_t child_upd_stride; /* upd_stride of level-1 (0 at the leaf level) */
  int64_t elem_stride;      /* doubles between element matrices (0: uniform) */
  const int32_t* pattern_of;
  const int64_t* piv_off;
  const int32_t* pat;
  const int32_t* maps;
  double* aux;        /* large-front levels: per front, the unit-lower inverses of its
                         64-wide diagonal blocks (ceil(k/64) x 64 x 64, row-major) */
  int64_t aux_stride; /* doubles per front in aux (tf_level_aux_doubles) */
  int64_t front_base; /* tree index of this view's front 0 (a rank's slice; 0 = whole level) */
  int64_t child_base; /* tree index of the front held in slot 0 of the child-level buffer */
  int64_t level_fronts; /* fronts of the whole level (a slice keeps the full count, so every
                           rank picks the same kernel variants) */
  const uint8_t* zero_upd; /* optional, per front: bit 0 when the front and its whole subtree
                              have no pivots, so its forward update block is identically zero:
                              the solve neither writes nor reads it (NULL: leaves with k == 0
                              only); bit 1 when every child has such a subtree, so no child reads
                              the front's backward block (it is not written) */
  const uint8_t* implicit_upd; /* optional, per front: 1 when its forward update is -L21 w_piv with
                                  no child contribution (k > 0, pivot-free children); the sweep
                                  then stores only the k unscaled pivot rows w_piv and the parent
                                  forms -L21 w_piv itself from `factors` (NULL: none) */
  const double* factors;       /* this level's factor buffer (read by the parent level's forward
                                  sweep for implicit updates; may be NULL otherwise) */
  int32_t leaf_direct; /* optional leaf pass-through (0: off).  Leaf level: fronts without
                          pivots write no update (it is their element matrix in front order).
                          Level 1 (shared-memory fronts only): such a leaf child is read from
                          its element matrix (elem, elem_stride of this view) instead of the
                          child-update buffer, through the tables below. */
  const int32_t* src_pattern_of; /* level 1 with leaf_direct: the leaf level's pattern_of */
  const int32_t* src_pat;        /* and pat; */
  const int32_t* src_maps;       /* per leaf pattern p: src_maps[p] = offset in src_maps of the
                                    table e -> element index (row-major, lower part) of entry e
                                    of the leaf's packed update */
} tf_level_view;

/* Doubles of `aux` each front of this level needs under the current
 * shared-memory / large-front split (0 for shared-memory levels). */
int64_t tf_level_aux_doubles(const tf_level_view* lv);

/* Workspace bytes tf_level_factor may use for this level (0 when none): the
 * root-dataflow kernel's acquire/release flags.  Passing a caller-owned
 * workspace of this size keeps concurrent factorizations (different plans /
 * streams) from sharing flags; with workspace == NULL a per-device scratch
 * buffer is used. */
int64_t tf_level_factor_workspace(const tf_level_view* lv);

/* One Foata class (tree level) of the numeric factorization: extend-add of
 * children update matrices (or element matrices at the leaves), partial
 * LDL^T of the k fully-summed pivots, Schur complement.  Replaces the
 * Division/Multiplication/Subtraction tasks of one level (engine.py:78-107,
 * 290-306) and factorize_nested_loops' per-level loop (engine.py:518-547).
 * factors: n_fronts * fac_stride (row-major m x k panel per front: the
 * strictly-lower part holds l(x,z) = u(z,x), the diagonal holds u(z,z)).
 * upd_out: n_fronts * upd_stride (packed lower (m-k)^2 Schur complement).
 * err: device uint64, atomicMin of the pivot-order position of the first
 * pivot with |d| <= threshold (engine.py:91-92, 158-159, 529-530). */
int tf_level_factor(const tf_level_view* lv, const double* child_upd, const double* elem,
                    double* factors, double* upd_out, double threshold,
                    unsigned long long* err, void* workspace, int64_t workspace_bytes,
                    void* stream);

/* Bottom-level fusion: how many of the lowest levels (views[0..n_levels)) one
 * subtree kernel can run with their intermediate Schur blocks kept in shared
 * memory (0 or >= 2). */
int32_t tf_subtree_fusable(const tf_level_view* views, int32_t n_levels);

/* Levels 0..nlev-1 in one launch (one CTA per level-(nlev-1) subtree): same
 * arithmetic and outputs as nlev tf_level_factor calls -- factors[L] for
 * every fused level and the packed updates of level nlev-1 in upd_out -- but
 * the updates between the fused levels never leave shared memory. */
int tf_subtree_factor(const tf_level_view* views, int32_t nlev, double* const* factors,
                      const double* elem, double* upd_out, double threshold,
                      unsigned long long* err, void* stream);

/* Forward sweep of solve (engine.py:481-487) for one level, nrhs columns,
 * row-major (n x nrhs) vectors in pivot order.  child: view of level-1 (NULL
 * at the leaves); w_child: its front blocks (stride child_rows * nrhs);
 * w_out: this level's front blocks (stride out_rows * nrhs, out_rows >=
 * max_m).  A front's update rows are left in its block at rows [0, m-k) on
 * shared-memory levels and in place at rows [k, m) on large-front levels;
 * y: pivot-order RHS, overwritten by D^-1 L^-1 b at this level's pivots.
 * workspace: tf_level_solve_workspace bytes (flags + blocks of the
 * wavefront sweep on large-front levels; 0 bytes otherwise). */
int tf_level_solve_fwd(const tf_level_view* lv, const tf_level_view* child,
                       const double* factors, const double* w_child, int64_t child_rows,
                       double* w_out, int64_t out_rows, double* y, int32_t nrhs,
                       void* workspace, int64_t workspace_bytes, void* stream);

/* Backward sweep (engine.py:488-492) for one level.  parent: view of
 * level+1 (NULL at the root level) and its x buffer (stride parent_rows*nrhs);
 * x_out: this level's front x vectors (stride out_rows*nrhs); y: pivot-order
 * vector, overwritten with x at this level's pivots. */
int tf_level_solve_bwd(const tf_level_view* lv, const tf_level_view* parent,
                       const double* factors, const double* x_parent, int64_t parent_rows,
                       double* x_out, int64_t out_rows, double* y, int32_t nrhs,
                       void* workspace, int64_t workspace_bytes, void* stream);

/* Tiny trees (1D meshes, small 2D ones): the whole factorization (every
 * level of tf_level_factor) and, optionally, a single-RHS solve (permute,
 * every forward and backward level sweep, scatter back) in ONE launch of one
 * CTA -- the per-level launches, not the work, are the cost there.  views:
 * all levels (factors attached, whole levels); upd0/upd1: the ping-pong
 * update buffers (level L writes upd[L & 1]); perm/n_pivots: the pivot order
 * (1-based, tf_plan_pivot_order); b -> x (n_dof, may alias); y: n_pivots
 * scratch; blk0/blk1: solve blocks (n_fronts * max_m doubles per level).
 * tf_tree_small_ok: 1 when the tree qualifies (levels all shared-memory
 * levels with small fronts, <= 4096 leaves). */
int32_t tf_tree_small_ok(const tf_level_view* views, int32_t n_levels);
int tf_tree_factor_solve(const tf_level_view* views, int32_t n_levels, const double* elem,
                         double* upd0, double* upd1, double threshold, unsigned long long* err,
                         const int32_t* perm, int64_t n_pivots, int64_t n_dof, const double* b,
                         double* x, double* y, double* blk0, double* blk1, int32_t do_factor,
                         int32_t do_solve, void* stream);

/* Workspace bytes tf_level_solve_fwd / tf_level_solve_bwd need for this level and nrhs. */
int64_t tf_level_solve_workspace(const tf_level_view* lv, int32_t nrhs);

/* out[i, :] = in[idx[i]-1, :] (natural -> pivot order); inverse when scatter != 0. */
int tf_permute_rows(const int32_t* idx, int64_t n, const double* in, double* out, int32_t nrhs,
                    int32_t scatter, void* stream);

/* Kernel launches one call issues for this level: phase 0 tf_level_factor,
 * 1 tf_level_solve_fwd, 2 tf_level_solve_bwd. */
int32_t tf_level_launch_count(const tf_level_view* lv, int32_t nrhs, int32_t phase);

/* Front order up to which a level runs the shared-memory kernels (default and
 * maximum 232); smaller values route levels through the blocked large-front
 * kernels (a test and tuning knob).  Returns the previous value. */
int32_t tf_set_small_max_m(int32_t m);

/* Optional device timing of every kernel the library launches, by kernel class
 * (CUDA events recorded on the launch stream around each launch).  collect()
 * synchronises, returns the number of classes and fills per-class total ms and
 * launch counts (arrays of n), then resets. */
void tf_timing_enable(int32_t on);
int32_t tf_timing_collect(double* ms, int64_t* count, int32_t n);
const char* tf_timing_class_name(int32_t cls);

/* Library build identification (arch, compile flags). */
const char* tf_build_info(void);

/* 1 when this level's forward (fwd != 0) or backward sweep for nrhs columns
 * runs the cooperative wavefront kernels (their whole grid must be
 * co-resident), 0 otherwise.  Callers overlapping the forward sweep with the
 * factorization of later levels keep cooperative sweeps after it. */
int32_t tf_level_solve_cooperative(const tf_level_view* lv, int32_t nrhs, int32_t fwd);

/* Test hook (race detection without compute-sanitizer): seed != 0 makes the
 * CTAs of the flag-synchronised kernels (root dataflow, wavefront sweeps)
 * sleep pseudo-random times at each work item and after each acquire; 0
 * restores normal scheduling.  Results must be bitwise unchanged. */
int tf_set_jitter(uint32_t seed);

#ifdef __cplusplus
}
#endif
#endif
