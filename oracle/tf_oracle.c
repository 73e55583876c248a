/*
 * TEST INFRASTRUCTURE ONLY — C port of the reference's cell-level arithmetic.
 *
 * Restates, with the same floating-point operations in the same order:
 *   GlobalSystem.add / assemble (fem.py:145-147, 218-232; 2D/3D: the golden
 *     generator's element-order GlobalSystem.add loop)
 *   sort order / pairwise tree, membership (tree.py:88-160)
 *   factorize_nested_loops (engine.py:500-552): per pivot z, row/col scan of
 *     the stored cells, q = a(z,y)/a(z,z); a(x,y) -= q*a(x,z); l = a(x,z)/a(z,z)
 *   solve (engine.py:468-493)
 * Compiled with -ffp-contract=off so no FMA changes the rounding: its factors
 * and solutions are bitwise equal to the reference's (pinned by
 * tests/test_oracle.py against the tests/golden npz files).  Used only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 * Single-threaded: the per-cell subtraction chains (tasks.py:242-249) fix the
 * order of updates to shared cells, so a faithful port is sequential.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t* keys; /* (x << 32 | y) + 1, 0 = empty */
  double* vals;
  int64_t cap, n;
} cellmap;

static uint64_t hash64(uint64_t k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL;
  return k ^ (k >> 33);
}

static int cm_init(cellmap* m, int64_t cap) {
  int64_t c = 1024;
  while (c < cap * 2) c <<= 1;
  m->keys = (uint64_t*)calloc((size_t)c, sizeof(uint64_t));
  m->vals = (double*)malloc((size_t)c * sizeof(double));
  m->cap = c; m->n = 0;
  return m->keys && m->vals ? 0 : -1;
}

static int cm_grow(cellmap* m);

/* slot of key (inserting with value 0.0 if absent); *fresh = 1 on insert */
static int64_t cm_slot(cellmap* m, uint32_t x, uint32_t y, int* fresh) {
  if (m->n * 10 >= m->cap * 7) { if (cm_grow(m)) return -1; }
  uint64_t key = (((uint64_t)x << 32) | y) + 1;
  int64_t mask = m->cap - 1, i = (int64_t)(hash64(key) & (uint64_t)mask);
  while (m->keys[i] && m->keys[i] != key) i = (i + 1) & mask;
  if (!m->keys[i]) { m->keys[i] = key; m->vals[i] = 0.0; m->n++; if (fresh) *fresh = 1; }
  else if (fresh) *fresh = 0;
  return i;
}

static int64_t cm_find(const cellmap* m, uint32_t x, uint32_t y) {
  uint64_t key = (((uint64_t)x << 32) | y) + 1;
  int64_t mask = m->cap - 1, i = (int64_t)(hash64(key) & (uint64_t)mask);
  while (m->keys[i] && m->keys[i] != key) i = (i + 1) & mask;
  return m->keys[i] ? i : -1;
}

static int cm_grow(cellmap* m) {
  cellmap n2;
  if (cm_init(&n2, m->cap)) return -1;
  for (int64_t i = 0; i < m->cap; i++) {
    if (!m->keys[i]) continue;
    uint64_t key = m->keys[i] - 1;
    int64_t mask = n2.cap - 1, j = (int64_t)(hash64(key + 1) & (uint64_t)mask);
    while (n2.keys[j]) j = (j + 1) & mask;
    n2.keys[j] = key + 1; n2.vals[j] = m->vals[i]; n2.n++;
  }
  free(m->keys); free(m->vals);
  *m = n2;
  return 0;
}

typedef struct { int32_t* v; int64_t n, cap; } ivec;
static int iv_push(ivec* a, int32_t x) {
  if (a->n == a->cap) {
    int64_t c = a->cap ? a->cap * 2 : 8;
    int32_t* nv = (int32_t*)realloc(a->v, (size_t)c * sizeof(int32_t));
    if (!nv) return -1;
    a->v = nv; a->cap = c;
  }
  a->v[a->n++] = x;
  return 0;
}
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* one open-addressing table per matrix row x, keyed by column y: the inner
 * update loop of a pivot walks one row at a time (cache-resident). */
typedef struct { int32_t* keys; double* vals; int32_t cap, n; } rowmap; /* key y+1, 0 empty */

static int rm_grow(rowmap* r);
static int32_t rm_slot(rowmap* r, int32_t y, int* fresh) {
  if ((int64_t)r->n * 10 >= (int64_t)r->cap * 7) { if (rm_grow(r)) return -1; }
  const int32_t key = y + 1, mask = r->cap - 1;
  int32_t i = (int32_t)((uint32_t)y * 2654435761u) & mask;
  while (r->keys[i] && r->keys[i] != key) i = (i + 1) & mask;
  if (!r->keys[i]) { r->keys[i] = key; r->vals[i] = 0.0; r->n++; *fresh = 1; }
  else *fresh = 0;
  return i;
}
static int32_t rm_find(const rowmap* r, int32_t y) {
  if (!r->cap) return -1;
  const int32_t key = y + 1, mask = r->cap - 1;
  int32_t i = (int32_t)((uint32_t)y * 2654435761u) & mask;
  while (r->keys[i] && r->keys[i] != key) i = (i + 1) & mask;
  return r->keys[i] ? i : -1;
}
static int rm_grow(rowmap* r) {
  const int32_t oc = r->cap, nc = oc ? oc * 2 : 8;
  int32_t* ok = r->keys; double* ov = r->vals;
  r->keys = (int32_t*)calloc((size_t)nc, sizeof(int32_t));
  r->vals = (double*)malloc((size_t)nc * sizeof(double));
  if (!r->keys || !r->vals) return -1;
  r->cap = nc; r->n = 0;
  for (int32_t i = 0; i < oc; i++)
    if (ok[i]) { int f; int32_t s = rm_slot(r, ok[i] - 1, &f); r->vals[s] = ov[i]; }
  free(ok); free(ov);
  return 0;
}

typedef struct {
  int64_t n_dof, n_piv;
  int32_t* pivot_order;
  /* u: (z, y, q) in insertion order; diag stored separately */
  int64_t n_u, n_l, cap_u, cap_l;
  int32_t* u_z; int32_t* u_y; double* u_v;
  int32_t* l_x; int32_t* l_z; double* l_v;
  double* diag; /* by global index */
  int64_t* u_row_ptr; /* per pivot position: range of off-diagonal u entries */
  int64_t* l_col_ptr;
  int64_t zp_front, zp_pivot; /* zero pivot (front node id, pivot), -1 if none */
} oracle_result;

static int push_u(oracle_result* r, int32_t z, int32_t y, double v) {
  if (r->n_u == r->cap_u) {
    int64_t c = r->cap_u ? r->cap_u * 2 : 1024;
    r->u_z = realloc(r->u_z, c * 4); r->u_y = realloc(r->u_y, c * 4);
    r->u_v = realloc(r->u_v, c * 8); r->cap_u = c;
    if (!r->u_z || !r->u_y || !r->u_v) return -1;
  }
  r->u_z[r->n_u] = z; r->u_y[r->n_u] = y; r->u_v[r->n_u++] = v;
  return 0;
}
static int push_l(oracle_result* r, int32_t x, int32_t z, double v) {
  if (r->n_l == r->cap_l) {
    int64_t c = r->cap_l ? r->cap_l * 2 : 1024;
    r->l_x = realloc(r->l_x, c * 4); r->l_z = realloc(r->l_z, c * 4);
    r->l_v = realloc(r->l_v, c * 8); r->cap_l = c;
    if (!r->l_x || !r->l_z || !r->l_v) return -1;
  }
  r->l_x[r->n_l] = x; r->l_z[r->n_l] = z; r->l_v[r->n_l++] = v;
  return 0;
}

void oracle_free(oracle_result* r) {
  if (!r) return;
  free(r->pivot_order); free(r->u_z); free(r->u_y); free(r->u_v);
  free(r->l_x); free(r->l_z); free(r->l_v); free(r->diag);
  free(r->u_row_ptr); free(r->l_col_ptr);
  free(r);
}

/* Elements given in leaf (sorted) order; elem_vals row-major nloc x nloc each
 * (elem_stride 0 = shared).  Returns 0 ok, 2 zero pivot, <0 error. */
int oracle_factor(int64_t n_dof, int64_t n_elem, int32_t nloc, const int32_t* dofs,
                  const double* elem_vals, int64_t elem_stride, oracle_result** out) {
  oracle_result* R = (oracle_result*)calloc(1, sizeof(oracle_result));
  if (!R) return -1;
  *out = R;
  R->n_dof = n_dof;
  R->zp_front = R->zp_pivot = -1;
  R->diag = (double*)calloc((size_t)n_dof + 1, sizeof(double));
  R->pivot_order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_dof + 1));
  R->u_row_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_dof + 2));
  R->l_col_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_dof + 2));
  if (!R->diag || !R->pivot_order || !R->u_row_ptr || !R->l_col_ptr) return -1;

  /* assembly: GlobalSystem.add(ga, gb, E[a][b]) for ga >= gb, element order */
  rowmap* V = (rowmap*)calloc((size_t)n_dof + 1, sizeof(rowmap)); /* cells (x, y) by row x */
  if (!V) return -1;
  cellmap A; /* lower-triangle assembled entries */
  if (cm_init(&A, n_elem * (int64_t)nloc * nloc)) return -1;
  int32_t* low_i = NULL; int32_t* low_j = NULL; int64_t n_low = 0, cap_low = 0;
  for (int64_t e = 0; e < n_elem; e++) {
    const int32_t* d = dofs + e * nloc;
    const double* E = elem_vals + e * elem_stride;
    for (int a = 0; a < nloc; a++)
      for (int b = 0; b < nloc; b++) {
        if (d[a] < d[b]) continue;
        int fresh;
        int64_t s = cm_slot(&A, (uint32_t)d[a], (uint32_t)d[b], &fresh);
        if (s < 0) return -1;
        A.vals[s] = A.vals[s] + E[a * nloc + b];
        if (fresh) {
          if (n_low == cap_low) {
            cap_low = cap_low ? cap_low * 2 : 4096;
            low_i = realloc(low_i, cap_low * 4); low_j = realloc(low_j, cap_low * 4);
          }
          low_i[n_low] = d[a]; low_j[n_low++] = d[b];
        }
      }
  }
  double peak = 0.0;
  for (int64_t t = 0; t < n_low; t++) {
    double v = A.vals[cm_find(&A, (uint32_t)low_i[t], (uint32_t)low_j[t])];
    if (fabs(v) > peak) peak = fabs(v);
    int fresh;
    int32_t s = rm_slot(&V[low_i[t]], low_j[t], &fresh);
    if (s < 0) return -1;
    V[low_i[t]].vals[s] = v;
    if (low_i[t] != low_j[t]) {
      s = rm_slot(&V[low_j[t]], low_i[t], &fresh);
      if (s < 0) return -1;
      V[low_j[t]].vals[s] = v;
    }
  }
  free(low_i); free(low_j);
  free(A.keys); free(A.vals);
  const double threshold = 1e-14 * peak;

  /* tree levels by the pairing rule; membership via ancestor counts */
  int32_t n_levels = 1;
  for (int64_t n = n_elem; n > 1; n = (n + 1) / 2) n_levels++;
  /* leaves of each DOF (CSR) */
  int64_t* lp = (int64_t*)calloc((size_t)n_dof + 2, sizeof(int64_t));
  for (int64_t t = 0; t < n_elem * nloc; t++) lp[dofs[t] + 1]++;
  for (int64_t g = 0; g <= n_dof; g++) lp[g + 1] += lp[g];
  int64_t* leaf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_elem * nloc));
  int64_t* fillp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_dof + 1));
  memcpy(fillp, lp, sizeof(int64_t) * (size_t)(n_dof + 1));
  for (int64_t e = 0; e < n_elem; e++)
    for (int a = 0; a < nloc; a++) leaf[fillp[dofs[e * nloc + a]]++] = e;
  free(fillp);
  char* elim = (char*)calloc((size_t)n_dof + 1, 1);
  int64_t* node_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_dof + 1));
  int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_dof + 1));
  int64_t npiv = 0, node_base = 0, lsize = n_elem;
  ivec rowbuf = {0}, colbuf = {0};
  double* colv = NULL; double* qv = NULL; int64_t colv_cap = 0;
  for (int32_t L = 0; L < n_levels; L++) {
    /* eligible DOFs of this level, keyed by node */
    int64_t nc = 0;
    for (int64_t g = 1; g <= n_dof; g++) {
      if (elim[g] || lp[g] == lp[g + 1]) continue;
      int64_t anc = leaf[lp[g]] >> L; /* parent(i) = i / 2 applied L times */
      int one = 1;
      for (int64_t t = lp[g] + 1; t < lp[g + 1]; t++)
        if ((leaf[t] >> L) != anc) { one = 0; break; }
      if (one || L == n_levels - 1) { node_of[g] = anc; cand[nc++] = (int32_t)g; }
    }
    /* order: node ascending, then global index ascending (stable in g) */
    int64_t* cnt = (int64_t*)calloc((size_t)lsize + 1, sizeof(int64_t));
    for (int64_t t = 0; t < nc; t++) cnt[node_of[cand[t]] + 1]++;
    for (int64_t i = 0; i < lsize; i++) cnt[i + 1] += cnt[i];
    int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nc + 1));
    for (int64_t t = 0; t < nc; t++) ord[cnt[node_of[cand[t]]]++] = cand[t];
    free(cnt);
    for (int64_t t = 0; t < nc; t++) {
      const int32_t z = ord[t];
      const int32_t zs = rm_find(&V[z], z);
      const double pv = zs >= 0 ? V[z].vals[zs] : 0.0;
      if (fabs(pv) <= threshold) {
        R->zp_front = node_base + node_of[z];
        R->zp_pivot = z;
        free(ord);
        goto done_zero;
      }
      rowbuf.n = 0; colbuf.n = 0;
      for (int32_t q = 0; q < V[z].cap; q++) {
        const int32_t y = V[z].keys[q] - 1;
        if (y >= 0 && y != z && !elim[y]) iv_push(&rowbuf, y);
      }
      qsort(rowbuf.v, (size_t)rowbuf.n, sizeof(int32_t), cmp_i32);
      /* col = x with (x, z) stored: the pattern is symmetric, so same set as row */
      for (int64_t q = 0; q < rowbuf.n; q++) iv_push(&colbuf, rowbuf.v[q]);
      R->u_row_ptr[npiv] = R->n_u;
      if (colv_cap < rowbuf.n) {
        colv_cap = rowbuf.n * 2;
        colv = (double*)realloc(colv, sizeof(double) * (size_t)colv_cap);
        qv = (double*)realloc(qv, sizeof(double) * (size_t)colv_cap);
      }
      /* Row z and column z are not written while pivot z updates (x, y != z),
       * so q(z,y) = a(z,y)/a(z,z) and a(x,z) are read once up front, and each
       * cell a(x,y) still receives exactly a(x,y) - q(z,y)*a(x,z) once per
       * pivot: the visiting order of distinct cells does not change any
       * rounding (engine.py:536-545). */
      for (int64_t a = 0; a < rowbuf.n; a++) {
        const int32_t y = rowbuf.v[a];
        qv[a] = V[z].vals[rm_find(&V[z], y)] / pv;
        push_u(R, z, y, qv[a]);
      }
      for (int64_t b = 0; b < colbuf.n; b++)
        colv[b] = V[colbuf.v[b]].vals[rm_find(&V[colbuf.v[b]], z)];
      for (int64_t b = 0; b < colbuf.n; b++) {
        rowmap* row = &V[colbuf.v[b]];
        const double cx = colv[b];
        for (int64_t a = 0; a < rowbuf.n; a++) {
          const double prod = qv[a] * cx;
          int fresh;
          const int32_t s = rm_slot(row, rowbuf.v[a], &fresh);
          if (s < 0) return -1;
          row->vals[s] = row->vals[s] - prod;
        }
      }
      R->diag[z] = pv;
      R->l_col_ptr[npiv] = R->n_l;
      for (int64_t b = 0; b < colbuf.n; b++) {
        const int32_t x = colbuf.v[b];
        push_l(R, x, z, V[x].vals[rm_find(&V[x], z)] / pv);
      }
      R->pivot_order[npiv++] = z;
      elim[z] = 1;
    }
    free(ord);
    node_base += lsize;
    lsize = (lsize + 1) / 2;
  }
  R->u_row_ptr[npiv] = R->n_u;
  R->l_col_ptr[npiv] = R->n_l;
done_zero:
  R->n_piv = npiv;
  free(rowbuf.v); free(colbuf.v); free(colv); free(qv);
  free(lp); free(leaf); free(elim); free(node_of); free(cand);
  for (int64_t g = 0; g <= n_dof; g++) { free(V[g].keys); free(V[g].vals); }
  free(V);
  return R->zp_pivot >= 0 ? 2 : 0;
}

/* solve (engine.py:468-493) for one column, in place on b (n_dof). */
void oracle_solve(const oracle_result* R, double* b) {
  for (int64_t t = 0; t < R->n_piv; t++) {
    const int32_t z = R->pivot_order[t];
    const double bz = b[z - 1];
    for (int64_t q = R->l_col_ptr[t]; q < R->l_col_ptr[t + 1]; q++)
      b[R->l_x[q] - 1] -= R->l_v[q] * bz;
  }
  for (int64_t t = 0; t < R->n_piv; t++) {
    const int32_t z = R->pivot_order[t];
    b[z - 1] /= R->diag[z];
  }
  for (int64_t t = R->n_piv - 1; t >= 0; t--) {
    const int32_t z = R->pivot_order[t];
    double acc = b[z - 1];
    for (int64_t q = R->u_row_ptr[t]; q < R->u_row_ptr[t + 1]; q++)
      acc -= R->u_v[q] * b[R->u_y[q] - 1];
    b[z - 1] = acc;
  }
}

int64_t oracle_n_piv(const oracle_result* R) { return R->n_piv; }
int64_t oracle_n_u(const oracle_result* R) { return R->n_u; }
int64_t oracle_n_l(const oracle_result* R) { return R->n_l; }
void oracle_zero_pivot(const oracle_result* R, int64_t* front, int64_t* pivot) {
  *front = R->zp_front; *pivot = R->zp_pivot;
}
void oracle_get(const oracle_result* R, int32_t* pivots, int32_t* u_z, int32_t* u_y, double* u_v,
                int32_t* l_x, int32_t* l_z, double* l_v, double* diag_by_pivot) {
  if (pivots) memcpy(pivots, R->pivot_order, sizeof(int32_t) * (size_t)R->n_piv);
  if (u_z) memcpy(u_z, R->u_z, sizeof(int32_t) * (size_t)R->n_u);
  if (u_y) memcpy(u_y, R->u_y, sizeof(int32_t) * (size_t)R->n_u);
  if (u_v) memcpy(u_v, R->u_v, sizeof(double) * (size_t)R->n_u);
  if (l_x) memcpy(l_x, R->l_x, sizeof(int32_t) * (size_t)R->n_l);
  if (l_z) memcpy(l_z, R->l_z, sizeof(int32_t) * (size_t)R->n_l);
  if (l_v) memcpy(l_v, R->l_v, sizeof(double) * (size_t)R->n_l);
  if (diag_by_pivot)
    for (int64_t t = 0; t < R->n_piv; t++) diag_by_pivot[t] = R->diag[R->pivot_order[t]];
}
