// Host-side symbolic analysis: tensor meshes, elimination tree, pivot order,
// per-level front patterns and extend-add maps.
//
// Replaces, for fronts given in sorted (leaf) order:
//   sort_fronts / build_elimination_tree   tree.py:44-48, 106-160
//   symbolic_eliminate                     tasks.py:88-159
// without materialising per-node index unions or the filled adjacency.
//
// Key identity: pairwise joining of consecutive
// nodes plus one-child carry nodes means leaf j's ancestor at level L is node
// j >> L.  A DOF's membership at level L is 1 exactly when all leaves that
// contain it share the same (j >> L), so the reference eliminates DOF g at
//   L*(g) = bitlen(minleaf(g) XOR maxleaf(g))        in node minleaf(g) >> L*
// (the root level catches nothing extra: L* <= n_levels-1 always).  The
// pivot order of tasks.py:109-151 (level, node, ascending index) is then a
// counting sort, and each front's non-eliminated set is the union of its
// children's shared sets, laid out [eliminable ascending | shared ascending]
// exactly like NodeReorder (tasks.py:114-130).
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <new>
#include <unordered_map>
#include <vector>

#include "tracefront_b200.h"

namespace {

inline int bitlen64(uint64_t x) { return x == 0 ? 0 : 64 - __builtin_clzll(x); }

constexpr int32_t kScatterMaxM = 232;  // = kSmallMaxM of the shared-memory kernels

struct Level {
  int32_t n_fronts = 0, n_patterns = 0, max_m = 0, max_k = 0, max_upd = 0;
  int64_t node_base = 0, piv_base = 0, n_pivots = 0;
  std::vector<int32_t> pattern_of;
  std::vector<int64_t> piv_off;
  std::vector<int32_t> pat;
  std::vector<int32_t> maps;
  // optional per-node [elim | shared] lists
  std::vector<int64_t> list_ptr;
  std::vector<int32_t> list_k;
  std::vector<int32_t> list_idx;
};

inline uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdULL;
  return h ^ (h >> 33);
}

}  // namespace

struct tf_plan {
  int64_t n_dof = 0, n_leaves = 0, n_nodes = 0, n_pivots = 0;
  int32_t n_levels = 0, max_m = 0, max_k = 0, keep = 0;
  std::vector<int32_t> pivot_order;
  std::vector<Level> levels;
};

static int kp_align() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("TFB_KP_ALIGN");
    v = e ? atoi(e) : 2;
    if (v != 2 && v != 4) v = 2;
  }
  return v;
}

extern "C" int tf_mesh_tensor(int32_t dim, const int64_t* ns, int32_t p, int64_t* n_dof_out,
                              int64_t* n_elem_out, int32_t* elem_dofs) {
  if (dim < 1 || dim > 3 || p < 1 || !ns) return TF_ERR_INVALID;
  int64_t n[3] = {1, 1, 1};
  int64_t n_elem = 1, n_dof = 1;
  for (int a = 0; a < dim; a++) {
    if (ns[a] < 1) return TF_ERR_INVALID;
    n[a] = ns[a];
    n_elem *= n[a];
    n_dof *= n[a] * p + 1;
  }
  if (n_dof_out) *n_dof_out = n_dof;
  if (n_elem_out) *n_elem_out = n_elem;
  if (!elem_dofs) return TF_OK;
  if (n_dof >= (int64_t)INT32_MAX) return TF_ERR_INVALID;
  // Morton key per element (bit b of axis a at position dim*b + a).
  std::vector<std::pair<uint64_t, int64_t>> keyed(n_elem);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < n_elem; e++) {
    int64_t c[3] = {e % n[0], (e / n[0]) % n[1], e / (n[0] * n[1])};
    uint64_t key = 0;
    for (int b = 0; b < 21; b++)
      for (int a = 0; a < dim; a++) key |= (uint64_t)((c[a] >> b) & 1) << (dim * b + a);
    keyed[e] = {key, e};
  }
  bool sorted = true;
  for (int64_t e = 1; e < n_elem && sorted; e++) sorted = keyed[e - 1].first < keyed[e].first;
  if (!sorted) std::sort(keyed.begin(), keyed.end());
  std::vector<int64_t> rank_of(n_elem), first_gid(n_elem);
  int64_t acc = 0;
  for (int64_t r = 0; r < n_elem; r++) {
    int64_t e = keyed[r].second;
    rank_of[e] = r;
    int64_t c[3] = {e % n[0], (e / n[0]) % n[1], e / (n[0] * n[1])};
    int64_t owned = 1;
    for (int a = 0; a < dim; a++) owned *= p + (c[a] == n[a] - 1 ? 1 : 0);
    first_gid[r] = acc;
    acc += owned;
  }
  if (acc != n_dof) return TF_ERR_INVALID;
  const int64_t np1 = p + 1;
  int64_t nloc = 1;
  for (int a = 0; a < dim; a++) nloc *= np1;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n_elem; r++) {
    int64_t e = keyed[r].second;
    int64_t c[3] = {e % n[0], (e / n[0]) % n[1], e / (n[0] * n[1])};
    int32_t* out = elem_dofs + r * nloc;
    for (int64_t loc = 0; loc < nloc; loc++) {
      int64_t a_loc[3] = {loc % np1, (loc / np1) % np1, loc / (np1 * np1)};
      int64_t owner[3] = {0, 0, 0}, off[3] = {0, 0, 0}, w[3] = {1, 1, 1};
      for (int a = 0; a < dim; a++) {
        int64_t i = c[a] * p + a_loc[a];
        owner[a] = std::min(i / p, n[a] - 1);
        off[a] = i - owner[a] * p;
        w[a] = p + (owner[a] == n[a] - 1 ? 1 : 0);
      }
      int64_t oe = owner[0] + n[0] * (owner[1] + n[1] * owner[2]);
      int64_t lr = off[0] + w[0] * (off[1] + w[1] * off[2]);
      out[loc] = (int32_t)(first_gid[rank_of[oe]] + lr + 1);
    }
  }
  return TF_OK;
}

extern "C" int tf_plan_create(int64_t n_dof, int64_t n_elem, const int64_t* elem_ptr,
                              int32_t nloc, const int32_t* dofs, int32_t keep,
                              tf_plan** out) {
  if (!out) return TF_ERR_INVALID;
  *out = nullptr;
  if (n_elem < 1 || n_dof < 1 || !dofs || n_dof >= (int64_t)INT32_MAX) return TF_ERR_INVALID;
  if (!elem_ptr && nloc < 1) return TF_ERR_INVALID;
  auto eptr = [&](int64_t e) -> int64_t { return elem_ptr ? elem_ptr[e] : e * (int64_t)nloc; };
  tf_plan* P = new (std::nothrow) tf_plan();
  if (!P) return TF_ERR_INVALID;
  P->n_dof = n_dof;
  P->n_leaves = n_elem;
  P->keep = keep;

  // 1. leaf range of every DOF (elements are visited in ascending leaf order).
  std::vector<int64_t> minleaf(n_dof + 1, -1), maxleaf(n_dof + 1, -1);
  for (int64_t e = 0; e < n_elem; e++) {
    for (int64_t t = eptr(e); t < eptr(e + 1); t++) {
      int32_t g = dofs[t];
      if (g < 1 || g > n_dof) { delete P; return TF_ERR_INVALID; }
      if (minleaf[g] < 0) minleaf[g] = e;
      maxleaf[g] = e;
    }
  }
  // 2. level sizes and reference node ids (tree.py:133,153).
  std::vector<int64_t> lsize{n_elem};
  while (lsize.back() > 1) lsize.push_back((lsize.back() + 1) / 2);
  const int32_t n_levels = (int32_t)lsize.size();
  std::vector<int64_t> node_base(n_levels + 1, 0);
  for (int L = 0; L < n_levels; L++) node_base[L + 1] = node_base[L] + lsize[L];
  P->n_levels = n_levels;
  P->n_nodes = node_base[n_levels];

  // 3. elimination level / node per DOF and the pivot order (counting sort).
  std::vector<int8_t> elev(n_dof + 1, -1);
  std::vector<int64_t> count(P->n_nodes + 1, 0);
  for (int64_t g = 1; g <= n_dof; g++) {
    if (minleaf[g] < 0) continue;  // DOF in no front: never eliminated (as the reference)
    int L = bitlen64((uint64_t)(minleaf[g] ^ maxleaf[g]));
    elev[g] = (int8_t)L;
    count[node_base[L] + (minleaf[g] >> L) + 1]++;
  }
  for (int64_t i = 0; i < P->n_nodes; i++) count[i + 1] += count[i];
  P->n_pivots = count[P->n_nodes];
  P->pivot_order.resize(P->n_pivots);
  {
    std::vector<int64_t> fill(count.begin(), count.end() - 1);
    for (int64_t g = 1; g <= n_dof; g++) {
      if (elev[g] < 0) continue;
      int L = elev[g];
      P->pivot_order[fill[node_base[L] + (minleaf[g] >> L)]++] = (int32_t)g;
    }
  }
  minleaf.clear(); minleaf.shrink_to_fit();
  maxleaf.clear(); maxleaf.shrink_to_fit();

  // 4. per level: fronts, maps, patterns.
  P->levels.resize(n_levels);
  std::vector<int64_t> sh_ptr, sh_ptr_next;
  std::vector<int32_t> sh_idx, sh_idx_next;
  for (int L = 0; L < n_levels; L++) {
    Level& lv = P->levels[L];
    const int64_t nf = lsize[L];
    lv.n_fronts = (int32_t)nf;
    lv.node_base = node_base[L];
    lv.piv_base = count[node_base[L]];
    lv.n_pivots = count[node_base[L] + nf] - lv.piv_base;
    std::vector<int32_t> fm(nf), fk(nf), fsrc(nf);  // m, k, map length
    // pass 1: sizes
    bool bad = false;
#pragma omp parallel for schedule(dynamic, 1024) reduction(|| : bad)
    for (int64_t i = 0; i < nf; i++) {
      int32_t m = 0, k = 0, src = 0;
      if (L == 0) {
        int64_t b = eptr(i), e = eptr(i + 1);
        std::vector<int32_t> s(dofs + b, dofs + e);
        std::sort(s.begin(), s.end());
        if (std::adjacent_find(s.begin(), s.end()) != s.end()) bad = true;  // fem.py:197-198
        m = (int32_t)s.size();
        for (int32_t g : s) k += (elev[g] == 0);
        src = (int32_t)(e - b);
      } else {
        int64_t c0 = 2 * i, c1 = 2 * i + 1;
        const int32_t* a = sh_idx.data() + sh_ptr[c0];
        const int32_t* ae = sh_idx.data() + sh_ptr[c0 + 1];
        const int32_t* bb = c1 < lsize[L - 1] ? sh_idx.data() + sh_ptr[c1] : nullptr;
        const int32_t* be = c1 < lsize[L - 1] ? sh_idx.data() + sh_ptr[c1 + 1] : nullptr;
        src = (int32_t)(ae - a) + (bb ? (int32_t)(be - bb) : 0);
        while (a < ae || (bb && bb < be)) {
          int32_t g;
          if (!bb || bb >= be) g = *a++;
          else if (a >= ae) g = *bb++;
          else if (*a < *bb) g = *a++;
          else if (*bb < *a) g = *bb++;
          else { g = *a++; bb++; }
          m++;
          k += (elev[g] == L);
        }
      }
      fm[i] = m; fk[i] = k; fsrc[i] = src;
    }
    if (bad) { delete P; return TF_ERR_INVALID; }
    std::vector<int64_t> fptr(nf + 1, 0), mptr(nf + 1, 0);
    sh_ptr_next.assign(nf + 1, 0);
    for (int64_t i = 0; i < nf; i++) {
      fptr[i + 1] = fptr[i] + fm[i];
      mptr[i + 1] = mptr[i] + fsrc[i];
      sh_ptr_next[i + 1] = sh_ptr_next[i] + (fm[i] - fk[i]);
      // every pivot assigned to this node by the counting sort must be eliminable here
      if (fk[i] != count[node_base[L] + i + 1] - count[node_base[L] + i]) bad = true;
    }
    if (bad) { delete P; return TF_ERR_INVALID; }
    if (L == n_levels - 1 && sh_ptr_next[nf] != 0) { delete P; return TF_ERR_INVALID; }
    std::vector<int32_t> flist(fptr[nf]);
    std::vector<int32_t> fmap(mptr[nf]);
    sh_idx_next.assign(sh_ptr_next[nf], 0);
    // pass 2: fill front lists [elim | shared], shared lists, maps
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < nf; i++) {
      int32_t* fl = flist.data() + fptr[i];
      int32_t* sh = sh_idx_next.data() + sh_ptr_next[i];
      int32_t* mp = fmap.data() + mptr[i];
      const int32_t k = fk[i];
      std::vector<int32_t> u;
      u.reserve(fm[i]);
      if (L == 0) {
        u.assign(dofs + eptr(i), dofs + eptr(i + 1));
        std::sort(u.begin(), u.end());
      } else {
        int64_t c0 = 2 * i, c1 = 2 * i + 1;
        const int32_t* a = sh_idx.data() + sh_ptr[c0];
        const int32_t* ae = sh_idx.data() + sh_ptr[c0 + 1];
        const int32_t* bb = c1 < lsize[L - 1] ? sh_idx.data() + sh_ptr[c1] : nullptr;
        const int32_t* be = c1 < lsize[L - 1] ? sh_idx.data() + sh_ptr[c1 + 1] : nullptr;
        while (a < ae || (bb && bb < be)) {
          if (!bb || bb >= be) u.push_back(*a++);
          else if (a >= ae) u.push_back(*bb++);
          else if (*a < *bb) u.push_back(*a++);
          else if (*bb < *a) u.push_back(*bb++);
          else { u.push_back(*a++); bb++; }
        }
      }
      // positions in the [elim | shared] layout
      std::vector<int32_t> pos(u.size());
      int32_t re = 0, rs = 0;
      for (size_t t = 0; t < u.size(); t++) {
        if (elev[u[t]] == L) { pos[t] = re; fl[re++] = u[t]; }
        else { pos[t] = k + rs; fl[k + rs] = u[t]; sh[rs++] = u[t]; }
      }
      // maps: source position -> front position
      if (L == 0) {
        int64_t b = eptr(i), e = eptr(i + 1);
        for (int64_t t = b; t < e; t++) {
          size_t at = std::lower_bound(u.begin(), u.end(), dofs[t]) - u.begin();
          mp[t - b] = pos[at];
        }
      } else {
        int w = 0;
        for (int c = 0; c < 2; c++) {
          int64_t ch = 2 * i + c;
          if (ch >= lsize[L - 1]) break;
          size_t at = 0;
          for (int64_t t = sh_ptr[ch]; t < sh_ptr[ch + 1]; t++) {
            int32_t g = sh_idx[t];
            while (u[at] != g) at++;  // child list is a sorted subsequence of u
            mp[w++] = pos[at];
          }
        }
      }
    }
    // dedup patterns
    std::vector<uint64_t> fh(nf);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nf; i++) {
      uint64_t h = mix(mix(mix(0x1234567ULL, fm[i]), fk[i]), fsrc[i]);
      int64_t c1 = 2 * i + 1;
      uint64_t l0 = L == 0 ? fsrc[i] : sh_ptr[2 * i + 1] - sh_ptr[2 * i];
      uint64_t two = (L > 0 && c1 < lsize[L - 1]) ? 1 : 0;
      h = mix(mix(h, l0), two);
      for (int64_t t = mptr[i]; t < mptr[i + 1]; t++) h = mix(h, (uint64_t)fmap[t]);
      fh[i] = h;
    }
    lv.pattern_of.resize(nf);
    lv.piv_off.resize(nf);
    std::unordered_map<uint64_t, std::vector<int32_t>> buckets;
    std::vector<int64_t> pat_rep;  // representative front of each pattern
    for (int64_t i = 0; i < nf; i++) {
      lv.piv_off[i] = count[node_base[L] + i];
      int32_t nsrc = 1, len0 = fsrc[i], len1 = 0;
      if (L > 0) {
        len0 = (int32_t)(sh_ptr[2 * i + 1] - sh_ptr[2 * i]);
        if (2 * i + 1 < lsize[L - 1]) { nsrc = 2; len1 = fsrc[i] - len0; }
      }
      auto& bucket = buckets[fh[i]];
      int32_t found = -1;
      for (int32_t pid : bucket) {
        const int32_t* pr = lv.pat.data() + (int64_t)pid * TF_PAT_WIDTH;
        if (pr[TF_PAT_M] != fm[i] || pr[TF_PAT_K] != fk[i] || pr[TF_PAT_NSRC] != nsrc ||
            pr[TF_PAT_LEN0] != len0 || pr[TF_PAT_LEN1] != len1)
          continue;
        if (std::memcmp(lv.maps.data() + pr[TF_PAT_OFF0], fmap.data() + mptr[i],
                        sizeof(int32_t) * fsrc[i]) != 0)
          continue;
        found = pid;
        break;
      }
      if (found < 0) {
        found = lv.n_patterns++;
        int32_t off0 = (int32_t)lv.maps.size();
        lv.maps.insert(lv.maps.end(), fmap.begin() + mptr[i], fmap.begin() + mptr[i + 1]);
        // inverse (gather) maps: front position -> source position, -1 when absent
        int32_t ioff = (int32_t)lv.maps.size();
        lv.maps.insert(lv.maps.end(), (size_t)fm[i] * nsrc, -1);
        for (int c = 0; c < nsrc; c++) {
          const int32_t* fwd = fmap.data() + mptr[i] + (c == 0 ? 0 : len0);
          const int32_t len = c == 0 ? len0 : len1;
          for (int32_t a = 0; a < len; a++) lv.maps[ioff + (size_t)c * fm[i] + fwd[a]] = a;
        }
        // panel row stride: k rounded up to kp_align (2: rows stay 16-byte
        // aligned for cp.async / vector loads; TFB_KP_ALIGN=4 is the round-1 layout)
        const int32_t kp = (fk[i] + kp_align() - 1) / kp_align() * kp_align();
        // scatter table for the shared-memory front kernels (small fronts)
        int32_t soff = -1;
        if (fm[i] <= kScatterMaxM) {
          soff = (int32_t)lv.maps.size();
          const int64_t m = fm[i], k = fk[i], u = m - k, tk = k * (k + 1) / 2, ks = kp + 1;
          auto pos = [&](int64_t R, int64_t C) -> int32_t {  // C <= R
            if (R < k) return (int32_t)(R * (R + 1) / 2 + C);
            if (C < k) return (int32_t)(tk + (R - k) * ks + C);
            return (int32_t)(tk + u * ks + (R - k) * (R - k + 1) / 2 + (C - k));
          };
          for (int c = 0; c < nsrc; c++) {
            const int32_t* fwd = fmap.data() + mptr[i] + (c == 0 ? 0 : len0);
            const int32_t len = c == 0 ? len0 : len1;
            for (int32_t a = 0; a < len; a++)
              for (int32_t b = 0; b <= a; b++) {
                const int64_t R = std::max(fwd[a], fwd[b]), C = std::min(fwd[a], fwd[b]);
                lv.maps.push_back(pos(R, C));
              }
          }
        }
        int32_t row[TF_PAT_WIDTH] = {fm[i], fk[i], nsrc, len0, len1, off0, off0 + len0,
                                     L == 0 ? 1 : 0, ioff, kp, fm[i] * kp + kp, soff};
        lv.pat.insert(lv.pat.end(), row, row + TF_PAT_WIDTH);
        bucket.push_back(found);
        lv.max_m = std::max(lv.max_m, fm[i]);
        lv.max_k = std::max(lv.max_k, fk[i]);
        lv.max_upd = std::max(lv.max_upd, fm[i] - fk[i]);
      }
      lv.pattern_of[i] = found;
    }
    P->max_m = std::max(P->max_m, lv.max_m);
    P->max_k = std::max(P->max_k, lv.max_k);
    if (keep) {
      lv.list_ptr = std::move(fptr);
      lv.list_k = std::move(fk);
      lv.list_idx = std::move(flist);
    }
    sh_ptr.swap(sh_ptr_next);
    sh_idx.swap(sh_idx_next);
  }
  *out = P;
  return TF_OK;
}

extern "C" void tf_plan_destroy(tf_plan* plan) { delete plan; }

extern "C" int tf_plan_summary_get(const tf_plan* P, tf_plan_summary* s) {
  if (!P || !s) return TF_ERR_INVALID;
  s->n_dof = P->n_dof;
  s->n_leaves = P->n_leaves;
  s->n_nodes = P->n_nodes;
  s->n_pivots = P->n_pivots;
  s->n_levels = P->n_levels;
  s->max_m = P->max_m;
  s->max_k = P->max_k;
  s->keep_lists = P->keep;
  return TF_OK;
}

extern "C" int tf_plan_level(const tf_plan* P, int32_t L, tf_level_host* o) {
  if (!P || !o || L < 0 || L >= P->n_levels) return TF_ERR_INVALID;
  const Level& lv = P->levels[L];
  o->level = L;
  o->n_fronts = lv.n_fronts;
  o->n_patterns = lv.n_patterns;
  o->max_m = lv.max_m;
  o->max_k = lv.max_k;
  o->max_upd = lv.max_upd;
  o->node_base = lv.node_base;
  o->piv_base = lv.piv_base;
  o->n_pivots = lv.n_pivots;
  o->maps_len = (int64_t)lv.maps.size();
  o->pattern_of = lv.pattern_of.data();
  o->piv_off = lv.piv_off.data();
  o->pat = lv.pat.data();
  o->maps = lv.maps.data();
  return TF_OK;
}

extern "C" int tf_plan_pivot_order(const tf_plan* P, int32_t* out) {
  if (!P || !out) return TF_ERR_INVALID;
  std::memcpy(out, P->pivot_order.data(), sizeof(int32_t) * P->pivot_order.size());
  return TF_OK;
}

extern "C" int64_t tf_plan_node_lists_len(const tf_plan* P, int32_t L) {
  if (!P || L < 0 || L >= P->n_levels || !P->keep) return -1;
  return (int64_t)P->levels[L].list_idx.size();
}

extern "C" int tf_plan_node_lists(const tf_plan* P, int32_t L, int64_t* ptr, int32_t* k,
                                  int32_t* idx) {
  if (!P || L < 0 || L >= P->n_levels || !P->keep) return TF_ERR_INVALID;
  const Level& lv = P->levels[L];
  if (ptr) std::memcpy(ptr, lv.list_ptr.data(), sizeof(int64_t) * lv.list_ptr.size());
  if (k) std::memcpy(k, lv.list_k.data(), sizeof(int32_t) * lv.list_k.size());
  if (idx) std::memcpy(idx, lv.list_idx.data(), sizeof(int32_t) * lv.list_idx.size());
  return TF_OK;
}

// ---------------------------------------------------------------------------
// Canonical atomic Diekert graph + Foata normal form, streamed.
//
// Replaces enumerate_tasks / build_dependency_edges (tasks.py:162-252) and
// compute_fnf (schedule.py:60-82) for statistics and validation.  The graph
// is never materialised: walking the pivot steps in elimination order, every
// task's class follows from its predecessors' classes, which are final by
// then.
//   Assert(c)   = 1 + class(last Sub on c)      (1 when c is never updated)
//   Div(z,y)    = 1 + max(Assert(z,y), Assert(z,z))                J1
//   Mul(z,x,y)  = 1 + max(Div(z,y), Assert(x,z))                   J2
//   Sub(z,x,y)  = 1 + max(Mul(z,x,y), previous Sub on (x,y))       J3
// An Assert of row/column z is read only at step z, after which no step
// touches that row or column again (z leaves every active set), so its class
// is final when read (J4).  Per-pivot active sets come from the same boolean
// dense-front simulation as symbolic.py's EliminationPlan._structure: a
// front's pattern is the OR of its sources' patterns, and each pivot ORs its
// fill clique (tasks.py:142-150) into the trailing block.
namespace {

struct CellTable {  // open addressing (x,y) -> class of the last Sub (0: none)
  std::vector<uint64_t> keys;
  std::vector<int32_t> vals;
  uint64_t mask = 0;
  int64_t used = 0;
  explicit CellTable(int64_t hint) {
    uint64_t cap = 1024;
    while (cap < (uint64_t)(hint * 2)) cap <<= 1;
    keys.assign(cap, ~0ULL);
    vals.assign(cap, 0);
    mask = cap - 1;
  }
  void grow() {
    std::vector<uint64_t> ok;
    std::vector<int32_t> ov;
    ok.swap(keys);
    ov.swap(vals);
    keys.assign(ok.size() * 2, ~0ULL);
    vals.assign(ok.size() * 2, 0);
    mask = keys.size() - 1;
    used = 0;
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != ~0ULL) slot(ok[i]) = ov[i];
  }
  int32_t& slot(uint64_t key) {
    uint64_t h = mix(0, key) & mask;
    while (keys[h] != key) {
      if (keys[h] == ~0ULL) {
        if ((uint64_t)(used + 1) * 10 > keys.size() * 7) {
          grow();
          return slot(key);
        }
        keys[h] = key;
        ++used;
        break;
      }
      h = (h + 1) & mask;
    }
    return vals[h];
  }
  int32_t& at(int32_t x, int32_t y) { return slot(((uint64_t)(uint32_t)x << 32) | (uint32_t)y); }
};

}  // namespace

extern "C" int tf_atomic_fnf(const tf_plan* P, tf_fnf_stats* st, int64_t* widths, int32_t* kinds,
                             int32_t cap) {
  if (!P || !st) return TF_ERR_INVALID;
  if (!P->keep) return TF_ERR_INVALID;  // needs the per-node index lists
  std::memset(st, 0, sizeof(*st));
  std::vector<int64_t> w;
  std::vector<int32_t> kd;
  auto bump = [&](int32_t c, int kind, int64_t cnt) {
    if ((size_t)c > w.size()) {
      w.resize(c, 0);
      kd.resize(c, 0);
    }
    w[c - 1] += cnt;
    kd[c - 1] |= 1 << (kind - 1);
  };
  int64_t n_edges = 0, n_steps_tasks = 0;
  CellTable cells(P->n_dof * 16);
  std::vector<std::vector<uint8_t>> prev, cur;
  std::vector<std::pair<int32_t, int32_t>> act;  // (global, position)
  std::vector<int32_t> divc;
  for (int32_t L = 0; L < P->n_levels; ++L) {
    const Level& lv = P->levels[L];
    cur.assign(lv.n_fronts, {});
    for (int32_t i = 0; i < lv.n_fronts; ++i) {
      const int32_t* row = &lv.pat[(size_t)lv.pattern_of[i] * TF_PAT_WIDTH];
      const int32_t m = row[TF_PAT_M], k = row[TF_PAT_K], nsrc = row[TF_PAT_NSRC];
      std::vector<uint8_t> B((size_t)m * m, 0);
      for (int32_t c = 0; c < nsrc; ++c) {
        const int32_t* mp = &lv.maps[row[TF_PAT_OFF0 + c]];
        const int32_t len = row[TF_PAT_LEN0 + c];
        const uint8_t* src = L == 0 ? nullptr : prev[2 * (size_t)i + c].data();
        for (int32_t a = 0; a < len; ++a)
          for (int32_t b = 0; b < len; ++b)
            if (!src || src[(size_t)a * len + b]) B[(size_t)mp[a] * m + mp[b]] = 1;
      }
      const int32_t* lst = &lv.list_idx[lv.list_ptr[i]];
      for (int32_t c = 0; c < k; ++c) {
        const int32_t z = lst[c];
        if (!B[(size_t)c * m + c]) {
          st->singular = z;
          return TF_ERR_STRAY;
        }
        act.clear();
        for (int32_t j = c + 1; j < m; ++j)
          if (B[(size_t)c * m + j]) act.emplace_back(lst[j], j);
        std::sort(act.begin(), act.end());
        const int64_t a = (int64_t)act.size();
        n_steps_tasks += a + 2 * a * a;
        st->n_divisions += a;
        st->n_multiplications += a * a;
        const int32_t azz = 1 + cells.at(z, z);
        divc.resize(a);
        for (int64_t q = 0; q < a; ++q) {
          divc[q] = 1 + std::max(1 + cells.at(z, act[q].first), azz);
          bump(divc[q], 1, 1);
        }
        n_edges += 2 * a + 3 * a * a;  // J1, J2 (two each), J3 Mul -> Sub
        for (int64_t p = 0; p < a; ++p) {
          const int32_t x = act[p].first;
          const int32_t axz = 1 + cells.at(x, z);
          for (int64_t q = 0; q < a; ++q) {
            const int32_t mul = 1 + std::max(divc[q], axz);
            bump(mul, 2, 1);
            int32_t& s = cells.at(x, act[q].first);
            if (s) ++n_edges;  // J3 chain
            s = 1 + std::max(mul, s);
            bump(s, 3, 1);
          }
        }
        for (int64_t p = 0; p < a; ++p) {  // fill clique
          const int32_t pp = act[p].second;
          for (int64_t q = 0; q < a; ++q) B[(size_t)pp * m + act[q].second] = 1;
        }
      }
      const int32_t u = m - k;
      cur[i].resize((size_t)u * u);
      for (int32_t r = 0; r < u; ++r)
        std::memcpy(&cur[i][(size_t)r * u], &B[(size_t)(k + r) * m + k], u);
    }
    prev.swap(cur);
  }
  for (size_t h = 0; h < cells.keys.size(); ++h) {
    if (cells.keys[h] == ~0ULL) continue;
    const int32_t s = cells.vals[h];
    if (s) ++n_edges;  // J4
    bump(1 + s, 4, 1);
  }
  st->n_cells = cells.used;
  st->n_tasks = cells.used + n_steps_tasks;
  st->n_edges = n_edges;
  st->n_classes = (int32_t)w.size();
  int64_t mx = 0;
  for (int64_t v : w) mx = std::max(mx, v);
  st->max_width = mx;
  if (widths && kinds) {
    if (cap < (int32_t)w.size()) return TF_ERR_INVALID;
    std::copy(w.begin(), w.end(), widths);
    std::copy(kd.begin(), kd.end(), kinds);
  }
  return TF_OK;
}
