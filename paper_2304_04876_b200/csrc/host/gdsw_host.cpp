// Host-side symbolic / setup runtime (see include/gdsw_host.h for the map of
// every entry point to the reference loop kernel it restates).
//
// Build: g++ -O2 -fPIC -shared -ffp-contract=off (no FMA contraction: the
// numeric routines here must round exactly like the reference's sequential
// loops, _kernels.py:12-16 compiles them without fastmath).
#include "../../../include/gdsw_host.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

using i64 = int64_t;
using VI = std::vector<i64>;

namespace {

thread_local std::string g_err;

struct Arr {
  int kind = 0;  // 0 int64, 1 f64, 2 f32
  VI i;
  std::vector<double> d;
  std::vector<float> f;
  i64 size() const { return kind == 0 ? (i64)i.size() : kind == 1 ? (i64)d.size() : (i64)f.size(); }
};

}  // namespace

struct gh_result {
  std::vector<Arr> arrs;
  void add(VI&& v) { Arr a; a.kind = 0; a.i = std::move(v); arrs.push_back(std::move(a)); }
  void add(std::vector<double>&& v) { Arr a; a.kind = 1; a.d = std::move(v); arrs.push_back(std::move(a)); }
  void add(std::vector<float>&& v) { Arr a; a.kind = 2; a.f = std::move(v); arrs.push_back(std::move(a)); }
};

#define GH_TRY(...)                                   \
  try {                                               \
    __VA_ARGS__;                                      \
    return 0;                                         \
  } catch (const std::exception& e) {                 \
    g_err = e.what();                                 \
    return 1;                                         \
  } catch (...) {                                     \
    g_err = "unknown host error";                     \
    return 1;                                         \
  }

namespace {

// ---------------------------------------------------------------------------
// small CSR pattern helpers
// ---------------------------------------------------------------------------
struct Pat {
  i64 n = 0;
  VI ptr, idx;
};

// BFS levels from root (reference: _kernels.py:209-226). level must be -1.
i64 bfs_levels(const Pat& p, i64 root, VI& level, VI& queue) {
  level[root] = 0;
  queue[0] = root;
  i64 head = 0, tail = 1;
  while (head < tail) {
    i64 v = queue[head++];
    for (i64 q = p.ptr[v]; q < p.ptr[v + 1]; ++q) {
      i64 w = p.idx[q];
      if (level[w] < 0) {
        level[w] = level[v] + 1;
        queue[tail++] = w;
      }
    }
  }
  return tail;
}

// rows x cols gather with relabelled columns, rows re-sorted
// (reference: _kernels.py:118-149). src gives the source entry position.
void gather(const i64* a_ptr, const i64* a_idx, const i64* rows, i64 m,
            const i64* col_map, VI& o_ptr, VI& o_idx, VI* o_src) {
  o_ptr.assign(m + 1, 0);
  for (i64 r = 0; r < m; ++r) {
    i64 i = rows[r], cnt = 0;
    for (i64 p = a_ptr[i]; p < a_ptr[i + 1]; ++p)
      if (col_map[a_idx[p]] >= 0) ++cnt;
    o_ptr[r + 1] = o_ptr[r] + cnt;
  }
  o_idx.resize(o_ptr[m]);
  if (o_src) o_src->resize(o_ptr[m]);
  std::vector<std::pair<i64, i64>> tmp;
  for (i64 r = 0; r < m; ++r) {
    i64 i = rows[r], t = o_ptr[r];
    bool sorted = true;
    i64 last = -1;
    for (i64 p = a_ptr[i]; p < a_ptr[i + 1]; ++p) {
      i64 lc = col_map[a_idx[p]];
      if (lc >= 0) {
        if (lc < last) sorted = false;
        last = lc;
        o_idx[t] = lc;
        if (o_src) (*o_src)[t] = p;
        ++t;
      }
    }
    if (!sorted) {
      i64 lo = o_ptr[r], hi = o_ptr[r + 1];
      tmp.clear();
      for (i64 q = lo; q < hi; ++q) tmp.emplace_back(o_idx[q], o_src ? (*o_src)[q] : 0);
      std::sort(tmp.begin(), tmp.end());
      for (i64 q = lo; q < hi; ++q) {
        o_idx[q] = tmp[q - lo].first;
        if (o_src) (*o_src)[q] = tmp[q - lo].second;
      }
    }
  }
}

// pattern of A + A^T with sorted rows (reference: local_solvers.py:61-70)
Pat symmetrize(i64 n, const i64* ptr, const i64* idx) {
  VI cnt(n + 1, 0);
  for (i64 i = 0; i < n; ++i)
    for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) {
      cnt[i + 1]++;
      cnt[idx[p] + 1]++;
    }
  for (i64 i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  VI all(cnt[n]);
  VI off(cnt.begin(), cnt.end() - 1);
  for (i64 i = 0; i < n; ++i)
    for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) {
      all[off[i]++] = idx[p];
      all[off[idx[p]]++] = i;
    }
  Pat s;
  s.n = n;
  s.ptr.assign(n + 1, 0);
  s.idx.reserve(all.size());
  for (i64 i = 0; i < n; ++i) {
    auto b = all.begin() + cnt[i], e = all.begin() + cnt[i + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    for (auto it = b; it != u; ++it) s.idx.push_back(*it);
    s.ptr[i + 1] = (i64)s.idx.size();
  }
  return s;
}

Pat extract(const Pat& p, const VI& sel) {
  // sel sorted ascending -> relabel monotone; gather keeps rows sorted
  VI cmap(p.n, -1);
  for (i64 k = 0; k < (i64)sel.size(); ++k) cmap[sel[k]] = k;
  Pat s;
  s.n = (i64)sel.size();
  gather(p.ptr.data(), p.idx.data(), sel.data(), s.n, cmap.data(), s.ptr, s.idx, nullptr);
  return s;
}

// ---------------------------------------------------------------------------
// nested dissection (reference: local_solvers.py:72-143)
// ---------------------------------------------------------------------------
std::vector<VI> components(const Pat& p) {
  i64 n = p.n;
  std::vector<char> visited(n, 0);
  std::vector<VI> comps;
  VI lev(n, -1), queue(std::max<i64>(n, 1));
  for (i64 start = 0; start < n; ++start) {
    if (visited[start]) continue;
    i64 reached = bfs_levels(p, start, lev, queue);
    VI comp(queue.begin(), queue.begin() + reached);
    std::sort(comp.begin(), comp.end());
    for (i64 v : comp) {
      visited[v] = 1;
      lev[v] = -1;
    }
    comps.push_back(std::move(comp));
  }
  return comps;
}

VI peripheral_levels(const Pat& sub) {
  i64 n = sub.n;
  VI lev(n, -1), queue(n);
  bfs_levels(sub, 0, lev, queue);
  i64 ecc = *std::max_element(lev.begin(), lev.end());
  for (int it = 0; it < 3; ++it) {
    i64 cand = -1;
    for (i64 v = 0; v < n; ++v)
      if (lev[v] == ecc) { cand = v; break; }
    VI lev2(n, -1);
    bfs_levels(sub, cand, lev2, queue);
    i64 ecc2 = *std::max_element(lev2.begin(), lev2.end());
    lev.swap(lev2);
    if (ecc2 <= ecc) break;
    ecc = ecc2;
  }
  return lev;
}

VI dissect(const Pat& p, i64 leaf) {
  i64 n = p.n;
  VI out;
  out.reserve(n);
  if (n <= leaf) {
    for (i64 i = 0; i < n; ++i) out.push_back(i);
    return out;
  }
  for (const VI& comp : components(p)) {
    i64 csz = (i64)comp.size();
    if (csz <= leaf) {
      out.insert(out.end(), comp.begin(), comp.end());
      continue;
    }
    Pat sub = extract(p, comp);
    VI lev = peripheral_levels(sub);
    // lexsort((arange, lev))[size // 2] has the (size//2)-th smallest level
    VI sorted_lev(lev);
    std::nth_element(sorted_lev.begin(), sorted_lev.begin() + csz / 2, sorted_lev.end());
    i64 sep = sorted_lev[csz / 2];
    VI h0, h1, hs;
    for (i64 v = 0; v < csz; ++v) {
      if (lev[v] < sep) h0.push_back(v);
      else if (lev[v] > sep) h1.push_back(v);
      else hs.push_back(v);
    }
    if (h0.empty() || h1.empty()) {
      out.insert(out.end(), comp.begin(), comp.end());
      continue;
    }
    // halves ordered by their first original vertex
    if (comp[h1[0]] < comp[h0[0]]) std::swap(h0, h1);
    for (const VI* half : {&h0, &h1}) {
      Pat inner = extract(sub, *half);
      VI r = dissect(inner, leaf);
      for (i64 k : r) out.push_back(comp[(*half)[k]]);
    }
    for (i64 v : hs) out.push_back(comp[v]);
  }
  return out;
}

// ---------------------------------------------------------------------------
// symbolic factorizations
// ---------------------------------------------------------------------------
VI elimination_tree(const Pat& s) {  // _kernels.py:233-248
  i64 n = s.n;
  VI parent(n, -1), ancestor(n, -1);
  for (i64 i = 0; i < n; ++i)
    for (i64 p = s.ptr[i]; p < s.ptr[i + 1]; ++p) {
      i64 k = s.idx[p];
      while (k != -1 && k < i) {
        i64 knext = ancestor[k];
        ancestor[k] = i;
        if (knext == -1) {
          parent[k] = i;
          k = -1;
        } else {
          k = knext;
        }
      }
    }
  return parent;
}

void lu_rows(const Pat& s, const VI& parent, VI& l_ptr, VI& l_idx) {  // _kernels.py:251-281
  i64 n = s.n;
  VI mark(n, -1);
  l_ptr.assign(n + 1, 0);
  l_idx.clear();
  for (i64 i = 0; i < n; ++i) {
    mark[i] = i;
    i64 start = (i64)l_idx.size();
    for (i64 p = s.ptr[i]; p < s.ptr[i + 1]; ++p) {
      i64 k = s.idx[p];
      while (k >= 0 && k < i && mark[k] != i) {
        mark[k] = i;
        l_idx.push_back(k);
        k = parent[k];
      }
    }
    std::sort(l_idx.begin() + start, l_idx.end());
    l_ptr[i + 1] = (i64)l_idx.size();
  }
}

void transpose_pattern(i64 n_rows, i64 n_cols, const i64* ptr, const i64* idx,
                       VI& t_ptr, VI& t_idx, VI& t_src) {  // _kernels.py:284-301
  i64 nnz = ptr[n_rows];
  t_ptr.assign(n_cols + 1, 0);
  for (i64 p = 0; p < nnz; ++p) t_ptr[idx[p] + 1]++;
  for (i64 j = 0; j < n_cols; ++j) t_ptr[j + 1] += t_ptr[j];
  t_idx.resize(nnz);
  t_src.resize(nnz);
  VI off(t_ptr.begin(), t_ptr.end() - 1);
  for (i64 i = 0; i < n_rows; ++i)
    for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) {
      i64 t = off[idx[p]]++;
      t_idx[t] = i;
      t_src[t] = p;
    }
}

Pat permute_sym(i64 n, const i64* ptr, const i64* idx, const i64* perm) {
  VI inv(n);
  for (i64 i = 0; i < n; ++i) inv[perm[i]] = i;
  Pat p;
  p.n = n;
  gather(ptr, idx, perm, n, inv.data(), p.ptr, p.idx, nullptr);
  return p;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* gh_last_error(void) { return g_err.c_str(); }
int64_t gh_result_count(const gh_result* r) { return (int64_t)r->arrs.size(); }
int64_t gh_result_size(const gh_result* r, int64_t k) { return r->arrs.at(k).size(); }
int gh_result_kind(const gh_result* r, int64_t k) { return r->arrs.at(k).kind; }
int gh_result_copy(const gh_result* r, int64_t k, void* dst) {
  const Arr& a = r->arrs.at(k);
  if (a.kind == 0) std::memcpy(dst, a.i.data(), a.i.size() * sizeof(i64));
  else if (a.kind == 1) std::memcpy(dst, a.d.data(), a.d.size() * sizeof(double));
  else std::memcpy(dst, a.f.data(), a.f.size() * sizeof(float));
  return 0;
}
void gh_result_free(gh_result* r) { delete r; }

int gh_node_graph(int64_t n_nodes, int64_t dpn, const int64_t* a_ptr,
                  const int64_t* a_idx, gh_result** out) {
  GH_TRY({
    VI marker(n_nodes, -1), ptr(n_nodes + 1, 0), idx;
    for (i64 u = 0; u < n_nodes; ++u) {
      i64 start = (i64)idx.size();
      for (i64 d = u * dpn; d < (u + 1) * dpn; ++d)
        for (i64 p = a_ptr[d]; p < a_ptr[d + 1]; ++p) {
          i64 v = a_idx[p] / dpn;
          if (marker[v] != u) {
            marker[v] = u;
            idx.push_back(v);
          }
        }
      std::sort(idx.begin() + start, idx.end());
      ptr[u + 1] = (i64)idx.size();
    }
    auto* r = new gh_result;
    r->add(std::move(ptr));
    r->add(std::move(idx));
    *out = r;
  })
}

int gh_expand_layers(int64_t n, const int64_t* g_ptr, const int64_t* g_idx,
                     uint8_t* mask, int64_t layers) {
  GH_TRY({
    VI frontier, nxt;
    for (i64 v = 0; v < n; ++v)
      if (mask[v]) frontier.push_back(v);
    for (i64 l = 0; l < layers; ++l) {
      nxt.clear();
      for (i64 v : frontier)
        for (i64 p = g_ptr[v]; p < g_ptr[v + 1]; ++p) {
          i64 w = g_idx[p];
          if (!mask[w]) {
            mask[w] = 1;
            nxt.push_back(w);
          }
        }
      frontier.swap(nxt);
      if (frontier.empty()) break;
    }
  })
}

// overlap node sets of the listed subdomains: seeds = nodes owned by s,
// grown by `layers` graph layers (same sets as extend_overlap,
// decomposition.py:150-166), without a full-size mask per subdomain
int gh_overlap_sets(int64_t n_nodes, const int64_t* g_ptr, const int64_t* g_idx,
                    const int64_t* node_owner, int64_t n_parts, int64_t n_subs,
                    const int64_t* subs, int64_t layers, gh_result** out) {
  GH_TRY({
    VI cnt(n_parts + 1, 0);
    for (i64 u = 0; u < n_nodes; ++u) cnt[node_owner[u] + 1]++;
    for (i64 s = 0; s < n_parts; ++s) cnt[s + 1] += cnt[s];
    VI byown(n_nodes), off(cnt.begin(), cnt.end() - 1);
    for (i64 u = 0; u < n_nodes; ++u) byown[off[node_owner[u]]++] = u;
    VI stamp(n_nodes, -1), ptr(1, 0), nodes, frontier, nxt;
    for (i64 t = 0; t < n_subs; ++t) {
      const i64 s = subs[t];
      const i64 start = (i64)nodes.size();
      frontier.assign(byown.begin() + cnt[s], byown.begin() + cnt[s + 1]);
      for (i64 u : frontier) {
        stamp[u] = t;
        nodes.push_back(u);
      }
      for (i64 l = 0; l < layers; ++l) {
        nxt.clear();
        for (i64 v : frontier)
          for (i64 p = g_ptr[v]; p < g_ptr[v + 1]; ++p) {
            i64 w = g_idx[p];
            if (stamp[w] != t) {
              stamp[w] = t;
              nxt.push_back(w);
              nodes.push_back(w);
            }
          }
        frontier.swap(nxt);
        if (frontier.empty()) break;
      }
      std::sort(nodes.begin() + start, nodes.end());
      ptr.push_back((i64)nodes.size());
    }
    auto* r = new gh_result;
    r->add(std::move(ptr));
    r->add(std::move(nodes));
    *out = r;
  })
}

int gh_nested_dissection(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                         int64_t leaf_size, int64_t* perm_out) {
  GH_TRY({
    Pat s = symmetrize(n, a_ptr, a_idx);
    VI perm = dissect(s, leaf_size);
    if ((i64)perm.size() != n) throw std::runtime_error("nested dissection lost vertices");
    std::copy(perm.begin(), perm.end(), perm_out);
  })
}

int gh_symbolic_lu(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                   const int64_t* perm, gh_result** out) {
  GH_TRY({
    Pat p = permute_sym(n, a_ptr, a_idx, perm);
    Pat s = symmetrize(n, p.ptr.data(), p.idx.data());
    VI parent = elimination_tree(s);
    VI l_ptr, l_idx;
    lu_rows(s, parent, l_ptr, l_idx);
    VI t_ptr, t_idx, t_src;
    transpose_pattern(n, n, l_ptr.data(), l_idx.data(), t_ptr, t_idx, t_src);
    VI u_ptr(n + 1, 0), u_idx;
    u_idx.reserve(t_idx.size() + n);
    for (i64 i = 0; i < n; ++i) {
      u_idx.push_back(i);
      for (i64 q = t_ptr[i]; q < t_ptr[i + 1]; ++q) u_idx.push_back(t_idx[q]);
      u_ptr[i + 1] = (i64)u_idx.size();
    }
    auto* r = new gh_result;
    r->add(std::move(l_ptr));
    r->add(std::move(l_idx));
    r->add(std::move(u_ptr));
    r->add(std::move(u_idx));
    *out = r;
  })
}

int gh_symbolic_iluk(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                     const int64_t* perm, int64_t fill_level, gh_result** out) {
  GH_TRY({
    Pat p = permute_sym(n, a_ptr, a_idx, perm);
    const i64 HEAD = n;
    VI nxt(n + 1), lev(n);
    VI l_ptr(n + 1, 0), u_ptr(n + 1, 0), l_cols, u_cols, u_lev;
    l_cols.reserve(p.idx.size());
    u_cols.reserve(p.idx.size());
    u_lev.reserve(p.idx.size());
    for (i64 i = 0; i < n; ++i) {
      i64 prev = HEAD;
      nxt[HEAD] = n;
      bool seen_diag = false;
      for (i64 q = p.ptr[i]; q < p.ptr[i + 1]; ++q) {
        i64 j = p.idx[q];
        if (j == i) seen_diag = true;
        nxt[prev] = j;
        nxt[j] = n;
        lev[j] = 0;
        prev = j;
      }
      if (!seen_diag) {
        i64 s = HEAD;
        while (nxt[s] < i) s = nxt[s];
        nxt[i] = nxt[s];
        nxt[s] = i;
        lev[i] = 0;
      }
      i64 k = nxt[HEAD];
      while (k < i) {
        i64 lev_ik = lev[k], scan = k;
        for (i64 q = u_ptr[k]; q < u_ptr[k + 1]; ++q) {
          i64 j = u_cols[q];
          if (j <= k) continue;
          i64 nl = lev_ik + u_lev[q] + 1;
          if (nl > fill_level) continue;
          while (nxt[scan] < j) scan = nxt[scan];
          if (nxt[scan] == j) {
            if (nl < lev[j]) lev[j] = nl;
          } else {
            nxt[j] = nxt[scan];
            nxt[scan] = j;
            lev[j] = nl;
          }
        }
        k = nxt[k];
      }
      for (i64 j = nxt[HEAD]; j < n; j = nxt[j]) {
        if (j < i) {
          l_cols.push_back(j);
        } else {
          u_cols.push_back(j);
          u_lev.push_back(lev[j]);
        }
      }
      l_ptr[i + 1] = (i64)l_cols.size();
      u_ptr[i + 1] = (i64)u_cols.size();
    }
    auto* r = new gh_result;
    r->add(std::move(l_ptr));
    r->add(std::move(l_cols));
    r->add(std::move(u_ptr));
    r->add(std::move(u_cols));
    *out = r;
  })
}

int gh_level_schedule(int64_t n, const int64_t* ptr, const int64_t* idx, int upper,
                      int64_t* level_out, gh_result** out) {
  GH_TRY({
    VI level(n, 0);
    if (!upper) {
      for (i64 i = 0; i < n; ++i) {
        i64 lv = 0;
        for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) lv = std::max(lv, level[idx[p]] + 1);
        level[i] = lv;
      }
    } else {
      for (i64 i = n - 1; i >= 0; --i) {
        i64 lv = 0;
        for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) {
          i64 j = idx[p];
          if (j > i) lv = std::max(lv, level[j] + 1);
        }
        level[i] = lv;
      }
    }
    i64 nlev = 0;
    for (i64 i = 0; i < n; ++i) nlev = std::max(nlev, level[i] + 1);
    VI lptr(nlev + 1, 0), rows(n);
    for (i64 i = 0; i < n; ++i) lptr[level[i] + 1]++;
    for (i64 l = 0; l < nlev; ++l) lptr[l + 1] += lptr[l];
    VI off(lptr.begin(), lptr.end() - 1);
    for (i64 i = 0; i < n; ++i) rows[off[level[i]]++] = i;  // stable argsort
    if (level_out) std::copy(level.begin(), level.end(), level_out);
    auto* r = new gh_result;
    r->add(std::move(lptr));
    r->add(std::move(rows));
    *out = r;
  })
}

int gh_csr_gather(int64_t m, const int64_t* a_ptr, const int64_t* a_idx,
                  const int64_t* rows, const int64_t* col_map, gh_result** out) {
  GH_TRY({
    VI o_ptr, o_idx, o_src;
    gather(a_ptr, a_idx, rows, m, col_map, o_ptr, o_idx, &o_src);
    auto* r = new gh_result;
    r->add(std::move(o_ptr));
    r->add(std::move(o_idx));
    r->add(std::move(o_src));
    *out = r;
  })
}

int gh_transpose_pattern(int64_t n_rows, int64_t n_cols, const int64_t* ptr,
                         const int64_t* idx, gh_result** out) {
  GH_TRY({
    VI t_ptr, t_idx, t_src;
    transpose_pattern(n_rows, n_cols, ptr, idx, t_ptr, t_idx, t_src);
    auto* r = new gh_result;
    r->add(std::move(t_ptr));
    r->add(std::move(t_idx));
    r->add(std::move(t_src));
    *out = r;
  })
}

}  // extern "C"

namespace {
// Gustavson keeping computed zeros; rows sorted by column afterwards
// (reference: _kernels.py:51-94 and sparse_core.py:207-228).
template <typename T>
void spgemm(i64 n_rows, i64 n_cols, const i64* a_ptr, const i64* a_idx, const T* a_val,
            const i64* b_ptr, const i64* b_idx, const T* b_val, gh_result* r) {
  VI marker(n_cols, -1), o_ptr(n_rows + 1, 0), o_idx, row_cols;
  std::vector<T> acc(n_cols, T(0)), o_val;
  for (i64 i = 0; i < n_rows; ++i) {
    row_cols.clear();
    for (i64 p = a_ptr[i]; p < a_ptr[i + 1]; ++p) {
      i64 k = a_idx[p];
      T a_ik = a_val[p];
      for (i64 q = b_ptr[k]; q < b_ptr[k + 1]; ++q) {
        i64 j = b_idx[q];
        if (marker[j] != i) {
          marker[j] = i;
          acc[j] = a_ik * b_val[q];
          row_cols.push_back(j);
        } else {
          acc[j] += a_ik * b_val[q];
        }
      }
    }
    std::sort(row_cols.begin(), row_cols.end());
    for (i64 j : row_cols) {
      o_idx.push_back(j);
      o_val.push_back(acc[j]);
    }
    o_ptr[i + 1] = (i64)o_idx.size();
  }
  r->add(std::move(o_ptr));
  r->add(std::move(o_idx));
  r->add(std::move(o_val));
}

// IKJ numeric LU restricted to the pattern (reference: _kernels.py:429-466)
template <typename T>
i64 lu_numeric(i64 n, const i64* l_ptr, const i64* l_idx, const i64* u_ptr, const i64* u_idx,
               const i64* a_ptr, const i64* a_idx, const T* a_val, T* l_val, T* u_val,
               double pivot_tol) {
  std::vector<T> w(n, T(0));
  VI stamp(n, -1);
  for (i64 i = 0; i < n; ++i) {
    for (i64 p = l_ptr[i]; p < l_ptr[i + 1]; ++p) { stamp[l_idx[p]] = i; w[l_idx[p]] = T(0); }
    for (i64 p = u_ptr[i]; p < u_ptr[i + 1]; ++p) { stamp[u_idx[p]] = i; w[u_idx[p]] = T(0); }
    for (i64 p = a_ptr[i]; p < a_ptr[i + 1]; ++p)
      if (stamp[a_idx[p]] == i) w[a_idx[p]] = a_val[p];
    for (i64 p = l_ptr[i]; p < l_ptr[i + 1]; ++p) {
      i64 k = l_idx[p];
      T u_kk = u_val[u_ptr[k]];
      T l_ik = w[k] / u_kk;
      w[k] = l_ik;
      for (i64 q = u_ptr[k] + 1; q < u_ptr[k + 1]; ++q) {
        i64 j = u_idx[q];
        if (stamp[j] == i) w[j] -= l_ik * u_val[q];
      }
    }
    // numba compares abs(w[i]) (element type) against the float64 tolerance
    if ((double)std::fabs(w[i]) <= pivot_tol) return i + 1;
    for (i64 p = l_ptr[i]; p < l_ptr[i + 1]; ++p) l_val[p] = w[l_idx[p]];
    for (i64 p = u_ptr[i]; p < u_ptr[i + 1]; ++p) u_val[p] = w[u_idx[p]];
  }
  return 0;
}
}  // namespace

extern "C" {

int gh_spgemm_f64(int64_t n_rows, int64_t n_cols, const int64_t* a_ptr, const int64_t* a_idx,
                  const double* a_val, const int64_t* b_ptr, const int64_t* b_idx,
                  const double* b_val, gh_result** out) {
  GH_TRY({
    auto* r = new gh_result;
    spgemm<double>(n_rows, n_cols, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val, r);
    *out = r;
  })
}

int gh_spgemm_f32(int64_t n_rows, int64_t n_cols, const int64_t* a_ptr, const int64_t* a_idx,
                  const float* a_val, const int64_t* b_ptr, const int64_t* b_idx,
                  const float* b_val, gh_result** out) {
  GH_TRY({
    auto* r = new gh_result;
    spgemm<float>(n_rows, n_cols, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val, r);
    *out = r;
  })
}

int64_t gh_lu_numeric_f64(int64_t n, const int64_t* l_ptr, const int64_t* l_idx,
                          const int64_t* u_ptr, const int64_t* u_idx, const int64_t* a_ptr,
                          const int64_t* a_idx, const double* a_val, double* l_val,
                          double* u_val, double pivot_tol) {
  return lu_numeric<double>(n, l_ptr, l_idx, u_ptr, u_idx, a_ptr, a_idx, a_val, l_val, u_val,
                            pivot_tol);
}

int64_t gh_lu_numeric_f32(int64_t n, const int64_t* l_ptr, const int64_t* l_idx,
                          const int64_t* u_ptr, const int64_t* u_idx, const int64_t* a_ptr,
                          const int64_t* a_idx, const float* a_val, float* l_val,
                          float* u_val, double pivot_tol) {
  return lu_numeric<float>(n, l_ptr, l_idx, u_ptr, u_idx, a_ptr, a_idx, a_val, l_val, u_val,
                           pivot_tol);
}

int gh_spmv_f64(int64_t n, const int64_t* ptr, const int64_t* idx, const double* val,
                const double* x, double* y, double alpha, double beta) {
  GH_TRY({
    for (i64 i = 0; i < n; ++i) {
      double acc = 0.0;
      for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) acc += val[p] * x[idx[p]];
      y[i] = alpha * acc + beta * y[i];
    }
  })
}

int gh_spmv_f32(int64_t n, const int64_t* ptr, const int64_t* idx, const float* val,
                const float* x, float* y, float alpha, float beta) {
  GH_TRY({
    for (i64 i = 0; i < n; ++i) {
      float acc = 0.0f;
      for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) acc += val[p] * x[idx[p]];
      y[i] = alpha * acc + beta * y[i];
    }
  })
}

int gh_align_pattern(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                     const int64_t* f_ptr, const int64_t* f_idx, int64_t* out) {
  GH_TRY({
    for (i64 i = 0; i < n; ++i) {
      i64 p = a_ptr[i], pe = a_ptr[i + 1];
      for (i64 t = f_ptr[i]; t < f_ptr[i + 1]; ++t) {
        i64 j = f_idx[t];
        while (p < pe && a_idx[p] < j) ++p;
        out[t] = (p < pe && a_idx[p] == j) ? p : -1;
      }
    }
  })
}

int gh_fastilu_plan(int64_t n, const int64_t* l_ptr, const int64_t* l_idx,
                    const int64_t* u_ptr, const int64_t* u_idx, const int64_t* a_ptr,
                    const int64_t* a_idx, gh_result** out) {
  GH_TRY({
    VI uc_ptr, uc_rows, uc_src;
    transpose_pattern(n, n, u_ptr, u_idx, uc_ptr, uc_rows, uc_src);
    // bounded merge of L row i with U column j, k < bound (_kernels.py:547-571)
    auto merge = [&](i64 i, i64 j, i64 bound, VI& pl, VI& pu) {
      i64 p = l_ptr[i], pe = l_ptr[i + 1], q = uc_ptr[j], qe = uc_ptr[j + 1];
      while (p < pe && q < qe) {
        i64 kl = l_idx[p];
        if (kl >= bound) break;
        i64 ku = uc_rows[q];
        if (ku >= bound) break;
        if (kl == ku) {
          pl.push_back(p);
          pu.push_back(uc_src[q]);
          ++p;
          ++q;
        } else if (kl < ku) {
          ++p;
        } else {
          ++q;
        }
      }
    };
    i64 nl = l_ptr[n], nu = u_ptr[n];
    VI e_ptr(nl + nu + 1, 0), pair_l, pair_u;
    for (i64 i = 0; i < n; ++i)
      for (i64 p = l_ptr[i]; p < l_ptr[i + 1]; ++p) {
        i64 j = l_idx[p];
        merge(i, j, j, pair_l, pair_u);
        e_ptr[p + 1] = (i64)pair_l.size();
      }
    for (i64 i = 0; i < n; ++i)
      for (i64 p = u_ptr[i]; p < u_ptr[i + 1]; ++p) {
        merge(i, u_idx[p], i, pair_l, pair_u);
        e_ptr[nl + p + 1] = (i64)pair_l.size();
      }
    // residual plan over A's pattern (_kernels.py:598-617)
    VI l_of_a(a_ptr[n]), u_of_a(a_ptr[n]);
    for (i64 i = 0; i < n; ++i) {
      i64 lp = l_ptr[i], up = u_ptr[i];
      for (i64 p = a_ptr[i]; p < a_ptr[i + 1]; ++p) {
        i64 j = a_idx[p];
        while (lp < l_ptr[i + 1] && l_idx[lp] < j) ++lp;
        l_of_a[p] = (lp < l_ptr[i + 1] && l_idx[lp] == j) ? lp : -1;
        while (up < u_ptr[i + 1] && u_idx[up] < j) ++up;
        u_of_a[p] = (up < u_ptr[i + 1] && u_idx[up] == j) ? up : -1;
      }
    }
    i64 na = a_ptr[n];
    VI r_ptr(na + 1, 0), r_l, r_u, tail_l(na), tail_u(na);
    for (i64 i = 0; i < n; ++i)
      for (i64 p = a_ptr[i]; p < a_ptr[i + 1]; ++p) {
        i64 j = a_idx[p];
        merge(i, j, i < j ? i : j, r_l, r_u);
        r_ptr[p + 1] = (i64)r_l.size();
        if (i > j) {
          tail_l[p] = l_of_a[p];
          tail_u[p] = u_ptr[j];
        } else {
          tail_l[p] = -1;
          tail_u[p] = u_of_a[p];
        }
      }
    auto* r = new gh_result;
    r->add(std::move(e_ptr));
    r->add(std::move(pair_l));
    r->add(std::move(pair_u));
    r->add(std::move(r_ptr));
    r->add(std::move(r_l));
    r->add(std::move(r_u));
    r->add(std::move(tail_l));
    r->add(std::move(tail_u));
    *out = r;
  })
}

// Interface classification (reference: decomposition.py:173-250). Returns the
// connected pieces of interface nodes that share one closure set, with their
// kinds; the caller orders components by first dof.
int gh_classify_interface(int64_t n_nodes, const int64_t* g_ptr, const int64_t* g_idx,
                          const int64_t* node_owner, gh_result** out) {
  GH_TRY({
    VI key_of(n_nodes, -1);
    std::map<VI, i64> key_id;
    std::vector<VI> keys;
    VI iface, mult;
    VI tmp;
    for (i64 u = 0; u < n_nodes; ++u) {
      tmp.clear();
      tmp.push_back(node_owner[u]);
      for (i64 p = g_ptr[u]; p < g_ptr[u + 1]; ++p) tmp.push_back(node_owner[g_idx[p]]);
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      if (tmp.size() < 2) continue;
      auto it = key_id.find(tmp);
      i64 id;
      if (it == key_id.end()) {
        id = (i64)keys.size();
        key_id.emplace(tmp, id);
        keys.push_back(tmp);
      } else {
        id = it->second;
      }
      key_of[u] = id;
      iface.push_back(u);
      mult.push_back((i64)tmp.size());
    }
    // connected pieces inside each closure class (DFS over same-key nodes)
    VI piece_of(n_nodes, -1), piece_ptr(1, 0), piece_nodes, piece_key, stack;
    for (i64 u : iface) {
      if (piece_of[u] >= 0) continue;
      i64 pid = (i64)piece_key.size();
      i64 start = (i64)piece_nodes.size();
      stack.assign(1, u);
      piece_of[u] = pid;
      while (!stack.empty()) {
        i64 v = stack.back();
        stack.pop_back();
        piece_nodes.push_back(v);
        for (i64 p = g_ptr[v]; p < g_ptr[v + 1]; ++p) {
          i64 w = g_idx[p];
          if (piece_of[w] < 0 && key_of[w] == key_of[u]) {
            piece_of[w] = pid;
            stack.push_back(w);
          }
        }
      }
      std::sort(piece_nodes.begin() + start, piece_nodes.end());
      piece_ptr.push_back((i64)piece_nodes.size());
      piece_key.push_back(key_of[u]);
    }
    i64 np_ = (i64)piece_key.size();
    // piece adjacency + maximality clause
    std::vector<VI> adj(np_);
    for (i64 u : iface) {
      i64 pu = piece_of[u];
      for (i64 p = g_ptr[u]; p < g_ptr[u + 1]; ++p) {
        i64 pv = piece_of[g_idx[p]];
        if (pv >= 0 && pv != pu) adj[pu].push_back(pv);
      }
    }
    VI kind(np_), key_ptr(1, 0), key_flat;
    for (i64 pid = 0; pid < np_; ++pid) {
      const VI& key = keys[piece_key[pid]];
      i64 card = (i64)key.size();
      if (card == 2) {
        kind[pid] = 2;  // face
      } else if (card >= 5) {
        kind[pid] = 0;  // vertex
      } else {
        bool dominated = false;
        for (i64 q : adj[pid]) {
          const VI& other = keys[piece_key[q]];
          if (other.size() > key.size() &&
              std::includes(other.begin(), other.end(), key.begin(), key.end())) {
            dominated = true;
            break;
          }
        }
        kind[pid] = dominated ? 1 : 0;
      }
      key_flat.insert(key_flat.end(), key.begin(), key.end());
      key_ptr.push_back((i64)key_flat.size());
    }
    auto* r = new gh_result;
    r->add(std::move(iface));
    r->add(std::move(mult));
    r->add(std::move(piece_ptr));
    r->add(std::move(piece_nodes));
    r->add(std::move(key_ptr));
    r->add(std::move(key_flat));
    r->add(std::move(kind));
    *out = r;
  })
}

}  // extern "C"

// ===========================================================================
// supernodal partitioned inverses of exact-LU factors (the device solve of
// coarse_factor.cuh; Python restatement: coarse_factor._records_from_csr and
// _assemble, which the tests compare against this)
// ===========================================================================
#include <atomic>
#include <iterator>
#include <thread>

namespace {

inline void require_host(bool ok, const char* msg) {
  if (!ok) throw std::runtime_error(msg);
}

struct PinvSn {
  i64 level = 0, parent = -1;
  VI cols, rows;  // block-local ND positions, ascending
  std::vector<double> d, m, nm;
};

// dense row-major helpers
// inverse of a unit lower triangular s x s (strict lower part of a used):
// row i of the inverse = e_i - sum_{k<i} a[i][k] * (row k of the inverse),
// rows streamed contiguously
void tri_inv_unit_lower(i64 s, const std::vector<double>& a, std::vector<double>& inv) {
  inv.assign((size_t)s * s, 0.0);
  for (i64 i = 0; i < s; ++i) {
    double* ri = &inv[i * s];
    for (i64 k = 0; k < i; ++k) {
      const double f = a[i * s + k];
      if (f == 0.0) continue;
      const double* rk = &inv[k * s];
      for (i64 j = 0; j <= k; ++j) ri[j] -= f * rk[j];
    }
    ri[i] = 1.0;
  }
}

// inverse of an upper triangular s x s: row i = (e_i - sum_{k>i} a[i][k] *
// row k) / a[i][i], from the last row up
void tri_inv_upper(i64 s, const std::vector<double>& a, std::vector<double>& inv) {
  inv.assign((size_t)s * s, 0.0);
  for (i64 i = s - 1; i >= 0; --i) {
    double* ri = &inv[i * s];
    ri[i] = 1.0;
    for (i64 k = i + 1; k < s; ++k) {
      const double f = a[i * s + k];
      if (f == 0.0) continue;
      const double* rk = &inv[k * s];
      for (i64 j = k; j < s; ++j) ri[j] -= f * rk[j];
    }
    const double d = a[i * s + i];
    for (i64 j = i; j < s; ++j) ri[j] /= d;
  }
}

std::vector<PinvSn> pinv_block(i64 n, const i64* lp, const i64* li, const double* lv, const i64* up,
                               const i64* ui, const double* uv, i64 relax, double zf, bool with_values) {
  // strictly lower symmetrized column structure
  std::vector<VI> col(n);
  for (i64 i = 0; i < n; ++i)
    for (i64 p = lp[i]; p < lp[i + 1]; ++p) col[li[p]].push_back(i);
  for (i64 j = 0; j < n; ++j)
    for (i64 p = up[j]; p < up[j + 1]; ++p)
      if (ui[p] > j) col[j].push_back(ui[p]);
  VI cc(n), parent(n, -1);
  for (i64 j = 0; j < n; ++j) {
    std::sort(col[j].begin(), col[j].end());
    col[j].erase(std::unique(col[j].begin(), col[j].end()), col[j].end());
    cc[j] = (i64)col[j].size();
    if (cc[j]) parent[j] = col[j][0];
  }
  VI nchild(n, 0);
  for (i64 j = 0; j < n; ++j)
    if (parent[j] >= 0) nchild[parent[j]]++;
  VI starts{0};
  for (i64 j = 1; j < n; ++j) {
    const bool fund = parent[j - 1] == j && cc[j - 1] == cc[j] + 1 && nchild[j] == 1;
    if (!fund) starts.push_back(j);
  }
  starts.push_back(n);
  const i64 nsn = (i64)starts.size() - 1;
  VI sn_of(n);
  for (i64 k = 0; k < nsn; ++k)
    for (i64 j = starts[k]; j < starts[k + 1]; ++j) sn_of[j] = k;
  std::vector<VI> cols(nsn), rows(nsn);
  VI nnz_l(nsn, 0);
  for (i64 k = 0; k < nsn; ++k) {
    for (i64 j = starts[k]; j < starts[k + 1]; ++j) {
      cols[k].push_back(j);
      nnz_l[k] += cc[j];
    }
    for (i64 r : col[starts[k]])
      if (r >= starts[k + 1]) rows[k].push_back(r);
  }
  col.clear();
  col.shrink_to_fit();
  auto set_union = [](const VI& a, const VI& b) {
    VI o;
    o.reserve(a.size() + b.size());
    std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
    return o;
  };
  auto set_diff = [](const VI& a, const VI& b) {
    VI o;
    std::set_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
    return o;
  };
  VI par(nsn, -1);
  for (i64 k = 0; k < nsn; ++k) {  // extend-add containment
    if (rows[k].empty()) continue;
    const i64 p = sn_of[rows[k][0]];
    par[k] = p;
    VI above;
    for (i64 r : rows[k])
      if (r >= starts[p + 1]) above.push_back(r);
    VI extra = set_diff(above, rows[p]);
    if (!extra.empty()) rows[p] = set_union(rows[p], extra);
  }
  VI rep(nsn), nch(nsn, 0);
  std::iota(rep.begin(), rep.end(), 0);
  for (i64 k = 0; k < nsn; ++k)
    if (par[k] >= 0) nch[par[k]]++;
  auto find = [&](i64 k) {
    while (rep[k] != k) {
      rep[k] = rep[rep[k]];
      k = rep[k];
    }
    return k;
  };
  for (i64 k = 0; k < nsn; ++k) {
    if (par[k] < 0) continue;
    const i64 p = find(par[k]);
    const i64 sz = (i64)(cols[k].size() + cols[p].size());
    bool merge = sz <= relax;
    VI mrows;
    if (!merge && cols[p][0] == cols[k].back() + 1 && nch[p] == 1) {
      mrows = set_diff(set_union(rows[p], rows[k]), set_union(cols[p], cols[k]));
      const double dense = (double)sz * (sz - 1) / 2.0 + (double)sz * mrows.size();
      merge = dense > 0 && 1.0 - (double)(nnz_l[k] + nnz_l[p]) / dense <= zf;
    }
    if (merge) {
      cols[p] = set_union(cols[p], cols[k]);
      rows[p] = set_diff(set_union(rows[p], rows[k]), cols[p]);
      nnz_l[p] += nnz_l[k];
      nch[p] += nch[k] - 1;
      rep[k] = p;
      VI().swap(cols[k]);
      VI().swap(rows[k]);
    }
  }
  VI alive, newid(nsn, -1);
  for (i64 k = 0; k < nsn; ++k)
    if (rep[k] == k) {
      newid[k] = (i64)alive.size();
      alive.push_back(k);
    }
  const i64 nq = (i64)alive.size();
  std::vector<PinvSn> out(nq);
  VI sn_col(n), cpos(n);
  for (i64 q = 0; q < nq; ++q) {
    const i64 k = alive[q];
    out[q].cols = std::move(cols[k]);
    out[q].rows = std::move(rows[k]);
    for (size_t t = 0; t < out[q].cols.size(); ++t) {
      sn_col[out[q].cols[t]] = q;
      cpos[out[q].cols[t]] = (i64)t;
    }
  }
  for (i64 q = 0; q < nq; ++q)
    if (!out[q].rows.empty()) out[q].parent = newid[find(sn_of[out[q].rows[0]])];
  for (i64 q = 0; q < nq; ++q)
    if (out[q].parent >= 0) out[out[q].parent].level = std::max(out[out[q].parent].level, out[q].level + 1);
  if (!with_values) return out;  // structure only (the device computes the blocks)
  // panels [L_CC; L_RC] ((s + r) x s) and [U_CC, U_CR] (s x (s + r))
  std::vector<std::vector<double>> lpan(nq), upan(nq);
  for (i64 q = 0; q < nq; ++q) {
    const i64 s = (i64)out[q].cols.size(), r = (i64)out[q].rows.size();
    lpan[q].assign((size_t)(s + r) * s, 0.0);
    upan[q].assign((size_t)s * (s + r), 0.0);
  }
  auto rpos = [&](i64 q, i64 g) {
    const VI& R = out[q].rows;
    auto it = std::lower_bound(R.begin(), R.end(), g);
    require_host(it != R.end() && *it == g, "partitioned inverse: row outside its supernode");
    return (i64)(it - R.begin());
  };
  for (i64 i = 0; i < n; ++i)
    for (i64 p = lp[i]; p < lp[i + 1]; ++p) {
      const i64 j = li[p], q = sn_col[j], s = (i64)out[q].cols.size();
      const i64 row = sn_col[i] == q ? cpos[i] : s + rpos(q, i);
      lpan[q][row * s + cpos[j]] = lv[p];
    }
  for (i64 i = 0; i < n; ++i)
    for (i64 p = up[i]; p < up[i + 1]; ++p) {
      const i64 j = ui[p], q = sn_col[i], s = (i64)out[q].cols.size(), r = (i64)out[q].rows.size();
      const i64 c = sn_col[j] == q ? cpos[j] : s + rpos(q, j);
      upan[q][cpos[i] * (s + r) + c] = uv[p];
    }
  std::vector<double> lkk, ukk, linv, uinv;
  for (i64 q = 0; q < nq; ++q) {
    const i64 s = (i64)out[q].cols.size(), r = (i64)out[q].rows.size();
    lkk.assign((size_t)s * s, 0.0);
    ukk.assign((size_t)s * s, 0.0);
    for (i64 i = 0; i < s; ++i)
      for (i64 j = 0; j < s; ++j) {
        lkk[i * s + j] = lpan[q][i * s + j];
        ukk[i * s + j] = upan[q][i * (s + r) + j];
      }
    for (i64 i = 0; i < s; ++i)
      require_host(ukk[i * s + i] != 0.0 && std::isfinite(ukk[i * s + i]), "matrix is singular");
    tri_inv_unit_lower(s, lkk, linv);
    tri_inv_upper(s, ukk, uinv);
    PinvSn& o = out[q];
    o.d.assign((size_t)s * s, 0.0);
    for (i64 i = 0; i < s; ++i)
      for (i64 j = 0; j < s; ++j) o.d[i * s + j] = j < i ? linv[i * s + j] : uinv[i * s + j];
    // M = L_RC linv (r x s): row i of L_RC times linv (lower), k >= j
    o.m.assign((size_t)r * s, 0.0);
    for (i64 i = 0; i < r; ++i) {
      const double* lr = &lpan[q][(s + i) * s];
      double* mr = &o.m[i * s];
      for (i64 k = 0; k < s; ++k) {
        const double a = lr[k];
        if (a == 0.0) continue;
        const double* lk = &linv[k * s];
        for (i64 j = 0; j <= k; ++j) mr[j] += a * lk[j];
      }
    }
    // N = uinv U_CR (s x r)
    o.nm.assign((size_t)s * r, 0.0);
    for (i64 i = 0; i < s; ++i) {
      double* nr = &o.nm[i * r];
      for (i64 k = i; k < s; ++k) {
        const double a = uinv[i * s + k];
        if (a == 0.0) continue;
        const double* ur = &upan[q][k * (s + r) + s];
        for (i64 j = 0; j < r; ++j) nr[j] += a * ur[j];
      }
    }
    std::vector<double>().swap(lpan[q]);
    std::vector<double>().swap(upan[q]);
  }
  return out;
}

}  // namespace

extern "C" int gh_partitioned_inverse(int64_t nblk, const int64_t* blk_n, const int64_t* blk_base,
                                      const int64_t* lp_off, const int64_t* lnz_off, const int64_t* up_off,
                                      const int64_t* unz_off, const int64_t* lp, const int64_t* li,
                                      const double* lv, const int64_t* up, const int64_t* ui,
                                      const double* uv, int64_t relax, double zero_frac, int64_t threads,
                                      int with_values, gh_result** res) {
  GH_TRY({
    std::vector<std::vector<PinvSn>> per(nblk);
    std::vector<std::string> errs(nblk);
    std::atomic<i64> next{0};
    auto work = [&] {
      for (;;) {
        const i64 b = next.fetch_add(1);
        if (b >= nblk) break;
        try {
          per[b] = pinv_block(blk_n[b], lp + lp_off[b], li + lnz_off[b], with_values ? lv + lnz_off[b] : nullptr,
                              up + up_off[b], ui + unz_off[b], with_values ? uv + unz_off[b] : nullptr, relax,
                              zero_frac, with_values != 0);
        } catch (const std::exception& e) {
          errs[b] = e.what();
        }
      }
    };
    std::vector<std::thread> pool;
    for (i64 t = 1; t < std::max<i64>(1, threads); ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (i64 b = 0; b < nblk; ++b)
      if (!errs[b].empty()) throw std::runtime_error("block " + std::to_string(b) + ": " + errs[b]);
    // global records in (block, local) order; processing order by (level, that)
    struct Ref { i64 b, q, g, level; };
    std::vector<Ref> refs;
    VI first(nblk + 1, 0);
    for (i64 b = 0; b < nblk; ++b) {
      first[b + 1] = first[b] + (i64)per[b].size();
      for (i64 q = 0; q < (i64)per[b].size(); ++q) refs.push_back({b, q, first[b] + q, per[b][q].level});
    }
    const i64 nsn = (i64)refs.size();
    std::vector<Ref> ord(refs);
    std::stable_sort(ord.begin(), ord.end(), [](const Ref& x, const Ref& y) { return x.level < y.level; });
    VI pos(nsn);
    for (i64 t = 0; t < nsn; ++t) pos[ord[t].g] = t;
    i64 nlev = 0;
    for (const Ref& r : ord) nlev = std::max(nlev, r.level + 1);
    VI level_ptr(nlev + 1, 0), sn_s(nsn), sn_r(nsn), col_ptr(nsn + 1, 0), row_ptr(nsn + 1, 0);
    for (const Ref& r : ord) level_ptr[r.level + 1]++;
    for (i64 l = 0; l < nlev; ++l) level_ptr[l + 1] += level_ptr[l];
    for (i64 t = 0; t < nsn; ++t) {
      const PinvSn& o = per[ord[t].b][ord[t].q];
      sn_s[t] = (i64)o.cols.size();
      sn_r[t] = (i64)o.rows.size();
      col_ptr[t + 1] = col_ptr[t] + sn_s[t];
      row_ptr[t + 1] = row_ptr[t] + sn_r[t];
    }
    VI col_ids(col_ptr[nsn]), row_ids(row_ptr[nsn]), d_off(nsn), m_off(nsn), n_off(nsn);
    i64 nval = 0;
    for (i64 t = 0; t < nsn; ++t) {
      const PinvSn& o = per[ord[t].b][ord[t].q];
      const i64 base = blk_base[ord[t].b];
      for (i64 c = 0; c < sn_s[t]; ++c) col_ids[col_ptr[t] + c] = base + o.cols[c];
      for (i64 c = 0; c < sn_r[t]; ++c) row_ids[row_ptr[t] + c] = base + o.rows[c];
      const i64 s_ = sn_s[t], r_ = sn_r[t];
      d_off[t] = nval;
      nval += s_ * s_;
      m_off[t] = nval;
      nval += r_ * s_;
      n_off[t] = nval;
      nval += s_ * r_;
    }
    std::vector<double> vals(with_values ? (size_t)nval : (size_t)0);
    for (i64 t = 0; t < nsn && with_values; ++t) {
      const PinvSn& o = per[ord[t].b][ord[t].q];
      std::copy(o.d.begin(), o.d.end(), vals.begin() + d_off[t]);
      std::copy(o.m.begin(), o.m.end(), vals.begin() + m_off[t]);
      std::copy(o.nm.begin(), o.nm.end(), vals.begin() + n_off[t]);
    }
    // extend-add lists: children (processing order) of each supernode
    std::vector<VI> children(nsn);
    for (i64 t = 0; t < nsn; ++t) {
      const PinvSn& o = per[ord[t].b][ord[t].q];
      if (o.parent >= 0) children[pos[first[ord[t].b] + o.parent]].push_back(t);
    }
    std::vector<VI> in_l(col_ptr[nsn]), out_l(row_ptr[nsn]);
    for (i64 t = 0; t < nsn; ++t) {
      const PinvSn& o = per[ord[t].b][ord[t].q];
      for (i64 c : children[t]) {
        const PinvSn& oc = per[ord[c].b][ord[c].q];
        for (i64 m = 0; m < (i64)oc.rows.size(); ++m) {
          const i64 g = oc.rows[m], slot = row_ptr[c] + m;
          auto it = std::lower_bound(o.cols.begin(), o.cols.end(), g);
          if (it != o.cols.end() && *it == g) {
            in_l[col_ptr[t] + (it - o.cols.begin())].push_back(slot);
          } else {
            auto jt = std::lower_bound(o.rows.begin(), o.rows.end(), g);
            require_host(jt != o.rows.end() && *jt == g, "supernode tree violates R_c within C_p + R_p");
            out_l[row_ptr[t] + (jt - o.rows.begin())].push_back(slot);
          }
        }
      }
    }
    auto flat = [](const std::vector<VI>& lists, VI& ptr, VI& idx) {
      ptr.assign(lists.size() + 1, 0);
      for (size_t i = 0; i < lists.size(); ++i) ptr[i + 1] = ptr[i] + (i64)lists[i].size();
      idx.clear();
      idx.reserve(ptr.back());
      for (const VI& l : lists) idx.insert(idx.end(), l.begin(), l.end());
    };
    VI in_ptr, in_idx, out_ptr, out_idx;
    flat(in_l, in_ptr, in_idx);
    flat(out_l, out_ptr, out_idx);
    auto* r = new gh_result;
    r->add(std::move(level_ptr));
    r->add(std::move(sn_s));
    r->add(std::move(sn_r));
    r->add(std::move(col_ptr));
    r->add(std::move(col_ids));
    r->add(std::move(row_ptr));
    r->add(std::move(row_ids));
    r->add(std::move(d_off));
    r->add(std::move(m_off));
    r->add(std::move(n_off));
    r->add(std::move(vals));
    r->add(std::move(in_ptr));
    r->add(std::move(in_idx));
    r->add(std::move(out_ptr));
    r->add(std::move(out_idx));
    *res = r;
  })
}
