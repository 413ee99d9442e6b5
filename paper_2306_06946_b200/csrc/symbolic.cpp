// Host symbolic analysis for the supernodal multifrontal Cholesky.
//
// Replaces the ordering + symbolic part of the reference's SuperLU call
// (linalg.py:71-76, permc_spec="MMD_AT_PLUS_A").  The sparsity pattern of a
// soft body's system matrix is fixed per mesh, so this runs once per body;
// only the numeric factorisation and the solves run on the GPU each step.
//
//   1. node graph (bs DoFs per FE node share one pattern);
//   2. nested dissection: geometric median bisection when node coordinates
//      are known (FE meshes), BFS level-structure bisection otherwise;
//      one-sided vertex separators, separators numbered last;
//   3. elimination tree (Liu, path compression) and postorder;
//   4. column structures, fundamental supernodes, relaxed amalgamation;
//   5. dense fronts, extend-add relative maps, CSR -> front value map and
//      the per-level task lists the GPU kernels walk.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <stdexcept>

#include "chol.h"

namespace cnb {

namespace {

struct Graph {
  int64_t nv = 0;
  std::vector<int64_t> ptr, adj;
};

Graph node_graph(int64_t n, const int64_t* rowptr, const int64_t* col, int bs) {
  Graph G;
  G.nv = n / bs;
  std::vector<std::vector<int64_t>> nb(G.nv);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = i / bs;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int64_t b = col[k] / bs;
      if (a != b) {
        nb[a].push_back(b);
        nb[b].push_back(a);
      }
    }
  }
  G.ptr.assign(G.nv + 1, 0);
  for (int64_t a = 0; a < G.nv; ++a) {
    auto& v = nb[a];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    G.ptr[a + 1] = G.ptr[a] + (int64_t)v.size();
  }
  G.adj.resize(G.ptr[G.nv]);
  for (int64_t a = 0; a < G.nv; ++a) std::copy(nb[a].begin(), nb[a].end(), G.adj.begin() + G.ptr[a]);
  return G;
}

struct Dissector {
  const Graph& G;
  const double* xyz;
  int leaf;
  std::vector<int64_t> order;
  std::vector<int64_t> label;  // scratch set labels
  int64_t next_label = 1;

  Dissector(const Graph& g, const double* c, int lf) : G(g), xyz(c), leaf(lf), label(g.nv, 0) {}

  void emit(std::vector<int64_t>& S) {
    std::sort(S.begin(), S.end());
    order.insert(order.end(), S.begin(), S.end());
  }

  // BFS over S (nodes labelled lab) from src; returns levels as lists.
  std::vector<std::vector<int64_t>> bfs(int64_t src, int64_t lab, std::vector<int64_t>& seen_stamp,
                                        int64_t stamp) {
    std::vector<std::vector<int64_t>> levels;
    std::vector<int64_t> cur{src};
    seen_stamp[src] = stamp;
    while (!cur.empty()) {
      levels.push_back(cur);
      std::vector<int64_t> nxt;
      for (int64_t v : cur)
        for (int64_t k = G.ptr[v]; k < G.ptr[v + 1]; ++k) {
          int64_t u = G.adj[k];
          if (label[u] == lab && seen_stamp[u] != stamp) {
            seen_stamp[u] = stamp;
            nxt.push_back(u);
          }
        }
      cur.swap(nxt);
    }
    return levels;
  }

  std::vector<int64_t> stamp_;
  int64_t stamp_ctr = 0;

  void run(std::vector<int64_t> S) {
    if ((int64_t)S.size() <= leaf) {
      emit(S);
      return;
    }
    const int64_t lab = next_label++;
    for (int64_t v : S) label[v] = lab;
    std::vector<int64_t> A, B, sep;
    if (xyz) {
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      for (int64_t v : S)
        for (int d = 0; d < 3; ++d) {
          lo[d] = std::min(lo[d], xyz[3 * v + d]);
          hi[d] = std::max(hi[d], xyz[3 * v + d]);
        }
      int ax = 0;
      for (int d = 1; d < 3; ++d)
        if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
      std::vector<int64_t> srt(S);
      std::sort(srt.begin(), srt.end(), [&](int64_t a, int64_t b) {
        double xa = xyz[3 * a + ax], xb = xyz[3 * b + ax];
        return xa < xb || (xa == xb && a < b);
      });
      // split at the median coordinate value (whole layers stay together)
      size_t mid = srt.size() / 2;
      const double med = xyz[3 * srt[mid] + ax];
      size_t cut = mid;
      while (cut > 0 && xyz[3 * srt[cut - 1] + ax] == med) --cut;
      if (cut == 0) {
        cut = mid;
        while (cut < srt.size() && xyz[3 * srt[cut] + ax] == med) ++cut;
        if (cut == srt.size()) cut = mid;
      }
      A.assign(srt.begin(), srt.begin() + cut);
      B.assign(srt.begin() + cut, srt.end());
    } else {
      if (stamp_.empty()) stamp_.assign(G.nv, 0);
      // pseudo-peripheral start, then level structure
      int64_t src = *std::min_element(S.begin(), S.end());
      std::vector<std::vector<int64_t>> lv;
      for (int rep = 0; rep < 3; ++rep) {
        lv = bfs(src, lab, stamp_, ++stamp_ctr);
        int64_t nsrc = lv.back()[0];
        for (int64_t v : lv.back()) nsrc = std::min(nsrc, v);
        if (rep > 0 && nsrc == src) break;
        src = nsrc;
      }
      int64_t reached = 0;
      for (auto& l : lv) reached += (int64_t)l.size();
      if (reached < (int64_t)S.size()) {
        // disconnected: order the reached component and the rest separately
        std::vector<int64_t> comp, rest;
        for (auto& l : lv) comp.insert(comp.end(), l.begin(), l.end());
        const int64_t st = stamp_ctr;
        for (int64_t v : S)
          if (stamp_[v] != st) rest.push_back(v);
        for (int64_t v : S) label[v] = 0;
        run(comp);
        run(rest);
        return;
      }
      if (lv.size() < 3) {
        emit(S);
        return;
      }
      int64_t half = (int64_t)S.size() / 2, acc = 0;
      size_t L = 1;
      for (size_t k = 0; k < lv.size(); ++k) {
        acc += (int64_t)lv[k].size();
        if (acc >= half) {
          L = std::max<size_t>(1, std::min(k, lv.size() - 2));
          break;
        }
      }
      for (size_t k = 0; k < lv.size(); ++k) {
        auto& dst = k < L ? A : (k == L ? sep : B);
        dst.insert(dst.end(), lv[k].begin(), lv[k].end());
      }
      for (int64_t v : S) label[v] = 0;
      run(A);
      run(B);
      emit(sep);
      return;
    }
    // one-sided separator: the smaller boundary layer
    const int64_t la = next_label++, lb = next_label++;
    for (int64_t v : A) label[v] = la;
    for (int64_t v : B) label[v] = lb;
    std::vector<int64_t> sa, sb;
    for (int64_t v : A)
      for (int64_t k = G.ptr[v]; k < G.ptr[v + 1]; ++k)
        if (label[G.adj[k]] == lb) {
          sa.push_back(v);
          break;
        }
    for (int64_t v : B)
      for (int64_t k = G.ptr[v]; k < G.ptr[v + 1]; ++k)
        if (label[G.adj[k]] == la) {
          sb.push_back(v);
          break;
        }
    const bool use_a = sa.size() <= sb.size();
    sep = use_a ? sa : sb;
    for (int64_t v : sep) label[v] = -1;
    std::vector<int64_t> A2, B2;
    for (int64_t v : A)
      if (label[v] != -1) A2.push_back(v);
    for (int64_t v : B)
      if (label[v] != -1) B2.push_back(v);
    for (int64_t v : S) label[v] = 0;
    if (A2.empty() || B2.empty()) {
      // no progress possible (degenerate geometry): fall back to leaf order
      emit(S);
      return;
    }
    run(std::move(A2));
    run(std::move(B2));
    emit(sep);
  }
};

}  // namespace

int analyze(Symbolic& S, int64_t n, const int64_t* rowptr, const int64_t* col, int bs, const double* coords,
            int leaf_nodes) {
  if (bs < 1 || n % bs != 0) throw std::runtime_error("analyze: n must be a multiple of the block size");
  S = Symbolic();
  S.n = n;
  S.bs = bs;
  Graph G = node_graph(n, rowptr, col, bs);
  const int64_t nv = G.nv;

  // ---- ordering ----
  Dissector nd(G, coords, std::max(1, leaf_nodes));
  {
    std::vector<int64_t> all(nv);
    std::iota(all.begin(), all.end(), 0);
    nd.order.reserve(nv);
    nd.run(std::move(all));
  }
  std::vector<int64_t> ord = nd.order;  // new -> old node
  if ((int64_t)ord.size() != nv) throw std::runtime_error("analyze: ordering lost nodes");
  std::vector<int64_t> inv(nv);
  for (int64_t k = 0; k < nv; ++k) inv[ord[k]] = k;

  // ---- elimination tree on the permuted graph ----
  std::vector<int64_t> par(nv, -1), anc(nv, -1);
  for (int64_t i = 0; i < nv; ++i) {
    const int64_t v = ord[i];
    for (int64_t k = G.ptr[v]; k < G.ptr[v + 1]; ++k) {
      int64_t r = inv[G.adj[k]];
      if (r >= i) continue;
      while (anc[r] != -1 && anc[r] != i) {
        int64_t nx = anc[r];
        anc[r] = i;
        r = nx;
      }
      if (anc[r] == -1) {
        anc[r] = i;
        par[r] = i;
      }
    }
  }
  // ---- postorder ----
  std::vector<int64_t> head(nv, -1), nxt(nv, -1);
  for (int64_t i = nv - 1; i >= 0; --i)
    if (par[i] >= 0) {
      nxt[i] = head[par[i]];
      head[par[i]] = i;
    }
  std::vector<int64_t> post;
  post.reserve(nv);
  {
    std::vector<int64_t> stack;
    for (int64_t r = 0; r < nv; ++r) {
      if (par[r] != -1) continue;
      stack.push_back(r);
      while (!stack.empty()) {
        int64_t v = stack.back();
        if (head[v] != -1) {
          int64_t c = head[v];
          head[v] = nxt[c];
          stack.push_back(c);
        } else {
          stack.pop_back();
          post.push_back(v);
        }
      }
    }
  }
  std::vector<int64_t> pinv(nv);
  for (int64_t k = 0; k < nv; ++k) pinv[post[k]] = k;
  std::vector<int64_t> order(nv), parent(nv);  // postordered numbering
  for (int64_t k = 0; k < nv; ++k) {
    order[k] = ord[post[k]];
    parent[k] = par[post[k]] >= 0 ? pinv[par[post[k]]] : -1;
  }
  for (int64_t k = 0; k < nv; ++k) inv[order[k]] = k;

  // ---- column structures (node level) ----
  std::vector<std::vector<int64_t>> st(nv);
  std::vector<std::vector<int64_t>> kids(nv);
  for (int64_t k = 0; k < nv; ++k)
    if (parent[k] >= 0) kids[parent[k]].push_back(k);
  {
    std::vector<int64_t> mark(nv, -1);
    for (int64_t i = 0; i < nv; ++i) {
      auto& s = st[i];
      const int64_t v = order[i];
      for (int64_t k = G.ptr[v]; k < G.ptr[v + 1]; ++k) {
        int64_t j = inv[G.adj[k]];
        if (j > i && mark[j] != i) {
          mark[j] = i;
          s.push_back(j);
        }
      }
      for (int64_t c : kids[i]) {
        for (int64_t j : st[c])
          if (j > i && mark[j] != i) {
            mark[j] = i;
            s.push_back(j);
          }
      }
      std::sort(s.begin(), s.end());
      if (!s.empty() && s[0] != parent[i]) throw std::runtime_error("analyze: etree/structure mismatch");
    }
  }
  // ---- fundamental supernodes ----
  std::vector<int64_t> sfirst;  // node ranges
  for (int64_t i = 0; i < nv; ++i) {
    bool join = i > 0 && parent[i - 1] == i && kids[i].size() == 1 && st[i - 1].size() == st[i].size() + 1;
    if (!join) sfirst.push_back(i);
  }
  sfirst.push_back(nv);
  // supernode of node, parents
  int64_t ns0 = (int64_t)sfirst.size() - 1;
  std::vector<int64_t> sn_of(nv);
  for (int64_t s = 0; s < ns0; ++s)
    for (int64_t i = sfirst[s]; i < sfirst[s + 1]; ++i) sn_of[i] = s;
  // ---- relaxed amalgamation (bottom-up in postorder) ----
  // merge child c into parent p when c ends right before p (p's last child)
  // and the structural zeros it adds stay small.
  std::vector<int64_t> sfirst_m(ns0), slast_m(ns0), sparent(ns0, -1), rsize(ns0);
  std::vector<char> alive(ns0, 1);
  for (int64_t s = 0; s < ns0; ++s) {
    sfirst_m[s] = sfirst[s];
    slast_m[s] = sfirst[s + 1] - 1;
    rsize[s] = (int64_t)st[slast_m[s]].size();
    sparent[s] = parent[slast_m[s]] >= 0 ? sn_of[parent[slast_m[s]]] : -1;
  }
  std::vector<int64_t> owner(ns0);
  std::iota(owner.begin(), owner.end(), 0);
  auto find = [&](int64_t s) {
    while (owner[s] != s) {
      owner[s] = owner[owner[s]];
      s = owner[s];
    }
    return s;
  };
  for (int64_t p = 0; p < ns0; ++p) {
    while (true) {
      if (sfirst_m[p] == 0) break;
      int64_t c = find(sn_of[sfirst_m[p] - 1]);
      if (c == p || !alive[c]) break;
      if (find(sparent[c] >= 0 ? sparent[c] : c) != p) break;
      const double ncc = (double)(slast_m[c] - sfirst_m[c] + 1), ncp = (double)(slast_m[p] - sfirst_m[p] + 1);
      const double rc = (double)rsize[c], rp = (double)rsize[p];
      const double orig = ncc * (ncc + 1) / 2 + ncc * rc + ncp * (ncp + 1) / 2 + ncp * rp;
      const double ncm = ncc + ncp;
      const double merged = ncm * (ncm + 1) / 2 + ncm * rp;
      const double zfrac = (merged - orig) / merged;
      const bool ok = (ncm <= 4) || (ncm <= 16 && zfrac <= 0.5) || (ncm <= 48 && zfrac <= 0.2) || zfrac <= 0.05;
      if (!ok) break;
      sfirst_m[p] = sfirst_m[c];
      alive[c] = 0;
      owner[c] = p;
    }
  }
  // final supernodes in ascending node order; supernodes wider than
  // kMaxSnCols DoFs are split into a chain of pieces (piece k's parent is
  // piece k+1, its rows the later columns of the supernode plus the
  // supernode's own rows).  The factor is unchanged; the inverted diagonal
  // blocks L11^{-1} of the solves stay at most kMaxSnCols wide (a 6750-wide
  // separator would otherwise cost nc^3/3 flops to invert).
  std::vector<int64_t> pf, pl, pend;  // piece first / last node, last node of the supernode
  const int64_t maxw = std::max<int64_t>(1, kMaxSnCols / bs);
  for (int64_t s = 0; s < ns0; ++s) {
    if (!alive[s]) continue;
    const int64_t a = sfirst_m[s], z = slast_m[s], w = z - a + 1;
    const int64_t np = (w + maxw - 1) / maxw;
    for (int64_t k = 0; k < np; ++k) {
      pf.push_back(a + (w * k) / np);  // near-equal pieces
      pl.push_back(a + (w * (k + 1)) / np - 1);
      pend.push_back(z);
    }
  }
  const int64_t ns = (int64_t)pf.size();
  S.ns = ns;
  S.first.assign(ns + 1, 0);
  S.parent.assign(ns, -1);
  S.rows_ptr.assign(ns + 1, 0);
  std::vector<int64_t> node_sn(nv);
  for (int64_t k = 0; k < ns; ++k) {
    S.first[k] = bs * pf[k];
    for (int64_t i = pf[k]; i <= pl[k]; ++i) node_sn[i] = k;
  }
  S.first[ns] = bs * nv;
  for (int64_t k = 0; k < ns; ++k) {
    const int64_t last = pend[k];
    if (pl[k] < last) {
      S.parent[k] = k + 1;
    } else {
      S.parent[k] = parent[last] >= 0 ? node_sn[parent[last]] : -1;
    }
    S.rows_ptr[k + 1] = S.rows_ptr[k] + bs * ((last - pl[k]) + (int64_t)st[last].size());
  }
  S.rows.resize(S.rows_ptr[ns]);
  for (int64_t k = 0; k < ns; ++k) {
    int64_t o = S.rows_ptr[k];
    for (int64_t j = pl[k] + 1; j <= pend[k]; ++j)
      for (int d = 0; d < bs; ++d) S.rows[o++] = bs * j + d;
    for (int64_t j : st[pend[k]])
      for (int d = 0; d < bs; ++d) S.rows[o++] = bs * j + d;
  }
  // DoF permutation
  S.perm.resize(n);
  S.iperm.resize(n);
  for (int64_t k = 0; k < nv; ++k)
    for (int d = 0; d < bs; ++d) {
      S.perm[bs * k + d] = bs * order[k] + d;
      S.iperm[bs * order[k] + d] = bs * k + d;
    }
  // children, levels
  S.child_ptr.assign(ns + 1, 0);
  for (int64_t k = 0; k < ns; ++k)
    if (S.parent[k] >= 0) S.child_ptr[S.parent[k] + 1]++;
  for (int64_t k = 0; k < ns; ++k) S.child_ptr[k + 1] += S.child_ptr[k];
  S.child.resize(S.child_ptr[ns]);
  {
    std::vector<int64_t> fill(S.child_ptr.begin(), S.child_ptr.end() - 1);
    for (int64_t k = 0; k < ns; ++k)
      if (S.parent[k] >= 0) S.child[fill[S.parent[k]]++] = k;
  }
  S.level.assign(ns, 0);
  for (int64_t k = 0; k < ns; ++k)
    for (int64_t c = S.child_ptr[k]; c < S.child_ptr[k + 1]; ++c)
      S.level[k] = std::max(S.level[k], S.level[S.child[c]] + 1);
  S.n_levels = 0;
  for (int64_t k = 0; k < ns; ++k) S.n_levels = std::max(S.n_levels, S.level[k] + 1);
  S.level_ptr.assign(S.n_levels + 1, 0);
  for (int64_t k = 0; k < ns; ++k) S.level_ptr[S.level[k] + 1]++;
  for (int l = 0; l < S.n_levels; ++l) S.level_ptr[l + 1] += S.level_ptr[l];
  S.level_sn.resize(ns);
  {
    std::vector<int64_t> fill(S.level_ptr.begin(), S.level_ptr.end() - 1);
    for (int64_t k = 0; k < ns; ++k) S.level_sn[fill[S.level[k]]++] = k;
  }
  // fronts
  S.front_off.assign(ns + 1, 0);
  S.nnz_L = 0;
  S.flops = 0.0;
  S.solve_flops_per_rhs = 0.0;
  for (int64_t k = 0; k < ns; ++k) {
    const int64_t f = S.f(k), nc = S.nc(k);
    S.front_off[k + 1] = S.front_off[k] + S.ldf(k) * f;
    S.nnz_L += nc * (nc + 1) / 2 + nc * S.nr(k);
    for (int64_t j = 0; j < nc; ++j) {
      const double m = (double)(f - j - 1);
      S.flops += m + m * (m + 1);
    }
    S.solve_flops_per_rhs += 4.0 * (double)(nc * (nc + 1) / 2 + nc * S.nr(k));
  }
  // relative maps child rows -> parent front positions
  S.rel_ptr.assign(ns + 1, 0);
  for (int64_t k = 0; k < ns; ++k) S.rel_ptr[k + 1] = S.rel_ptr[k] + (S.parent[k] >= 0 ? S.nr(k) : 0);
  S.rel.resize(S.rel_ptr[ns]);
  for (int64_t k = 0; k < ns; ++k) {
    const int64_t p = S.parent[k];
    if (p < 0) continue;
    const int64_t* pr = S.rows.data() + S.rows_ptr[p];
    const int64_t pnr = S.nr(p), pnc = S.nc(p);
    for (int64_t i = 0; i < S.nr(k); ++i) {
      const int64_t r = S.rows[S.rows_ptr[k] + i];
      int64_t pos;
      if (r >= S.first[p] && r < S.first[p + 1]) {
        pos = r - S.first[p];
      } else {
        const int64_t* it = std::lower_bound(pr, pr + pnr, r);
        if (it == pr + pnr || *it != r) throw std::runtime_error("analyze: child row missing in parent");
        pos = pnc + (it - pr);
      }
      S.rel[S.rel_ptr[k] + i] = (int32_t)pos;
    }
  }
  // CSR value map
  std::vector<int64_t> dof_sn(n);
  for (int64_t k = 0; k < ns; ++k)
    for (int64_t d = S.first[k]; d < S.first[k + 1]; ++d) dof_sn[d] = k;
  S.csr_nnz = rowptr[n];
  S.map_src.clear();
  S.map_dst.clear();
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int64_t pi = S.iperm[i], pj = S.iperm[col[e]];
      if (pi < pj) continue;
      const int64_t s = dof_sn[pj];
      const int64_t c = pj - S.first[s], f = S.f(s);
      int64_t r;
      if (pi < S.first[s + 1]) {
        r = pi - S.first[s];
      } else {
        const int64_t* rs = S.rows.data() + S.rows_ptr[s];
        const int64_t* it = std::lower_bound(rs, rs + S.nr(s), pi);
        if (it == rs + S.nr(s) || *it != pi) throw std::runtime_error("analyze: A entry outside L structure");
        r = S.nc(s) + (it - rs);
      }
      S.map_src.push_back(e);
      S.map_dst.push_back(S.front_off[s] + c * S.ldf(s) + r);
    }
  // per-level task lists
  S.tasks.assign(S.n_levels, LevelTasks());
  S.ea_rng.clear();
  for (int l = 0; l < S.n_levels; ++l) {
    LevelTasks& T = S.tasks[l];
    int64_t max_panels = 0;
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      if (S.child_ptr[s + 1] > S.child_ptr[s])
        for (int64_t lo = 0; lo < S.f(s); lo += kEaCols) {
          const int64_t hi = std::min<int64_t>(S.f(s), lo + kEaCols);
          T.ea.push_back((int32_t)s);
          T.ea.push_back((int32_t)lo);
          T.ea.push_back((int32_t)hi);
          T.ea.push_back((int32_t)(S.ea_rng.size() / 2));
          for (int64_t ci = S.child_ptr[s]; ci < S.child_ptr[s + 1]; ++ci) {  // rel is ascending per child
            const int64_t c = S.child[ci];
            const int32_t* r0 = S.rel.data() + S.rel_ptr[c];
            const int32_t* r1 = S.rel.data() + S.rel_ptr[c + 1];
            S.ea_rng.push_back((int32_t)(std::lower_bound(r0, r1, (int32_t)lo) - r0));
            S.ea_rng.push_back((int32_t)(std::lower_bound(r0, r1, (int32_t)hi) - r0));
          }
        }
      max_panels = std::max(max_panels, (S.nc(s) + kPanel - 1) / kPanel);
    }
    T.potrf.assign(max_panels, {});
    T.trsm.assign(max_panels, {});
    T.syrk.assign(max_panels, {});
    T.syrk_out.assign(max_panels, {});
    const int64_t blk = (int64_t)kBlkPanels * kPanel;
    for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
      const int64_t s = S.level_sn[q];
      const int64_t nc = S.nc(s), f = S.f(s);
      for (int64_t p = 0; p * kPanel < nc; ++p) {
        const int64_t k0 = p * kPanel, kw = std::min<int64_t>(kPanel, nc - k0);
        const int64_t below = f - k0 - kw;
        T.potrf[p].push_back((int32_t)s);
        for (int64_t c = 0; c * kTile < below; ++c) {
          T.trsm[p].push_back((int32_t)s);
          T.trsm[p].push_back((int32_t)c);
        }
        // in-block update: columns [k0 + kw, block end) of every row below
        const int64_t bend = std::min<int64_t>((k0 / blk + 1) * blk, nc);
        const int64_t t0 = k0 + kw;
        if (t0 < bend) {
          const int64_t ntr = (f - t0 + kTile - 1) / kTile, ntc = (bend - t0 + kTile - 1) / kTile;
          for (int64_t ti = 0; ti < ntr; ++ti)
            for (int64_t tj = 0; tj <= std::min(ti, ntc - 1); ++tj) {
              T.syrk[p].push_back((int32_t)s);
              T.syrk[p].push_back((int32_t)ti);
              T.syrk[p].push_back((int32_t)tj);
            }
        } else if (bend < f) {
          // last panel of a block: trailing update [bend, f) by the block's columns
          const int64_t nt = (f - bend + kTile - 1) / kTile;
          for (int64_t ti = 0; ti < nt; ++ti)
            for (int64_t tj = 0; tj <= ti; ++tj) {
              T.syrk_out[p].push_back((int32_t)s);
              T.syrk_out[p].push_back((int32_t)ti);
              T.syrk_out[p].push_back((int32_t)tj);
            }
        }
      }
    }
  }
  return 0;
}

}  // namespace cnb
