// Host symbolic analysis for the multifrontal LDL^T of SGN KKT matrices.
//
// Replaces the ordering half of the reference factorization: SuperLU's COLAMD column
// ordering inside spla.splu (pkg/src/sgnopt/linear_solvers.py:87) together with the
// structural-singularity checks of SparseFactorization.__init__ (linear_solvers.py:73-85).
// Runs once per sparsity pattern; deterministic (no hashing of pointers, no threads).
//
// KKT mode (n_x > 0): unknown u_x[i] is paired with the multiplier u_l[pi(i)] matched on
// the pattern of dc/dx (diagonal preferred), giving a 2x2 pivot block
// [[a+eps, g], [g, -eps]] whose determinant is bounded away from zero for the
// quasi-definite stabilized matrix.  Pair nodes are ordered by nested dissection of the
// (compressed) node graph; every parameter unknown is eliminated last in a single dense
// root front, whose Schur complement is the (SPD) reduced Gauss-Newton Hessian.
// Generic mode (n_x == 0): 1x1 pivots on every unknown, same nested dissection.
#include "sgn_internal.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>

namespace sgn {

std::string& last_error() {
  static thread_local std::string e;
  return e;
}

static std::atomic<int64_t> g_launches{0};
void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

namespace {

struct Csr {
  int32_t n = 0;
  std::vector<int64_t> ptr;
  std::vector<int32_t> adj;
};

// --------------------------------------------------------------------------------
// bipartite matching x_i -> lambda_j on the dc/dx pattern (K rows >= n_x+n_p of column i)
// --------------------------------------------------------------------------------
bool match_pairs(const Symbolic& s, std::vector<int64_t>& pi, int64_t* bad) {
  const int64_t nx = s.n_x, off = s.n_x + s.n_p;
  pi.assign(nx, -1);
  std::vector<int64_t> owner(nx, -1);   // lambda j -> x i
  for (int64_t i = 0; i < nx; ++i) {    // diagonal first
    for (int64_t k = s.indptr[i]; k < s.indptr[i + 1]; ++k) {
      if (s.indices[k] == off + i) { pi[i] = i; owner[i] = i; break; }
    }
  }
  struct Frame { int64_t i, k; };
  std::vector<int64_t> visit(nx, -1), via;
  std::vector<Frame> st;
  for (int64_t root = 0; root < nx; ++root) {
    if (pi[root] >= 0) continue;
    st.clear();
    st.push_back({root, s.indptr[root]});
    visit[root] = root;
    bool found = false;
    while (!st.empty() && !found) {
      const size_t depth = st.size() - 1;
      Frame& fr = st.back();
      bool advanced = false;
      for (; fr.k < s.indptr[fr.i + 1]; ++fr.k) {
        const int64_t r = s.indices[fr.k];
        if (r < off) continue;
        const int64_t j = r - off;
        if (via.size() <= depth) via.resize(depth + 1);
        if (owner[j] < 0) {
          via[depth] = j;
          for (size_t d = 0; d <= depth; ++d) { pi[st[d].i] = via[d]; owner[via[d]] = st[d].i; }
          found = true;
          break;
        }
        const int64_t i2 = owner[j];
        if (visit[i2] == root) continue;
        visit[i2] = root;
        via[depth] = j;
        ++fr.k;
        st.push_back({i2, s.indptr[i2]});
        advanced = true;
        break;
      }
      if (!found && !advanced) st.pop_back();
    }
    if (!found) { *bad = root; return false; }
  }
  return true;
}

// --------------------------------------------------------------------------------
// multilevel vertex separators: heavy-edge-matching coarsening, greedy-grown initial
// separators at the coarsest graph, one-sided node-FM refinement while uncoarsening
// (the scheme of Karypis & Kumar's multilevel nested dissection).  Deterministic: fixed
// visit orders, ties broken by vertex id.
// --------------------------------------------------------------------------------
struct WGraph {
  int32_t n = 0;
  std::vector<int64_t> xadj;
  std::vector<int32_t> adj;
  std::vector<int32_t> ew;
  std::vector<int64_t> vw;
  int64_t total() const { int64_t t = 0; for (int64_t w : vw) t += w; return t; }
};

// one level of heavy-edge matching; false when the graph no longer shrinks
bool coarsen_once(const WGraph& g, WGraph& c, std::vector<int32_t>& cmap, int64_t maxvw) {
  const int32_t n = g.n;
  std::vector<int32_t> order(n), match(n, -1);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return (g.xadj[a + 1] - g.xadj[a]) < (g.xadj[b + 1] - g.xadj[b]);
  });
  cmap.assign(n, -1);
  int32_t nc = 0;
  for (int32_t v : order) {
    if (match[v] >= 0) continue;
    int32_t best = -1, bw = -1;
    for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
      const int32_t u = g.adj[k];
      if (match[u] >= 0 || u == v || g.vw[v] + g.vw[u] > maxvw) continue;
      if (g.ew[k] > bw || (g.ew[k] == bw && u < best)) { bw = g.ew[k]; best = u; }
    }
    if (best >= 0) { match[v] = best; match[best] = v; cmap[v] = cmap[best] = nc++; }
    else { match[v] = v; cmap[v] = nc++; }
  }
  if (nc > (int32_t)(0.92 * n)) return false;
  std::vector<int32_t> rep(nc, -1);
  for (int32_t v : order) if (rep[cmap[v]] < 0) rep[cmap[v]] = v;
  c.n = nc;
  c.vw.assign(nc, 0);
  c.xadj.assign(nc + 1, 0);
  c.adj.clear(); c.ew.clear();
  std::vector<int32_t> slot(nc, -1);
  for (int32_t cv = 0; cv < nc; ++cv) {
    const int32_t v = rep[cv], u = match[v];
    const size_t start = c.adj.size();
    for (int mi = 0; mi < (u == v ? 1 : 2); ++mi) {
      const int32_t m = mi == 0 ? v : u;
      c.vw[cv] += g.vw[m];
      for (int64_t k = g.xadj[m]; k < g.xadj[m + 1]; ++k) {
        const int32_t cu = cmap[g.adj[k]];
        if (cu == cv) continue;
        if (slot[cu] < 0) { slot[cu] = (int32_t)c.adj.size(); c.adj.push_back(cu); c.ew.push_back(g.ew[k]); }
        else c.ew[slot[cu]] += g.ew[k];
      }
    }
    for (size_t k = start; k < c.adj.size(); ++k) slot[c.adj[k]] = -1;
    c.xadj[cv + 1] = (int64_t)c.adj.size();
  }
  return true;
}

// where: 0 / 1 = sides, 2 = separator; pw = side / separator weights
void node_fm(const WGraph& g, std::vector<int8_t>& where, int64_t pw[3], double maxfrac, int npasses) {
  const int32_t n = g.n;
  std::vector<int64_t> gain(n, 0);
  std::vector<char> locked(n, 0);
  struct Move { int32_t v; int8_t from; };
  std::vector<Move> moves;
  int bad_passes = 0;
  for (int pass = 0; pass < npasses && bad_passes < 2; ++pass) {
    const int to = (pw[0] < pw[1]) ? 0 : (pw[1] < pw[0] ? 1 : (pass & 1));
    const int other = 1 - to;
    const int64_t total = pw[0] + pw[1] + pw[2];
    const int64_t maxside = (int64_t)(maxfrac * (double)total);
    std::priority_queue<std::pair<int64_t, int32_t>> pq;   // (gain, -v) -> max gain, then min id
    auto push = [&](int32_t v) { pq.push({gain[v], -v}); };
    std::fill(locked.begin(), locked.end(), 0);
    for (int32_t v = 0; v < n; ++v) {
      if (where[v] != 2) continue;
      int64_t wo = 0;
      for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) if (where[g.adj[k]] == other) wo += g.vw[g.adj[k]];
      gain[v] = g.vw[v] - wo;
      push(v);
    }
    moves.clear();
    const int64_t start_sep = pw[2];
    int64_t best_sep = pw[2], best_imb = std::llabs(pw[0] - pw[1]);
    size_t best_pos = 0;
    int nbad = 0;
    const int limit = std::max(25, std::min(300, n / 20));
    while (!pq.empty()) {
      const auto top = pq.top(); pq.pop();
      const int32_t v = -top.second;
      if (where[v] != 2 || locked[v] || top.first != gain[v]) continue;
      int64_t wo = 0;
      for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) if (where[g.adj[k]] == other) wo += g.vw[g.adj[k]];
      if (pw[to] + g.vw[v] > maxside) break;
      where[v] = (int8_t)to; locked[v] = 1;
      pw[2] -= g.vw[v]; pw[to] += g.vw[v];
      moves.push_back({v, 2});
      for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
        const int32_t u = g.adj[k];
        if (where[u] != other) continue;
        where[u] = 2; pw[other] -= g.vw[u]; pw[2] += g.vw[u];
        moves.push_back({u, (int8_t)other});
        int64_t wu = 0;
        for (int64_t q = g.xadj[u]; q < g.xadj[u + 1]; ++q) {
          const int32_t z = g.adj[q];
          if (where[z] == other) wu += g.vw[z];
          else if (where[z] == 2 && !locked[z] && z != u) { gain[z] += g.vw[u]; push(z); }
        }
        if (!locked[u]) { gain[u] = g.vw[u] - wu; push(u); }
      }
      const bool balanced = std::max(pw[0], pw[1]) <= maxside;
      const int64_t imb = std::llabs(pw[0] - pw[1]);
      if (balanced && (pw[2] < best_sep || (pw[2] == best_sep && imb < best_imb))) {
        best_sep = pw[2]; best_imb = imb; best_pos = moves.size(); nbad = 0;
      } else if (++nbad > limit) {
        break;
      }
    }
    for (size_t k = moves.size(); k > best_pos; --k) {
      const Move& m = moves[k - 1];
      pw[where[m.v]] -= g.vw[m.v];
      where[m.v] = m.from;
      pw[m.from] += g.vw[m.v];
    }
    bad_passes = (best_sep < start_sep) ? 0 : bad_passes + 1;
  }
}

// greedy-grown separators from several seeds, each refined; the lightest balanced one wins
void initial_separator(const WGraph& g, std::vector<int8_t>& where, int64_t pw[3], double maxfrac) {
  const int32_t n = g.n;
  const int64_t total = g.total();
  int64_t best_score = INT64_MAX;
  std::vector<int8_t> w(n);
  std::vector<int32_t> q;
  std::vector<char> seen(n);
  const int ntry = std::min<int32_t>(n, 8);
  for (int t = 0; t < ntry; ++t) {
    const int32_t seed = (int32_t)(((int64_t)t * n) / ntry);
    std::fill(w.begin(), w.end(), 1);
    std::fill(seen.begin(), seen.end(), 0);
    int64_t pa = 0;
    q.assign(1, seed); seen[seed] = 1;
    for (size_t h = 0; h < q.size() && 2 * pa < total; ++h) {
      const int32_t v = q[h];
      w[v] = 0; pa += g.vw[v];
      for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k) {
        const int32_t u = g.adj[k];
        if (!seen[u]) { seen[u] = 1; q.push_back(u); }
      }
    }
    int64_t p[3] = {0, 0, 0};
    for (int32_t v = 0; v < n; ++v) {
      if (w[v] == 1)
        for (int64_t k = g.xadj[v]; k < g.xadj[v + 1]; ++k)
          if (w[g.adj[k]] == 0) { w[v] = 2; break; }
    }
    for (int32_t v = 0; v < n; ++v) p[w[v]] += g.vw[v];
    if (p[0] == 0 || p[1] == 0) continue;
    node_fm(g, w, p, maxfrac, 10);
    const int64_t score = p[2] * 4 + std::llabs(p[0] - p[1]) / 8;
    if (p[0] > 0 && p[1] > 0 && score < best_score) {
      best_score = score; where = w; pw[0] = p[0]; pw[1] = p[1]; pw[2] = p[2];
    }
  }
}

// 3-way partition of g (0 / 1 sides, 2 separator); false if no balanced separator was found
bool multilevel_separator(const WGraph& g0, std::vector<int8_t>& where, double maxfrac) {
  std::vector<WGraph> levels;
  std::vector<std::vector<int32_t>> cmaps;
  const WGraph* cur = &g0;
  const int64_t total = g0.total();
  levels.reserve(40);
  while (cur->n > 120 && levels.size() < 40) {
    WGraph c;
    std::vector<int32_t> cm;
    if (!coarsen_once(*cur, c, cm, std::max<int64_t>(1, (int64_t)(1.5 * (double)total / 60.0)))) break;
    levels.push_back(std::move(c));
    cmaps.push_back(std::move(cm));
    cur = &levels.back();
  }
  int64_t pw[3] = {0, 0, 0};
  std::vector<int8_t> w;
  initial_separator(*cur, w, pw, maxfrac);
  if (w.empty()) return false;
  for (int lv = (int)levels.size() - 1; lv >= 0; --lv) {
    const WGraph& fine = lv > 0 ? levels[lv - 1] : g0;
    const std::vector<int32_t>& cm = cmaps[lv];
    std::vector<int8_t> wf(fine.n);
    for (int32_t v = 0; v < fine.n; ++v) wf[v] = w[cm[v]];
    w.swap(wf);
    node_fm(fine, w, pw, maxfrac, 8);
  }
  where.swap(w);
  return pw[0] > 0 && pw[1] > 0;
}

// --------------------------------------------------------------------------------
// nested dissection on a weighted graph (BFS level structures, George-Liu style)
// --------------------------------------------------------------------------------
struct NdFront { std::vector<int32_t> verts; int32_t parent; };

class Dissector {
 public:
  Dissector(const Csr& g, const std::vector<int32_t>& w, int64_t leaf)
      : g_(g), w_(w), leaf_(leaf), mark_(g.n, -1), lev_(g.n, -1) {}

  std::vector<NdFront> run() {
    std::vector<int32_t> ord(g_.n);
    std::iota(ord.begin(), ord.end(), 0);
    ord_.swap(ord);
    tasks_.push_back({0, (int64_t)ord_.size(), -1});
    while (!tasks_.empty()) {
      Task t = tasks_.back();
      tasks_.pop_back();
      process(t);
    }
    return std::move(fronts_);
  }

 private:
  struct Task { int64_t b, e; int32_t parent; };
  const Csr& g_;
  const std::vector<int32_t>& w_;
  int64_t leaf_;
  std::vector<int32_t> mark_, lev_, ord_;
  int32_t stamp_ = 0;
  std::vector<Task> tasks_;
  std::vector<NdFront> fronts_;

  int32_t make_front(int64_t b, int64_t e, int32_t parent) {
    NdFront f;
    f.verts.assign(ord_.begin() + b, ord_.begin() + e);
    f.parent = parent;
    fronts_.push_back(std::move(f));
    return (int32_t)fronts_.size() - 1;
  }

  // BFS from r restricted to mark_ == stamp_; fills lev_; returns max level; order in q
  int32_t bfs(int32_t r, std::vector<int32_t>& q) {
    q.clear();
    q.push_back(r);
    lev_[r] = 0;
    int32_t stampv = stamp_ + 1;  // visited marker: use lev sentinel via vis_
    vis_stamp_++;
    if (vis_.size() < (size_t)g_.n) vis_.assign(g_.n, 0);
    vis_[r] = vis_stamp_;
    (void)stampv;
    size_t h = 0;
    int32_t maxl = 0;
    while (h < q.size()) {
      int32_t v = q[h++];
      for (int64_t k = g_.ptr[v]; k < g_.ptr[v + 1]; ++k) {
        int32_t u = g_.adj[k];
        if (mark_[u] != stamp_ || vis_[u] == vis_stamp_) continue;
        vis_[u] = vis_stamp_;
        lev_[u] = lev_[v] + 1;
        maxl = std::max(maxl, lev_[u]);
        q.push_back(u);
      }
    }
    return maxl;
  }
  std::vector<int32_t> vis_;
  int32_t vis_stamp_ = 0;

  int64_t deg_in(int32_t v) const {
    int64_t d = 0;
    for (int64_t k = g_.ptr[v]; k < g_.ptr[v + 1]; ++k) d += (mark_[g_.adj[k]] == stamp_);
    return d;
  }

  // multilevel vertex separator of the (connected) range; splits it like process() does
  bool multilevel(const Task& t, int64_t W) {
    WGraph g;
    const int32_t n = (int32_t)(t.e - t.b);
    if (loc_.size() < (size_t)g_.n) loc_.assign(g_.n, -1);
    for (int32_t i = 0; i < n; ++i) loc_[ord_[t.b + i]] = i;
    g.n = n;
    g.xadj.assign(n + 1, 0);
    g.vw.resize(n);
    for (int32_t i = 0; i < n; ++i) {
      const int32_t v = ord_[t.b + i];
      g.vw[i] = w_[v];
      for (int64_t k = g_.ptr[v]; k < g_.ptr[v + 1]; ++k) {
        const int32_t u = g_.adj[k];
        if (mark_[u] == stamp_ && u != v) { g.adj.push_back(loc_[u]); g.ew.push_back(1); }
      }
      g.xadj[i + 1] = (int64_t)g.adj.size();
    }
    (void)W;
    std::vector<int8_t> where;
    // sides may hold up to 55 % of the range (c4: 2.16e11 flops at 0.55, 2.26e11 at 0.6,
    // 2.21e11 at 0.52)
    if (!multilevel_separator(g, where, 0.55)) return false;
    std::vector<int32_t> A, B, S;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t v = ord_[t.b + i];
      (where[i] == 0 ? A : (where[i] == 1 ? B : S)).push_back(v);
    }
    if (A.empty() || B.empty() || S.empty()) return false;
    int64_t pos = t.b;
    const int64_t a_b = pos; for (int32_t v : A) ord_[pos++] = v; const int64_t a_e = pos;
    const int64_t b_b = pos; for (int32_t v : B) ord_[pos++] = v; const int64_t b_e = pos;
    const int64_t s_b = pos; for (int32_t v : S) ord_[pos++] = v; const int64_t s_e = pos;
    const int32_t f = make_front(s_b, s_e, t.parent);
    tasks_.push_back({b_b, b_e, f});
    tasks_.push_back({a_b, a_e, f});
    return true;
  }
  std::vector<int32_t> loc_;

  void process(const Task& t) {
    int64_t W = 0;
    ++stamp_;
    for (int64_t i = t.b; i < t.e; ++i) { mark_[ord_[i]] = stamp_; W += w_[ord_[i]]; }
    if (t.e - t.b <= 1) { make_front(t.b, t.e, t.parent); return; }

    // connected components of the range
    std::vector<int32_t> q;
    std::vector<std::vector<int32_t>> comps;
    {
      int64_t seen = 0;
      vis_stamp_++;
      if (vis_.size() < (size_t)g_.n) vis_.assign(g_.n, 0);
      int32_t my = vis_stamp_;
      for (int64_t i = t.b; i < t.e && seen < t.e - t.b; ++i) {
        int32_t r = ord_[i];
        if (vis_[r] == my) continue;
        std::vector<int32_t> c;
        c.push_back(r);
        vis_[r] = my;
        size_t h = 0;
        while (h < c.size()) {
          int32_t v = c[h++];
          for (int64_t k = g_.ptr[v]; k < g_.ptr[v + 1]; ++k) {
            int32_t u = g_.adj[k];
            if (mark_[u] != stamp_ || vis_[u] == my) continue;
            vis_[u] = my;
            c.push_back(u);
          }
        }
        seen += (int64_t)c.size();
        comps.push_back(std::move(c));
      }
    }
    if (comps.size() > 1) {
      // independent components: each becomes its own subtree under the same parent
      int64_t pos = t.b;
      for (auto& c : comps) {
        const int64_t b = pos;
        int64_t cw = 0;
        for (int32_t v : c) { ord_[pos++] = v; cw += w_[v]; }
        if (cw <= leaf_) make_front(b, pos, t.parent);
        else tasks_.push_back({b, pos, t.parent});
      }
      return;
    }

    if (W <= leaf_) { make_front(t.b, t.e, t.parent); return; }
    if (t.e - t.b > 32 && multilevel(t, W)) return;
    // small or unseparated range: BFS level structure from a pseudo-peripheral root
    int32_t r = ord_[t.b];
    {
      int64_t best = INT64_MAX;
      for (int64_t i = t.b; i < t.e; ++i) {
        int64_t d = deg_in(ord_[i]);
        if (d < best) { best = d; r = ord_[i]; }
      }
    }
    int32_t ecc = bfs(r, q);
    for (int it = 0; it < 6; ++it) {
      int32_t cand = -1;
      int64_t bd = INT64_MAX;
      for (int32_t v : q)
        if (lev_[v] == ecc) {
          int64_t d = deg_in(v);
          if (d < bd) { bd = d; cand = v; }
        }
      std::vector<int32_t> q2;
      int32_t e2 = bfs(cand, q2);
      if (e2 > ecc) { ecc = e2; r = cand; q.swap(q2); }
      else { bfs(r, q); break; }
    }
    const int32_t h = ecc;
    if (h < 2) { make_front(t.b, t.e, t.parent); return; }
    std::vector<int64_t> lw(h + 1, 0);
    for (int32_t v : q) lw[lev_[v]] += w_[v];
    // median level
    int64_t cum = 0;
    int32_t s0 = 1;
    for (int32_t l = 0; l <= h; ++l) {
      if (cum + lw[l] >= (W + 1) / 2) { s0 = l; break; }
      cum += lw[l];
    }
    s0 = std::max(1, std::min(h - 1, s0));
    // search nearby levels for a small, balanced separator
    int32_t best_s = s0;
    double best_cost = 1e300;
    {
      std::vector<int64_t> pre(h + 2, 0);
      for (int32_t l = 0; l <= h; ++l) pre[l + 1] = pre[l] + lw[l];
      int32_t span = std::max(2, h / 8);
      for (int32_t s = std::max(1, s0 - span); s <= std::min(h - 1, s0 + span); ++s) {
        double wa = (double)pre[s], wb = (double)(W - pre[s + 1]);
        double mn = std::min(wa, wb);
        if (mn < 0.2 * W && s != s0) continue;
        double cost = (double)lw[s] * (1.0 + 2.0 * std::fabs(wa - wb) / (double)W);
        if (cost < best_cost) { best_cost = cost; best_s = s; }
      }
    }
    const int32_t s = best_s;
    // refine: separator vertices must touch level s+1
    std::vector<int32_t> A, B, S;
    for (int32_t v : q) {
      int32_t l = lev_[v];
      if (l < s) A.push_back(v);
      else if (l > s) B.push_back(v);
      else {
        bool touches = false;
        for (int64_t k = g_.ptr[v]; k < g_.ptr[v + 1] && !touches; ++k) {
          int32_t u = g_.adj[k];
          touches = (mark_[u] == stamp_ && lev_[u] == s + 1);
        }
        (touches ? S : A).push_back(v);
      }
    }
    int64_t pos = t.b;
    int64_t a_b = pos; for (int32_t v : A) ord_[pos++] = v; int64_t a_e = pos;
    int64_t b_b = pos; for (int32_t v : B) ord_[pos++] = v; int64_t b_e = pos;
    int64_t s_b = pos; for (int32_t v : S) ord_[pos++] = v; int64_t s_e = pos;
    int32_t f = make_front(s_b, s_e, t.parent);
    if (b_e > b_b) tasks_.push_back({b_b, b_e, f});
    if (a_e > a_b) tasks_.push_back({a_b, a_e, f});
  }
};

}  // namespace

int build_symbolic(Symbolic& s, const SymOptions& opt, int64_t* pivot_index) {
  const int64_t n = s.n;
  *pivot_index = -1;
  if ((int64_t)s.indptr.size() != n + 1) { last_error() = "indptr size != n+1"; return 5; }
  const int64_t nnz = s.indptr[n];
  if ((int64_t)s.indices.size() != nnz) { last_error() = "indices size != nnz"; return 5; }
  for (int64_t j = 0; j < n; ++j) {
    if (s.indptr[j + 1] < s.indptr[j]) { last_error() = "indptr not monotone"; return 5; }
    for (int64_t k = s.indptr[j]; k < s.indptr[j + 1]; ++k) {
      int64_t r = s.indices[k];
      if (r < 0 || r >= n) { last_error() = "row index out of range"; return 5; }
      if (k > s.indptr[j] && s.indices[k - 1] >= r) { last_error() = "rows not sorted/unique"; return 5; }
    }
  }
  // structural symmetry check (the pattern of a symmetric KKT is symmetric)
  {
    std::vector<int64_t> cnt(n, 0);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = s.indptr[j]; k < s.indptr[j + 1]; ++k) cnt[s.indices[k]]++;
    for (int64_t j = 0; j < n; ++j)
      if (cnt[j] != s.indptr[j + 1] - s.indptr[j]) { last_error() = "pattern is not structurally symmetric"; return 5; }
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = s.indptr[j]; k < s.indptr[j + 1]; ++k) {
        int64_t r = s.indices[k];
        if (!std::binary_search(s.indices.begin() + s.indptr[r], s.indices.begin() + s.indptr[r + 1], j)) {
          last_error() = "pattern is not structurally symmetric";
          return 5;
        }
      }
  }
  const int64_t leaf_size = opt.leaf_size > 0 ? std::max<int64_t>(4, opt.leaf_size) : 64;
  s.pair_mode = (s.n_x > 0);
  s.p_order = (s.pair_mode && opt.p_order == 1) ? 1 : 0;
  if (s.pair_mode && (s.n_c != s.n_x || 2 * s.n_x + s.n_p != n)) {
    last_error() = "KKT mode needs n_c == n_x and n == 2*n_x + n_p";
    return 3;
  }

  // ---- nodes ----------------------------------------------------------------
  // node_unk: unknowns of each graph node.  p unknowns are not graph nodes in KKT mode:
  // with p_order 0 they are all eliminated last, in the root front; with p_order 1 the
  // pairs (p_2k, p_2k+1) are placed after the dissection (below), and an odd last p is
  // eliminated last.
  if (s.p_order) {
    for (int64_t c = s.n_x; c < s.n_x + s.n_p && s.p_order; ++c)
      for (int64_t k = s.indptr[c]; k < s.indptr[c + 1]; ++k) {
        const int64_t r = s.indices[k];
        if (r != c && r >= s.n_x && r < s.n_x + s.n_p) { s.p_order = 0; break; }
      }
  }
  const int64_t n_pp = s.p_order ? s.n_p / 2 : 0;
  std::vector<int64_t> node_of(n, -1);
  std::vector<std::array<int64_t, 2>> node_unk;
  std::vector<int32_t> node_w;
  if (s.pair_mode) {
    std::vector<int64_t> pi;
    int64_t bad = -1;
    if (!match_pairs(s, pi, &bad)) {
      *pivot_index = bad;
      last_error() = "structurally singular: no matching multiplier for state " + std::to_string(bad);
      return 1;
    }
    node_unk.resize(s.n_x);
    for (int64_t i = 0; i < s.n_x; ++i) {
      int64_t l = s.n_x + s.n_p + pi[i];
      node_unk[i] = {i, l};
      node_of[i] = i;
      node_of[l] = i;
    }
    node_w.assign(s.n_x, 2);
    // p pairs enter the dissection as guide nodes (so separators account for their
    // couplings); where they are eliminated is decided after it (p placement below)
    for (int64_t k = 0; k < n_pp; ++k) {
      const int64_t a = s.n_x + 2 * k;
      node_of[a] = node_of[a + 1] = (int64_t)node_unk.size();
      node_unk.push_back({a, a + 1});
      node_w.push_back(2);
    }
  } else {
    node_unk.resize(n);
    for (int64_t i = 0; i < n; ++i) { node_unk[i] = {i, -1}; node_of[i] = i; }
    node_w.assign(n, 1);
  }
  const int64_t N = (int64_t)node_unk.size();

  // ---- node graph -----------------------------------------------------------
  Csr g;
  g.n = (int32_t)N;
  g.ptr.assign(N + 1, 0);
  {
    std::vector<int64_t> stampv(N, -1);
    std::vector<int32_t> tmp;
    std::vector<int32_t> adj;
    for (int64_t a = 0; a < N; ++a) {
      tmp.clear();
      stampv[a] = a;
      for (int t = 0; t < 2; ++t) {
        int64_t u = node_unk[a][t];
        if (u < 0) continue;
        for (int64_t k = s.indptr[u]; k < s.indptr[u + 1]; ++k) {
          int64_t b = node_of[s.indices[k]];
          if (b < 0 || stampv[b] == a) continue;
          stampv[b] = a;
          tmp.push_back((int32_t)b);
        }
      }
      std::sort(tmp.begin(), tmp.end());
      adj.insert(adj.end(), tmp.begin(), tmp.end());
      g.ptr[a + 1] = (int64_t)adj.size();
    }
    g.adj.swap(adj);
  }

  // ---- compression of indistinguishable nodes (equal closed neighbourhoods) -----
  std::vector<int32_t> sv_of(N, -1);
  std::vector<std::vector<int32_t>> sv_members;
  {
    std::vector<uint64_t> key(N);
    auto mix = [](uint64_t x) { x += 1; x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; return x; };
    for (int64_t a = 0; a < N; ++a) {
      uint64_t h = mix((uint64_t)a);     // closed neighbourhood = adj(a) + {a}
      for (int64_t k = g.ptr[a]; k < g.ptr[a + 1]; ++k) h += mix((uint64_t)g.adj[k]);
      key[a] = h;
    }
    std::vector<int32_t> idx(N);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t x, int32_t y) {
      if (key[x] != key[y]) return key[x] < key[y];
      return x < y;
    });
    auto closed_equal = [&](int32_t a, int32_t b) {
      // closed nbhd(a) == closed nbhd(b)  <=>  adj(a)+{a} == adj(b)+{b}
      if (g.ptr[a + 1] - g.ptr[a] != g.ptr[b + 1] - g.ptr[b]) return false;
      if (node_w[a] != node_w[b]) return false;
      std::vector<int32_t> ca(g.adj.begin() + g.ptr[a], g.adj.begin() + g.ptr[a + 1]);
      std::vector<int32_t> cb(g.adj.begin() + g.ptr[b], g.adj.begin() + g.ptr[b + 1]);
      ca.push_back(a); cb.push_back(b);
      std::sort(ca.begin(), ca.end()); std::sort(cb.begin(), cb.end());
      return ca == cb;
    };
    for (int64_t i = 0; i < N;) {
      int64_t j = i;
      while (j < N && key[idx[j]] == key[idx[i]]) ++j;
      // group [i, j) by exact equality
      for (int64_t a = i; a < j; ++a) {
        int32_t va = idx[a];
        if (sv_of[va] >= 0) continue;
        int32_t id = (int32_t)sv_members.size();
        sv_members.push_back({va});
        sv_of[va] = id;
        for (int64_t b = a + 1; b < j; ++b) {
          int32_t vb = idx[b];
          if (sv_of[vb] < 0 && closed_equal(va, vb)) { sv_of[vb] = id; sv_members[id].push_back(vb); }
        }
      }
      i = j;
    }
    // canonical supervertex numbering: by smallest member
    std::vector<int32_t> order(sv_members.size());
    std::iota(order.begin(), order.end(), 0);
    for (auto& m : sv_members) std::sort(m.begin(), m.end());
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return sv_members[x][0] < sv_members[y][0]; });
    std::vector<std::vector<int32_t>> sorted(sv_members.size());
    for (size_t k = 0; k < order.size(); ++k) {
      sorted[k] = std::move(sv_members[order[k]]);
      for (int32_t v : sorted[k]) sv_of[v] = (int32_t)k;
    }
    sv_members.swap(sorted);
  }
  const int64_t NS = (int64_t)sv_members.size();
  Csr cg;
  std::vector<int32_t> cw(NS, 0);
  cg.n = (int32_t)NS;
  cg.ptr.assign(NS + 1, 0);
  {
    std::vector<int64_t> st(NS, -1);
    std::vector<int32_t> tmp, adj;
    for (int64_t a = 0; a < NS; ++a) {
      tmp.clear();
      st[a] = a;
      for (int32_t v : sv_members[a]) {
        cw[a] += node_w[v];
        for (int64_t k = g.ptr[v]; k < g.ptr[v + 1]; ++k) {
          int32_t b = sv_of[g.adj[k]];
          if (st[b] == a) continue;
          st[b] = a;
          tmp.push_back(b);
        }
      }
      std::sort(tmp.begin(), tmp.end());
      adj.insert(adj.end(), tmp.begin(), tmp.end());
      cg.ptr[a + 1] = (int64_t)adj.size();
    }
    cg.adj.swap(adj);
  }

  // ---- nested dissection -> front tree (top-down creation order) --------------
  std::vector<NdFront> nd;
  if (NS > 0) {
    Dissector d(cg, cw, leaf_size);
    nd = d.run();
  }
  // ---- p placement (p_order 1) -------------------------------------------------
  // Pair k = (p_2k, p_2k+1) joins the front that is the lowest common ancestor of the
  // fronts holding its coupled states / multipliers: it is eliminated right after the last
  // of them, as a 2x2 pivot on the Schur complement of everything it couples to (positive
  // definite when C > 0), so no early small pivot (C alone) enters the factor -- the
  // reduced-Hessian structure of the p-last root front, localized.  Pairs without state
  // couplings (or spanning disconnected components) go to the root p-front.  A p-p
  // coupling off the diagonal of C would need both p on one root path: p_order falls back to 0.
  std::vector<int32_t> pfront(n_pp, -1);
  if (n_pp > 0) {
    const int32_t NDF = (int32_t)nd.size();
    std::vector<int32_t> node_front(N, -1), depth(NDF, 0);
    for (int32_t f = 0; f < NDF; ++f) {
      for (int32_t sv : nd[f].verts)
        for (int32_t v : sv_members[sv])
          if (v < s.n_x) node_front[v] = f;
      depth[f] = nd[f].parent >= 0 ? depth[nd[f].parent] + 1 : 0;   // parents are created first
    }
    auto lca = [&](int32_t a, int32_t b) {
      while (a != b && a >= 0 && b >= 0) {
        if (depth[a] >= depth[b]) a = nd[a].parent;
        else b = nd[b].parent;
      }
      return (a == b) ? a : -1;
    };
    for (int64_t k = 0; k < n_pp; ++k) {
      int32_t at = -2;     // -2: no coupling seen yet
      for (int64_t u = s.n_x + 2 * k; u <= s.n_x + 2 * k + 1 && at != -1; ++u)
        for (int64_t q = s.indptr[u]; q < s.indptr[u + 1]; ++q) {
          const int64_t nd_ = node_of[s.indices[q]];
          if (nd_ < 0 || nd_ >= s.n_x) continue;
          const int32_t f = node_front[nd_];
          at = (at == -2) ? f : lca(at, f);
          if (at < 0) { at = -1; break; }
        }
      pfront[k] = at < 0 ? -1 : at;
    }
  }
  int64_t n_root_pairs = 0;
  for (int32_t f : pfront) n_root_pairs += (f < 0);
  const int64_t n_root_p = !s.pair_mode ? 0 : (s.p_order ? 2 * n_root_pairs + (s.n_p & 1) : s.n_p);
  std::vector<std::vector<int32_t>> pairs_of(nd.size());
  for (int64_t k = 0; k < n_pp; ++k)
    if (pfront[k] >= 0) pairs_of[pfront[k]].push_back((int32_t)k);
  if (n_pp > 0) {
    // drop the guide nodes from the fronts, then the fronts left without pivots (their
    // children move up to the nearest kept ancestor)
    const int32_t NDF = (int32_t)nd.size();
    std::vector<int32_t> keep_id(NDF, -1), eff(NDF, -1);
    std::vector<NdFront> kept;
    std::vector<std::vector<int32_t>> kept_pairs;
    for (int32_t f = 0; f < NDF; ++f) {
      std::vector<int32_t> vs;
      for (int32_t sv : nd[f].verts) {
        bool any = false;
        for (int32_t v : sv_members[sv]) any |= (v < s.n_x);
        if (any) vs.push_back(sv);
      }
      const int32_t par = nd[f].parent >= 0 ? eff[nd[f].parent] : -1;
      if (vs.empty() && pairs_of[f].empty()) { eff[f] = par; continue; }
      NdFront nf;
      nf.verts.swap(vs);
      nf.parent = par;
      keep_id[f] = eff[f] = (int32_t)kept.size();
      kept.push_back(std::move(nf));
      kept_pairs.push_back(std::move(pairs_of[f]));
    }
    nd.swap(kept);
    pairs_of.swap(kept_pairs);
  }

  int32_t proot = -1;
  if (s.pair_mode && n_root_p > 0) {
    NdFront pf;
    pf.parent = -1;
    nd.push_back(pf);
    proot = (int32_t)nd.size() - 1;
    for (int32_t f = 0; f < proot; ++f)
      if (nd[f].parent < 0) nd[f].parent = proot;
  }
  const int32_t NF = (int32_t)nd.size();

  // postorder
  std::vector<std::vector<int32_t>> kids(NF);
  std::vector<int32_t> roots;
  for (int32_t f = 0; f < NF; ++f) {
    if (nd[f].parent >= 0) kids[nd[f].parent].push_back(f);
    else roots.push_back(f);
  }
  std::vector<int32_t> post;
  post.reserve(NF);
  {
    std::vector<std::pair<int32_t, size_t>> st;
    for (int32_t r : roots) {
      st.push_back({r, 0});
      while (!st.empty()) {
        auto& top = st.back();
        if (top.second < kids[top.first].size()) {
          int32_t c = kids[top.first][top.second++];
          st.push_back({c, 0});
        } else {
          post.push_back(top.first);
          st.pop_back();
        }
      }
    }
  }
  std::vector<int32_t> newid(NF);
  for (int32_t k = 0; k < NF; ++k) newid[post[k]] = k;

  // ---- positions -------------------------------------------------------------
  s.perm.assign(n, -1);
  s.ipos.assign(n, -1);
  s.fronts.assign(NF, Front());
  s.front_of_pos.assign(n, -1);
  int64_t pos = 0;
  const bool generic_pairs = opt.generic_pairs != 0;
  for (int32_t k = 0; k < NF; ++k) {
    const NdFront& src = nd[post[k]];
    Front& F = s.fronts[k];
    F.first = pos;
    F.parent = src.parent >= 0 ? newid[src.parent] : -1;
    if (post[k] == proot) {
      F.is_root_p = 1;
      // the p block's Schur complement is the (regularized) reduced Gauss-Newton Hessian:
      // 2x2 pivots on consecutive p unknowns halve the serial pivot chain of the root's
      // diagonal blocks (an even count keeps every pair inside one 32-column tile)
      F.pivtype = (s.pair_mode && n_root_p % 2 == 0) ? 2 : 1;
      if (s.p_order) {
        for (int64_t k = 0; k < n_pp; ++k)
          if (pfront[k] < 0) { s.perm[pos++] = s.n_x + 2 * k; s.perm[pos++] = s.n_x + 2 * k + 1; }
        if (s.n_p & 1) s.perm[pos++] = s.n_x + s.n_p - 1;
      } else {
        for (int64_t u = s.n_x; u < s.n_x + s.n_p; ++u) s.perm[pos++] = u;
      }
    } else {
      F.pivtype = s.pair_mode ? 2 : 1;
      for (int32_t sv : src.verts)
        for (int32_t v : sv_members[sv]) {
          if (s.pair_mode && v >= s.n_x) continue;           // guide node (p pair placed below)
          for (int t = 0; t < 2; ++t)
            if (node_unk[v][t] >= 0) s.perm[pos++] = node_unk[v][t];
        }
      // then the p pairs placed here (after the states they couple to)
      for (int32_t k : pairs_of[post[k]]) { s.perm[pos++] = s.n_x + 2 * k; s.perm[pos++] = s.n_x + 2 * k + 1; }
    }
    F.npiv = (int32_t)(pos - F.first);
    // generic mode: consecutive unknowns of an even-sized front are pivoted as 2x2 blocks
    // (half the serial chain of the diagonal-block LDL^T).  A 2x2 principal block of an
    // SPD matrix is SPD, and a block is singular only if the 1x1 pair would be too
    // (d2 = det / a); SGN_GENERIC_PAIRS=0 keeps 1x1 pivots.
    if (!s.pair_mode && generic_pairs && F.npiv % 2 == 0) F.pivtype = 2;
  }
  if (pos != n) { last_error() = "internal: ordering does not cover all unknowns"; return 5; }
  for (int64_t q = 0; q < n; ++q) s.ipos[s.perm[q]] = q;
  for (int32_t k = 0; k < NF; ++k)
    for (int64_t q = s.fronts[k].first; q < s.fronts[k].first + s.fronts[k].npiv; ++q) s.front_of_pos[q] = k;

  // children lists (in postorder id order)
  s.children.clear();
  {
    std::vector<std::vector<int32_t>> ch(NF);
    for (int32_t k = 0; k < NF; ++k)
      if (s.fronts[k].parent >= 0) ch[s.fronts[k].parent].push_back(k);
    for (int32_t k = 0; k < NF; ++k) {
      s.fronts[k].child_begin = (int32_t)s.children.size();
      s.children.insert(s.children.end(), ch[k].begin(), ch[k].end());
      s.fronts[k].child_end = (int32_t)s.children.size();
    }
  }

  // ---- row structures --------------------------------------------------------
  s.srows.clear();
  {
    std::vector<int32_t> mark(n, -1);
    std::vector<int64_t> tmp;
    for (int32_t k = 0; k < NF; ++k) {
      Front& F = s.fronts[k];
      const int64_t last = F.first + F.npiv - 1;
      tmp.clear();
      for (int64_t q = F.first; q <= last; ++q) {
        int64_t u = s.perm[q];
        for (int64_t kk = s.indptr[u]; kk < s.indptr[u + 1]; ++kk) {
          int64_t pv = s.ipos[s.indices[kk]];
          if (pv > last && mark[pv] != k) { mark[pv] = k; tmp.push_back(pv); }
        }
      }
      for (int32_t ci = F.child_begin; ci < F.child_end; ++ci) {
        const Front& C = s.fronts[s.children[ci]];
        int64_t cn = C.nrow - C.npiv;
        for (int64_t t = 0; t < cn; ++t) {
          int64_t pv = s.srows[C.srow_off + t];
          if (pv > last && mark[pv] != k) { mark[pv] = k; tmp.push_back(pv); }
        }
      }
      std::sort(tmp.begin(), tmp.end());
      F.srow_off = (int64_t)s.srows.size();
      s.srows.insert(s.srows.end(), tmp.begin(), tmp.end());
      F.nrow = F.npiv + (int32_t)tmp.size();
      // every struct row must belong to an ancestor (assembly-tree property)
      if (!tmp.empty() && F.parent < 0) {
        last_error() = "internal: root front has a non-empty structure";
        return 5;
      }
    }
  }
  // rel maps
  s.rel.assign(s.srows.size(), 0);
  for (int32_t k = 0; k < NF; ++k) {
    const Front& C = s.fronts[k];
    int64_t cn = C.nrow - C.npiv;
    if (cn == 0) continue;
    const Front& P = s.fronts[C.parent];
    const int64_t plast = P.first + P.npiv - 1;
    const int64_t* pb = s.srows.data() + P.srow_off;
    const int64_t pn = P.nrow - P.npiv;
    for (int64_t t = 0; t < cn; ++t) {
      int64_t pv = s.srows[C.srow_off + t];
      int64_t local;
      if (pv >= P.first && pv <= plast) local = pv - P.first;
      else {
        const int64_t* it = std::lower_bound(pb, pb + pn, pv);
        if (it == pb + pn || *it != pv) { last_error() = "internal: child row missing from parent front"; return 5; }
        local = P.npiv + (it - pb);
      }
      s.rel[C.srow_off + t] = (int32_t)local;
    }
  }
  for (auto& F : s.fronts) F.rel_off = F.srow_off;

  // ---- levels, offsets, stats ------------------------------------------------
  s.n_levels = 0;
  for (int32_t k = 0; k < NF; ++k) {
    Front& F = s.fronts[k];
    int32_t lv = 0;
    for (int32_t ci = F.child_begin; ci < F.child_end; ++ci) lv = std::max(lv, s.fronts[s.children[ci]].level + 1);
    F.level = lv;
    s.n_levels = std::max(s.n_levels, lv + 1);
  }
  s.level_fronts.assign(s.n_levels, {});
  for (int32_t k = 0; k < NF; ++k) s.level_fronts[s.fronts[k].level].push_back(k);

  s.front_doubles = s.u_doubles = s.w_doubles = s.v_doubles = s.z_doubles = s.d_doubles = 0;
  s.ntiles = 0;
  s.nnz_l = 0;
  s.flops = 0;
  s.max_front = s.max_piv = 0;
  int32_t pair_tiles = 1 << 30;
  // The root p-front of a large n_p (>= kNoZTiles pivot tiles, no contribution rows) gets no
  // solve panel: forming L11^{-1} costs npiv^3/3 flops (as much as its factorization) and a
  // column-serial tail, to speed up a handful of solves.  Its solves are blocked
  // substitutions instead (T_RFWD / T_RBWD).  SGN_NOZ_TILES overrides (0: always Z).
  const int64_t kNoZTiles = opt.noz_tiles;   // 0 (default): off; pays only when few solves follow
  for (auto& F : s.fronts) {
    const int64_t nr = F.nrow, ns = F.nrow - F.npiv;
    F.noz = (kNoZTiles > 0 && F.is_root_p && ns == 0 && ptiles(F.npiv) >= kNoZTiles) ? 1 : 0;
    F.foff = s.front_doubles; s.front_doubles += front_ld((int)nr) * nr;
    F.uoff = s.u_doubles; s.u_doubles += ns;
    F.voff = s.v_doubles; s.v_doubles += nr;
    F.zoff = s.z_doubles; s.z_doubles += F.noz ? 0 : front_ld((int)nr) * F.npiv;
    F.doff = s.d_doubles; s.d_doubles += (int64_t)((F.npiv + kTile - 1) / kTile) * kDiagStride;
    const int64_t T = ntiles_front(F.npiv, F.nrow);
    F.tile_base = s.ntiles; s.ntiles += T * (T + 1) / 2;
    s.nnz_l += (int64_t)F.npiv * (F.npiv + 1) / 2 + (int64_t)F.npiv * ns;
    for (int64_t j = 0; j < F.npiv; ++j) {
      double r = (double)(nr - j - 1);
      s.flops += r * r + 2.0 * r;
    }
    s.max_front = std::max<int64_t>(s.max_front, nr);
    s.max_piv = std::max<int64_t>(s.max_piv, F.npiv);
  }

  // 64x64 update / Z blocks (upd_pair bits 0-1) pay where the factorization is throughput
  // bound; a small factorization is bound by its top fronts' pivot chain, which longer
  // tasks only lengthen (config 2: factor 1.63 -> 1.79 ms with pairs, config 4: 51.5 ->
  // 46.6 ms).  pair_min_tiles = 0 (auto): fronts of >= 4 tiles when the factorization has
  // >= 5e9 flops, else none.
  pair_tiles = opt.pair_min_tiles > 0 ? opt.pair_min_tiles : (s.flops >= 5e9 ? 4 : (1 << 30));

  // stabilization kind per position
  // generic mode: every diagonal takes +eps_x (tau-regularized Newton, forward.py:171-186)
  s.kind_pos.assign(n, s.pair_mode ? 0 : 1);
  if (s.pair_mode) {
    for (int64_t q = 0; q < n; ++q) {
      int64_t u = s.perm[q];
      s.kind_pos[q] = (u < s.n_x) ? 1 : (u >= s.n_x + s.n_p ? 2 : 0);
    }
  }

  // ---- assembly entry lists per tile (lower triangle in elimination order) -----
  {
    std::vector<int64_t> cnt(s.ntiles + 1, 0);
    std::vector<int64_t> ent_tile;
    std::vector<int64_t> ent_k;
    std::vector<int32_t> ent_loc;
    ent_tile.reserve(nnz / 2 + n);
    for (int64_t v = 0; v < n; ++v) {
      const int64_t pv = s.ipos[v];
      const int32_t f = s.front_of_pos[pv];
      const Front& F = s.fronts[f];
      const int64_t lc = pv - F.first;
      const int64_t last = F.first + F.npiv - 1;
      const int64_t* sb = s.srows.data() + F.srow_off;
      const int64_t sn = F.nrow - F.npiv;
      for (int64_t k = s.indptr[v]; k < s.indptr[v + 1]; ++k) {
        const int64_t pu = s.ipos[s.indices[k]];
        if (pu < pv) continue;
        int64_t lr;
        if (pu <= last) lr = pu - F.first;
        else {
          const int64_t* it = std::lower_bound(sb, sb + sn, pu);
          if (it == sb + sn || *it != pu) { last_error() = "internal: entry outside front"; return 5; }
          lr = F.npiv + (it - sb);
        }
        const int64_t ti = tile_of_row(F.npiv, (int)lr), tj = tile_of_row(F.npiv, (int)lc);
        const int64_t tile = F.tile_base + ti * (ti + 1) / 2 + tj;
        ent_tile.push_back(tile);
        ent_k.push_back(k);
        ent_loc.push_back((int32_t)((lr - tile_lo(F.npiv, (int)ti)) * kTile + (lc - tile_lo(F.npiv, (int)tj))));
        cnt[tile + 1]++;
      }
    }
    for (int64_t t = 0; t < s.ntiles; ++t) cnt[t + 1] += cnt[t];
    s.tile_ptr = cnt;
    s.tile_nnz.assign(ent_tile.size(), 0);
    s.tile_loc.assign(ent_tile.size(), 0);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (size_t e = 0; e < ent_tile.size(); ++e) {
      int64_t at = fill[ent_tile[e]]++;
      s.tile_nnz[at] = ent_k[e];
      s.tile_loc[at] = ent_loc[e];
    }
  }

  // child rel ranges per parent tile: rows of child c landing in parent tile a are
  // rel[reltile[c.woff + a] .. reltile[c.woff + a + 1])  (rel is increasing)
  s.reltile.clear();
  for (auto& C : s.fronts) {
    C.woff = (int64_t)s.reltile.size();
    if (C.parent < 0) continue;
    const Front& P = s.fronts[C.parent];
    const int32_t TP = ntiles_front(P.npiv, P.nrow);
    const int32_t* rc = s.rel.data() + C.rel_off;
    const int32_t cn = C.nrow - C.npiv;
    for (int32_t a = 0; a <= TP; ++a) {
      const int32_t lo = (a < TP) ? tile_lo(P.npiv, a) : P.nrow;
      s.reltile.push_back((int32_t)(std::lower_bound(rc, rc + cn, lo) - rc));
    }
  }
  s.w_doubles = 0;

  // ---- persistent factorization tasks (topological order) -----------------------------
  // per level: assembly tiles of its fronts; per pivot step k: panel tasks, then Schur
  // updates with the look-ahead column (tj == k+1) first so the next panel can start
  // while the rest of the trailing matrix is updated; finally the solve panels Z.
  s.work.clear();
  s.launches.clear();
  s.ftasks.clear();
  s.n_fcnt = 0;
  for (auto& F : s.fronts) {
    const int64_t P = ptiles(F.npiv), T = ntiles_front(F.npiv, F.nrow);
    F.cbase = s.n_fcnt;
    s.n_fcnt += 1 + 2 * P + T * (T + 1) / 2 + (F.nrow + kTile - 1) / kTile + P * T;   // ... ZC, PANT
    if (T >= (1 << 15)) { last_error() = "front too large for the task schedule"; return 5; }
    F.ftotal = 0;                                         // counted as the tasks are emitted
  }
  // Schur updates off the look-ahead column are applied in groups of up to kUpdGroup
  // consecutive pivot steps by one task (the C tile is read and written once per group;
  // the step tiles stream through shared memory): F_UPDATE b = tj | (ns << 16).
  // SGN_UPD_GROUP overrides (1 = one task per step).
  const int32_t kUpdGroup = std::max(1, opt.upd_group);
  std::vector<int64_t> fcount(s.fronts.size(), 0);
  // Small fronts (<= kFatTiles tiles: the bottom levels) run as ONE task (F_FAT): their
  // tasks and Z blocks back to back in one CTA, without a grab, wait and counter hop per
  // tile.  SGN_FAT_TILES overrides (0: off).
  const int32_t kFatTiles = opt.fat_tiles;   // 0 (default): off (measured: c2 span 1.53 -> 1.64 ms, c5 -1.7 %)
  const int32_t NFr = (int32_t)s.fronts.size();
  std::vector<char> is_fat(NFr, 0);
  std::vector<int64_t> fat_slot(NFr, -1);
  std::vector<std::vector<FTask>> fatbuf(NFr);
  for (int32_t f = 0; f < NFr; ++f) {
    const Front& F = s.fronts[f];
    is_fat[f] = (kFatTiles > 0 && F.npiv > 0 && !F.noz && ntiles_front(F.npiv, F.nrow) <= kFatTiles) ? 1 : 0;
  }
  s.fat.clear();
  auto ft = [&](int32_t kind, int32_t k, int32_t f, int32_t a, int32_t b) {
    if (kind != F_ZPANEL) ++fcount[f];                    // every other kind signals DONE
    if (is_fat[f]) {
      if (fat_slot[f] < 0) { fat_slot[f] = (int64_t)s.ftasks.size(); s.ftasks.push_back(FTask{F_FAT, f, 0, 0}); }
      fatbuf[f].push_back(FTask{kind | (k << 3), f, a, b});
      return;
    }
    s.ftasks.push_back(FTask{kind | (k << 3), f, a, b});
  };
  // Z blocks Z(t, cb) (f_ztask_pre): pivot tiles top-down, then the struct tiles.  Fronts
  // with at least kZInlineSteps pivot steps (the dependency-chain-bound upper fronts) get
  // their pivot-tile blocks right after pivot step t, so the panel is built while the
  // front is still being factored; all other blocks go to a queue (bottom levels first).
  const int32_t kZInlineSteps = std::max(1, opt.zinline);
  std::vector<FTask> zq;
  std::vector<int32_t> zq_level;
  auto z_inline = [&](const Front& F) { return ptiles(F.npiv) >= kZInlineSteps; };
  for (int32_t lv = 0; lv < s.n_levels; ++lv)
    for (int32_t f : s.level_fronts[lv]) {
      const Front& F = s.fronts[f];
      if (F.npiv == 0 || F.noz || is_fat[f]) continue;
      const int32_t P = ptiles(F.npiv), T = ntiles_front(F.npiv, F.nrow);
      for (int32_t t = z_inline(F) ? P : 0; t < P; ++t)
        for (int32_t cb = 0; cb <= t; ++cb) {
          zq.push_back(FTask{F_ZPANEL, f, t, cb});
          zq_level.push_back(lv);
        }
      const bool zpair = (opt.upd_pair & 2) && T >= pair_tiles;
      for (int32_t t = P; t < T; t += zpair ? 2 : 1)   // struct tiles: after every pivot tile
        for (int32_t cb = 0; cb < P; ++cb) {
          if (zpair && cb + 1 < P) {
            zq.push_back(FTask{F_ZPAN2, f, t, cb++});
          } else {
            zq.push_back(FTask{F_ZPANEL, f, t, cb});
            if (zpair && t + 1 < T) {
              zq.push_back(FTask{F_ZPANEL, f, t + 1, cb});
              zq_level.push_back(lv);
            }
          }
          zq_level.push_back(lv);
        }
    }
  // Queued blocks are interleaved into the upper levels' schedule: after every pivot step
  // of level lv, up to zquota blocks of fronts at levels <= lv - 2 (finished by the time
  // the grab reaches them, so they never hold a CTA waiting).  They fill the CTAs the
  // dependency chain of the upper fronts leaves idle; the rest go last.
  // SGN_ZQUOTA overrides the per-step quota (0 = all queued blocks last).
  size_t zhead = 0;
  const int64_t zquota = std::max(0, opt.zquota);
  auto emit_z = [&](int32_t lv) {
    for (int64_t q = 0; q < zquota && zhead < zq.size() && zq_level[zhead] <= lv - std::max(1, opt.zdist); ++q)
      s.ftasks.push_back(zq[zhead++]);
  };
  s.level_task_off.assign(s.n_levels, 0);
  // defer_groups: the grouped updates emitted at step k are held back until the panels and the
  // diagonal update of step k + 1 are in the list.  They are ready when grabbed (their last step's
  // TRSMs finished a step ago), so CTAs run them while step k + 1's TRSMs are in flight, instead of
  // grabbing that step's look-ahead updates early and spinning on the TRSM counters.  Every task
  // that consumes a deferred update (the column's single-step / look-ahead task, the next group,
  // the parent's assembly) still comes later in the list.
  struct Deferred { int32_t kind, k, f, a, b; };
  std::vector<Deferred> deferred;
  const bool defer_groups = opt.defer_groups != 0;
  auto flush_deferred = [&]() {
    for (const Deferred& d : deferred) ft(d.kind, d.k, d.f, d.a, d.b);
    deferred.clear();
  };
  auto fg = [&](int32_t kind, int32_t k, int32_t f, int32_t a, int32_t b) {   // a grouped update
    if (defer_groups) deferred.push_back(Deferred{kind, k, f, a, b});
    else ft(kind, k, f, a, b);
  };
  for (int32_t lv = 0; lv < s.n_levels; ++lv) {
    const auto& fl = s.level_fronts[lv];
    s.level_task_off[lv] = (int64_t)s.ftasks.size();
    for (int32_t f : fl) {
      const int32_t T = ntiles_front(s.fronts[f].npiv, s.fronts[f].nrow);
      if (opt.upd_pair & 4) {                        // 64x64 assembly blocks (F_ASM, k = 1)
        for (int32_t ti = 0; ti < T; ti += 2)
          for (int32_t tj = 0; tj <= ti; tj += 2) ft(F_ASM, 1, f, ti, tj);
      } else {
        for (int32_t ti = 0; ti < T; ++ti)
          for (int32_t tj = 0; tj <= ti; ++tj) ft(F_ASM, 0, f, ti, tj);
      }
    }
    int32_t maxp = 0;
    for (int32_t f : fl) maxp = std::max(maxp, ptiles(s.fronts[f].npiv));
    for (int32_t k = 0; k < maxp; ++k) {
      for (int32_t f : fl) {
        const Front& F = s.fronts[f];
        if (k >= ptiles(F.npiv)) continue;
        const int32_t np = panel_tasks(F.npiv, F.nrow, k);
        for (int32_t t = 0; t < np; ++t) ft(F_PANEL, k, f, t, 0);
      }
      for (int32_t f : fl) {                                 // next diagonal block
        const Front& F = s.fronts[f];
        if (k + 1 < ptiles(F.npiv)) ft(F_DIAGUPD, k, f, 0, 0);
      }
      flush_deferred();                                      // grouped updates of step k - 1
      for (int32_t f : fl) {                                 // look-ahead column first
        const Front& F = s.fronts[f];
        if (k >= ptiles(F.npiv)) continue;
        const int32_t T = ntiles_front(F.npiv, F.nrow);
        const bool diag_next = k + 1 < ptiles(F.npiv);
        if (k + 1 < T) {
          const int32_t t0 = diag_next ? k + 2 : k + 1;
          if ((opt.upd_pair & 8) && T >= pair_tiles) {       // row pairs (F_UPD2, one column)
            // bit 4: below the first row pair (the chain's tiles), the look-ahead column k + 1
            // and the single-step column k + 2 -- both take exactly step k -- go as one 64x64
            // block per row pair: half the tasks of the two most numerous task kinds
            const bool merge = (opt.upd_pair & 16) && diag_next && k + 2 < T;
            for (int32_t ti = t0; ti < T; ti += 2) {
              if (merge && ti > t0) ft(F_UPD2, k, f, ti, (k + 1) | (1 << 16));
              else ft(F_UPD2, k, f, ti, (k + 1) | 0x8000 | (1 << 16));
            }
          } else {
            for (int32_t ti = t0; ti < T; ++ti) ft(F_UPDATE, k, f, ti, k + 1);
          }
        }
      }
      for (int32_t f : fl) {
        const Front& F = s.fronts[f];
        if (k >= ptiles(F.npiv)) continue;
        const int32_t T = ntiles_front(F.npiv, F.nrow);
        const int32_t P = ptiles(F.npiv);
        // column tj: step tj-1 is the look-ahead update, step tj-2 stays a single-step
        // task (it sits one chain step from the pivot block tj), steps <= tj-3 are grouped
        // grouped columns emitting at this step with the same step range pair up: their
        // tiles are updated as 64x64 blocks {ti, ti+1} x {tj, tj+1} (F_UPD2, twice the
        // DMMA work per operand byte; profiles/micro/upd_bench.cu)
        // contribution-block columns (tj >= P) are read only by the parent's assembly, after
        // the front's last step: they take longer groups (upd_group_cb), so each C tile makes
        // fewer HBM round trips (a large front's trailing matrix does not fit in L2)
        auto grouped_ns = [&](int32_t tj) -> int32_t {   // 0: no grouped emission at k
          if (tj >= T || k > tj - 3) return 0;
          const int32_t G = (tj >= P) ? std::max(kUpdGroup, opt.upd_group_cb) : kUpdGroup;
          const int32_t kmax = std::min(tj - 3, P - 1);
          if ((k + 1) % G != 0 && k != kmax) return 0;
          return k - (k / G) * G + 1;
        };
        for (int32_t tj = k + 2; tj < T; ++tj) {
          int32_t ns = 1;
          if (k <= tj - 3) {
            ns = grouped_ns(tj);
            if (ns == 0) continue;
            if ((opt.upd_pair & 1) && T >= pair_tiles && grouped_ns(tj + 1) == ns) {
              for (int32_t ti = tj; ti < T; ti += 2) fg(F_UPD2, k, f, ti, tj | (ns << 16));
              ++tj;
              continue;
            }
          }
          const bool grouped = k <= tj - 3;
          if ((opt.upd_pair & 8) && T >= pair_tiles) {         // row pairs (F_UPD2, one column)
            // (bit 4: column k + 2's rows below its first pair went with the look-ahead column)
            const bool merged = (opt.upd_pair & 16) && !grouped && tj == k + 2 && k + 1 < P;
            for (int32_t ti = tj; ti < (merged ? std::min(tj + 2, T) : T); ti += 2)
              grouped ? fg(F_UPD2, k, f, ti, tj | 0x8000 | (ns << 16)) : ft(F_UPD2, k, f, ti, tj | 0x8000 | (ns << 16));
          } else {
            for (int32_t ti = tj; ti < T; ++ti)
              grouped ? fg(F_UPDATE, k, f, ti, tj | (ns << 16)) : ft(F_UPDATE, k, f, ti, tj | (ns << 16));
          }
        }
      }
      for (int32_t f : fl) {                                 // inline Z row of pivot tile k
        const Front& F = s.fronts[f];
        if (k < ptiles(F.npiv) && z_inline(F) && !F.noz)
          for (int32_t cb = 0; cb <= k; ++cb) ft(F_ZPANEL, 0, f, k, cb);
      }
      emit_z(lv);
    }
    flush_deferred();                                        // before the parents' assembly
  }
  while (zhead < zq.size()) s.ftasks.push_back(zq[zhead++]);
  for (int32_t f = 0; f < NFr; ++f) {                    // fat fronts: sub-tasks, then their Z blocks
    if (!is_fat[f] || fat_slot[f] < 0) continue;
    const Front& F = s.fronts[f];
    const int32_t P = ptiles(F.npiv), T = ntiles_front(F.npiv, F.nrow);
    for (int32_t t = 0; t < T; ++t)
      for (int32_t cb = 0; cb < std::min(t + 1, P); ++cb) fatbuf[f].push_back(FTask{F_ZPANEL, f, t, cb});
    const int64_t a = (int64_t)s.fat.size();
    s.fat.insert(s.fat.end(), fatbuf[f].begin(), fatbuf[f].end());
    if ((int64_t)s.fat.size() > INT32_MAX) { last_error() = "fat task list too large"; return 5; }
    s.ftasks[fat_slot[f]] = FTask{F_FAT, f, (int32_t)a, (int32_t)s.fat.size()};
  }
  for (size_t f = 0; f < s.fronts.size(); ++f) {
    if (fcount[f] > INT32_MAX) { last_error() = "front too large for the task schedule"; return 5; }
    s.fronts[f].ftotal = (int32_t)fcount[f];
  }
  // solve work lists: gather (f), forward GEMV (f, row0, chunk, group), backward dots
  // (f, col0, row chunk, group); each (front, tile) group combines its chunk partials
  s.fwd_off.assign(s.n_levels, 0); s.fwd_cnt.assign(s.n_levels, 0);
  s.bwd_off.assign(s.n_levels, 0); s.bwd_cnt.assign(s.n_levels, 0);
  s.gat_off.assign(s.n_levels, 0); s.gat_cnt.assign(s.n_levels, 0);
  s.lvl_max_piv.assign(s.n_levels, 0);
  s.grp_nchunk.clear(); s.grp_base.clear();
  s.part_doubles = 0;
  // small fronts (the bottom levels) solve as one task each (T_FWD_FAT / T_BWD_FAT);
  // SGN_FAT_SOLVE=0 keeps the tiled tasks
  const bool fat_solve = opt.fat_solve != 0;
  auto fat_front = [&](const Front& F, int32_t rows) {
    return fat_solve && F.npiv >= 1 && F.npiv <= kFwdCols && F.nrow <= rows;
  };
  auto new_group = [&](int32_t nch) {
    s.grp_nchunk.push_back(nch);
    s.grp_base.push_back(s.part_doubles);
    s.part_doubles += (int64_t)nch * 32;
    return (int32_t)s.grp_nchunk.size() - 1;
  };
  for (int32_t lv = 0; lv < s.n_levels; ++lv) {
    s.gat_off[lv] = (int64_t)s.work.size();
    for (int32_t f : s.level_fronts[lv]) {
      s.lvl_max_piv[lv] = std::max(s.lvl_max_piv[lv], s.fronts[f].npiv);
      s.work.push_back({f, 0, 0, 0});
    }
    s.gat_cnt[lv] = (int64_t)s.work.size() - s.gat_off[lv];
    s.fwd_off[lv] = (int64_t)s.work.size();
    for (int32_t f : s.level_fronts[lv]) {
      const Front& F = s.fronts[f];
      if (F.noz) {                                        // blocked substitution, tile by tile
        for (int32_t j = 0; j < ptiles(F.npiv); ++j) s.work.push_back({f, -2 - j, 0, new_group(1)});
        continue;
      }
      // one-task forward fronts of up to 512 rows pay where the solve is bound by its task count
      // (config 4: 95.6 k -> 80.8 k forward tasks, three solves 4.77 -> 4.54 ms); the chain-bound
      // smaller factorizations keep 256 (configs 2 / 3 lose 2-7 % of their solve time at 512)
      const int32_t fat_rows = std::min<int32_t>(kFatRows, s.flops >= 1e11 ? 512 : 256);
      if (fat_front(F, fat_rows)) { s.work.push_back({f, -1, 0, new_group(1)}); continue; }
      for (int32_t r0 = 0; r0 < F.nrow; r0 += kFwdRows) {
        const int32_t cend = (r0 < F.npiv) ? std::min(F.npiv, r0 + kFwdRows) : F.npiv;
        const int32_t nch = std::max(1, (cend + kFwdChunk - 1) / kFwdChunk);
        const int32_t g = new_group(nch);
        for (int32_t k = 0; k < nch; ++k) s.work.push_back({f, r0, k, g});
      }
    }
    s.fwd_cnt[lv] = (int64_t)s.work.size() - s.fwd_off[lv];
    s.bwd_off[lv] = (int64_t)s.work.size();
    for (int32_t f : s.level_fronts[lv]) {
      const Front& F = s.fronts[f];
      if (F.noz) {                                        // last tile first
        for (int32_t j = ptiles(F.npiv) - 1; j >= 0; --j) s.work.push_back({f, -2 - j, 0, new_group(1)});
        continue;
      }
      if (fat_front(F, kFatRowsBwd)) { s.work.push_back({f, -1, 0, new_group(1)}); continue; }
      for (int32_t c0 = 0; c0 < std::max(F.npiv, 1); c0 += kBwdCols) {
        const int32_t rs = (c0 / kBwdRows) * kBwdRows;          // first chunk holding rows >= c0
        const int32_t nch = std::max(1, (F.nrow - rs + kBwdRows - 1) / kBwdRows);
        const int32_t g = new_group(nch);
        for (int32_t k = 0; k < nch; ++k) s.work.push_back({f, c0, rs + k * kBwdRows, g});
      }
    }
    s.bwd_cnt[lv] = (int64_t)s.work.size() - s.bwd_off[lv];
  }
  s.n_groups = (int64_t)s.grp_nchunk.size();

  // ---- persistent solve DAG ------------------------------------------------------------
  // counters: CF(f) = f (forward row groups done), CB(f) = NF + f (backward groups done).
  // The extend-add gather of the forward solve is folded into the GEMV tasks through the
  // inverse map gptr/gsrc, so a front's forward tasks wait directly on its children.
  {
    std::vector<int32_t> nfg(NF, 0), nbg(NF, 0);
    for (int32_t lv = 0; lv < s.n_levels; ++lv) {
      for (int64_t w = s.fwd_off[lv]; w < s.fwd_off[lv] + s.fwd_cnt[lv]; ++w)
        if (s.work[w].b == 0) nfg[s.work[w].f]++;
      for (int64_t w = s.bwd_off[lv]; w < s.bwd_off[lv] + s.bwd_cnt[lv]; ++w)
        if (s.work[w].a <= -2 || s.work[w].b == (s.work[w].a / kBwdRows) * kBwdRows) nbg[s.work[w].f]++;
    }
    // inverse gather map
    {
      std::vector<int64_t> cnt(s.v_doubles + 1, 0);
      for (int32_t f = 0; f < NF; ++f) {
        const Front& F = s.fronts[f];
        for (int32_t ci = F.child_begin; ci < F.child_end; ++ci) {
          const Front& C = s.fronts[s.children[ci]];
          for (int64_t t = 0; t < C.nrow - C.npiv; ++t) cnt[F.voff + s.rel[C.rel_off + t] + 1]++;
        }
      }
      for (int64_t q = 0; q < s.v_doubles; ++q) cnt[q + 1] += cnt[q];
      s.gptr = cnt;
      s.gsrc.assign(cnt[s.v_doubles], 0);
      std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
      for (int32_t f = 0; f < NF; ++f) {
        const Front& F = s.fronts[f];
        for (int32_t ci = F.child_begin; ci < F.child_end; ++ci) {   // child order = sum order
          const Front& C = s.fronts[s.children[ci]];
          for (int64_t t = 0; t < C.nrow - C.npiv; ++t)
            s.gsrc[fill[F.voff + s.rel[C.rel_off + t]]++] = (int32_t)(C.uoff + t);
        }
      }
    }
    s.stasks.clear(); s.swaits.clear();
    s.n_scnt = 2 * NF;
    auto add = [&](int32_t kind, const Work& w, int32_t sig, const std::vector<std::pair<int32_t, int32_t>>& ws) {
      Task t{kind, w.f, w.a, w.b, w.c, sig, (int32_t)(s.swaits.size() / 2), 0};
      for (auto& p : ws) { s.swaits.push_back(p.first); s.swaits.push_back(p.second); }
      t.w1 = (int32_t)(s.swaits.size() / 2);
      s.stasks.push_back(t);
    };
    for (int32_t lv = 0; lv < s.n_levels; ++lv) {
      for (int64_t w = s.fwd_off[lv]; w < s.fwd_off[lv] + s.fwd_cnt[lv]; ++w) {
        const Front& F = s.fronts[s.work[w].f];
        std::vector<std::pair<int32_t, int32_t>> ch;
        for (int32_t ci = F.child_begin; ci < F.child_end; ++ci) ch.push_back({s.children[ci], nfg[s.children[ci]]});
        add(s.work[w].a <= -2 ? T_RFWD : (s.work[w].a < 0 ? T_FWD_FAT : T_FWD), s.work[w], s.work[w].f, ch);
      }
    }
    for (int32_t lv = s.n_levels - 1; lv >= 0; --lv) {
      for (int64_t w = s.bwd_off[lv]; w < s.bwd_off[lv] + s.bwd_cnt[lv]; ++w) {
        const int32_t f = s.work[w].f;
        const int32_t p = s.fronts[f].parent;
        const int32_t kind = s.work[w].a <= -2 ? T_RBWD : (s.work[w].a < 0 ? T_BWD_FAT : T_BWD);
        if (p >= 0) add(kind, s.work[w], NF + f, {{NF + p, nbg[p]}});
        else add(kind, s.work[w], NF + f, {{f, nfg[f]}});
      }
    }
  }
  return 0;
}

}  // namespace sgn
