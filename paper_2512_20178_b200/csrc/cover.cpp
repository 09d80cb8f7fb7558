// cover.cpp -- canonical minimum vertex cover of one off-diagonal block.
//
// PAPER.md L363-375 (section V-C): the block A^(p,q) is a bipartite graph
// G = (R u C, E) with one edge per nonzero; the optimal joint plan is a
// minimum (uniform-)weight vertex cover, found by the paper as a minimum s-t
// cut (Dinic).  For unit weights (the paper's "common case", L397) the cut is
// obtained more cheaply from a maximum matching (König-Egerváry): run
// Hopcroft-Karp (O(E sqrt V)), then Z = vertices reachable from unmatched
// rows by alternating paths (any edge row->col, matched edge col->row).  Z
// plus s is exactly the s-reachable set of the residual graph for the
// matching's flow, i.e. the minimal minimum cut, which is the same for EVERY
// maximum flow (R1, R16).  Hence the cover
//     rows R \ Z  (arc s->i cut)   and   cols C n Z  (arc j->t cut)
// is canonical ("row-max"), bit-identical to the oracle's Dinic read-off.
// The col-max rule is the row-max rule of the transposed block.
//
// Weighted covers (Eqs. 4-8): the exact
// minimum-weight cover is the minimum s-t cut of the paper's network (L373:
// s->i capacity w_row_i, j->t capacity w_col_j, i->j infinite), found by
// Dinic's algorithm (L375) -- BFS level graph, blocking flow by iterative DFS
// with current-arc pointers -- and read off the residual graph the same way
// (s-reachable set; canonical for every maximum flow).
#include <cstdint>
#include <limits>
#include <vector>

#include "shiro_internal.h"

namespace shiro {

namespace {

// Bipartite graph, rows 0..nr-1 with adjacency (ap, adj) to cols 0..nc-1.
struct Bip {
  int32_t nr = 0, nc = 0;
  std::vector<int64_t> ap;
  std::vector<int32_t> adj;
};

constexpr int32_t kInf = 0x7fffffff;

void hopcroft_karp(const Bip &g, std::vector<int32_t> &mr, std::vector<int32_t> &mc) {
  mr.assign(g.nr, -1);
  mc.assign(g.nc, -1);
  // greedy initial matching
  for (int32_t u = 0; u < g.nr; ++u)
    for (int64_t k = g.ap[u]; k < g.ap[u + 1]; ++k)
      if (mc[g.adj[k]] < 0) { mr[u] = g.adj[k]; mc[g.adj[k]] = u; break; }
  std::vector<int32_t> dist(g.nr), queue(g.nr), stack;
  std::vector<int64_t> it(g.nr);
  for (;;) {
    // BFS layering from free rows
    int32_t qh = 0, qt = 0;
    for (int32_t u = 0; u < g.nr; ++u) {
      if (mr[u] < 0) { dist[u] = 0; queue[qt++] = u; } else dist[u] = kInf;
    }
    bool found = false;
    while (qh < qt) {
      int32_t u = queue[qh++];
      for (int64_t k = g.ap[u]; k < g.ap[u + 1]; ++k) {
        int32_t w = mc[g.adj[k]];
        if (w < 0) found = true;
        else if (dist[w] == kInf) { dist[w] = dist[u] + 1; queue[qt++] = w; }
      }
    }
    if (!found) break;
    // iterative DFS along layers from every free row
    for (int32_t u = 0; u < g.nr; ++u) it[u] = g.ap[u];
    for (int32_t r0 = 0; r0 < g.nr; ++r0) {
      if (mr[r0] >= 0) continue;
      stack.clear();
      stack.push_back(r0);
      while (!stack.empty()) {
        int32_t u = stack.back();
        if (it[u] == g.ap[u + 1]) {         // dead end
          dist[u] = kInf;
          stack.pop_back();
          if (!stack.empty()) ++it[stack.back()];
          continue;
        }
        int32_t v = g.adj[it[u]];
        int32_t w = mc[v];
        if (w < 0) {                         // augment along the stack
          for (int32_t x : stack) {
            int32_t vx = g.adj[it[x]];
            mr[x] = vx;
            mc[vx] = x;
          }
          break;
        }
        if (dist[w] == dist[u] + 1) stack.push_back(w);
        else ++it[u];
      }
    }
  }
}

// Z-BFS: rows/cols reachable from unmatched rows by alternating paths.
void konig_cover(const Bip &g, const std::vector<int32_t> &mr, const std::vector<int32_t> &mc,
                 std::vector<uint8_t> &sel_row, std::vector<uint8_t> &sel_col) {
  std::vector<uint8_t> zr(g.nr, 0), zc(g.nc, 0);
  std::vector<int32_t> queue;
  queue.reserve(g.nr);
  for (int32_t u = 0; u < g.nr; ++u)
    if (mr[u] < 0) { zr[u] = 1; queue.push_back(u); }
  for (size_t h = 0; h < queue.size(); ++h) {
    int32_t u = queue[h];
    for (int64_t k = g.ap[u]; k < g.ap[u + 1]; ++k) {
      int32_t v = g.adj[k];
      if (zc[v]) continue;
      zc[v] = 1;
      int32_t w = mc[v];   // matched (else an augmenting path would exist)
      if (w >= 0 && !zr[w]) { zr[w] = 1; queue.push_back(w); }
    }
  }
  sel_row.resize(g.nr);
  sel_col.resize(g.nc);
  for (int32_t u = 0; u < g.nr; ++u) sel_row[u] = !zr[u];
  for (int32_t v = 0; v < g.nc; ++v) sel_col[v] = zc[v];
}

// Dinic on the block network.  Nodes: 0 = s, 1..nr rows, nr+1..nr+nc cols,
// nr+nc+1 = t.  Arcs in pairs (a, a^1).
struct FlowNet {
  int32_t n = 0;
  std::vector<int64_t> head_start;      // CSR of arcs per node
  std::vector<int32_t> to;
  std::vector<int64_t> cap;
  std::vector<int64_t> rev;             // index of the reverse arc
};

FlowNet build_net(int32_t nr, int32_t nc, const std::vector<int64_t> &ap,
                  const std::vector<int32_t> &adj, const std::vector<int64_t> &wr,
                  const std::vector<int64_t> &wc, int64_t inf) {
  FlowNet f;
  f.n = nr + nc + 2;
  const int32_t S = 0, T = nr + nc + 1;
  std::vector<int64_t> deg(f.n + 1, 0);
  auto cnt = [&](int32_t a, int32_t b) { deg[a + 1]++; deg[b + 1]++; };
  for (int32_t u = 0; u < nr; ++u) cnt(S, 1 + u);
  for (int32_t u = 0; u < nr; ++u)
    for (int64_t k = ap[u]; k < ap[u + 1]; ++k) cnt(1 + u, 1 + nr + adj[k]);
  for (int32_t v = 0; v < nc; ++v) cnt(1 + nr + v, T);
  for (int32_t x = 0; x < f.n; ++x) deg[x + 1] += deg[x];
  f.head_start = deg;
  const int64_t m = deg[f.n];
  f.to.resize(m);
  f.cap.resize(m);
  f.rev.resize(m);
  std::vector<int64_t> fill(deg.begin(), deg.end() - 1);
  auto add = [&](int32_t a, int32_t b, int64_t c) {
    const int64_t ia = fill[a]++, ib = fill[b]++;
    f.to[ia] = b; f.cap[ia] = c; f.rev[ia] = ib;
    f.to[ib] = a; f.cap[ib] = 0; f.rev[ib] = ia;
  };
  for (int32_t u = 0; u < nr; ++u) add(S, 1 + u, wr[u]);
  for (int32_t u = 0; u < nr; ++u)
    for (int64_t k = ap[u]; k < ap[u + 1]; ++k) add(1 + u, 1 + nr + adj[k], inf);
  for (int32_t v = 0; v < nc; ++v) add(1 + nr + v, T, wc[v]);
  return f;
}

int64_t dinic(FlowNet &f, int32_t S, int32_t T) {
  int64_t flow = 0;
  std::vector<int32_t> level(f.n), queue(f.n), path;
  std::vector<int64_t> it(f.n), path_arc;
  for (;;) {
    std::fill(level.begin(), level.end(), -1);
    int32_t qh = 0, qt = 0;
    level[S] = 0;
    queue[qt++] = S;
    while (qh < qt) {
      const int32_t x = queue[qh++];
      for (int64_t a = f.head_start[x]; a < f.head_start[x + 1]; ++a)
        if (f.cap[a] > 0 && level[f.to[a]] < 0) {
          level[f.to[a]] = level[x] + 1;
          queue[qt++] = f.to[a];
        }
    }
    if (level[T] < 0) break;
    for (int32_t x = 0; x < f.n; ++x) it[x] = f.head_start[x];
    // blocking flow: iterative DFS along the level graph
    for (;;) {
      path.assign(1, S);
      path_arc.clear();
      bool found = false;
      while (!path.empty()) {
        const int32_t x = path.back();
        if (x == T) { found = true; break; }
        int64_t &a = it[x];
        while (a < f.head_start[x + 1] && !(f.cap[a] > 0 && level[f.to[a]] == level[x] + 1)) ++a;
        if (a == f.head_start[x + 1]) {      // dead end: retreat
          level[x] = -1;
          path.pop_back();
          if (!path_arc.empty()) { path_arc.pop_back(); }
          if (!path.empty()) ++it[path.back()];
          continue;
        }
        path_arc.push_back(a);
        path.push_back(f.to[a]);
      }
      if (!found) break;
      int64_t push = std::numeric_limits<int64_t>::max();
      for (int64_t a : path_arc) push = std::min(push, f.cap[a]);
      for (int64_t a : path_arc) { f.cap[a] -= push; f.cap[f.rev[a]] += push; }
      flow += push;
    }
  }
  return flow;
}

// row-max canonical cut of the weighted network: S = s-reachable set
int64_t weighted_rowmax(int32_t nr, int32_t nc, const std::vector<int64_t> &ap,
                        const std::vector<int32_t> &adj, const std::vector<int64_t> &wr,
                        const std::vector<int64_t> &wc, std::vector<uint8_t> &sel_row,
                        std::vector<uint8_t> &sel_col) {
  int64_t inf = 1;
  for (int64_t w : wr) {
    if (w <= 0) throw Error(SHIRO_E_ARG, "weights must be positive");
    inf += w;
  }
  for (int64_t w : wc)
    if (w <= 0) throw Error(SHIRO_E_ARG, "weights must be positive");
  FlowNet f = build_net(nr, nc, ap, adj, wr, wc, inf);
  const int32_t S = 0, T = nr + nc + 1;
  const int64_t flow = dinic(f, S, T);
  std::vector<uint8_t> seen(f.n, 0);
  std::vector<int32_t> queue{S};
  seen[S] = 1;
  for (size_t h = 0; h < queue.size(); ++h) {
    const int32_t x = queue[h];
    for (int64_t a = f.head_start[x]; a < f.head_start[x + 1]; ++a)
      if (f.cap[a] > 0 && !seen[f.to[a]]) { seen[f.to[a]] = 1; queue.push_back(f.to[a]); }
  }
  if (seen[T]) throw Error(SHIRO_E_INTERNAL, "max flow left an augmenting path");
  sel_row.assign(nr, 0);
  sel_col.assign(nc, 0);
  for (int32_t u = 0; u < nr; ++u) sel_row[u] = !seen[1 + u];
  for (int32_t v = 0; v < nc; ++v) sel_col[v] = seen[1 + nr + v];
  return flow;
}

}  // namespace

int64_t block_cover_weighted(int32_t nr, int32_t nc, const std::vector<int64_t> &ap,
                             const std::vector<int32_t> &adj, const std::vector<int64_t> &w_row,
                             const std::vector<int64_t> &w_col, bool colmax,
                             std::vector<uint8_t> &sel_row, std::vector<uint8_t> &sel_col) {
  int64_t flow;
  if (!colmax) {
    flow = weighted_rowmax(nr, nc, ap, adj, w_row, w_col, sel_row, sel_col);
  } else {
    // col-max = row-max of the transposed block with the weights swapped
    std::vector<int64_t> tap(nc + 1, 0);
    for (int64_t k = 0; k < (int64_t)adj.size(); ++k) tap[adj[k] + 1]++;
    for (int32_t v = 0; v < nc; ++v) tap[v + 1] += tap[v];
    std::vector<int32_t> tadj(adj.size());
    std::vector<int64_t> fill(tap.begin(), tap.end() - 1);
    for (int32_t u = 0; u < nr; ++u)
      for (int64_t k = ap[u]; k < ap[u + 1]; ++k) tadj[fill[adj[k]]++] = u;
    flow = weighted_rowmax(nc, nr, tap, tadj, w_col, w_row, sel_col, sel_row);
  }
  // feasibility (Eq. 7) and max-flow = min-cut: weight of the cover = flow
  int64_t wsum = 0;
  for (int32_t u = 0; u < nr; ++u) wsum += sel_row[u] ? w_row[u] : 0;
  for (int32_t v = 0; v < nc; ++v) wsum += sel_col[v] ? w_col[v] : 0;
  for (int32_t u = 0; u < nr; ++u)
    for (int64_t k = ap[u]; k < ap[u + 1]; ++k)
      if (!sel_row[u] && !sel_col[adj[k]])
        throw Error(SHIRO_E_INTERNAL, "infeasible weighted cover (Eq. 7)");
  if (wsum != flow) throw Error(SHIRO_E_INTERNAL, "cover weight != max flow");
  return flow;
}

// rows: local row ids (ascending, distinct) of the block; for row t its
// column ids (already mapped to 0..nc-1) are adj[ap[t]..ap[t+1]).
int64_t block_cover(int32_t nr, int32_t nc, const std::vector<int64_t> &ap,
                    const std::vector<int32_t> &adj, bool colmax, std::vector<uint8_t> &sel_row,
                    std::vector<uint8_t> &sel_col) {
  std::vector<int32_t> mr, mc;
  if (!colmax) {
    Bip g;
    g.nr = nr; g.nc = nc; g.ap = ap; g.adj = adj;
    hopcroft_karp(g, mr, mc);
    konig_cover(g, mr, mc, sel_row, sel_col);
  } else {
    // transpose: rows' = cols
    Bip t;
    t.nr = nc; t.nc = nr;
    t.ap.assign(nc + 1, 0);
    for (int64_t k = 0; k < (int64_t)adj.size(); ++k) t.ap[adj[k] + 1]++;
    for (int32_t v = 0; v < nc; ++v) t.ap[v + 1] += t.ap[v];
    t.adj.resize(adj.size());
    std::vector<int64_t> fill(t.ap.begin(), t.ap.end() - 1);
    for (int32_t u = 0; u < nr; ++u)
      for (int64_t k = ap[u]; k < ap[u + 1]; ++k) t.adj[fill[adj[k]]++] = u;
    hopcroft_karp(t, mr, mc);
    konig_cover(t, mr, mc, sel_col, sel_row);   // roles swapped back
  }
  int64_t mu = 0;
  for (auto x : sel_row) mu += x;
  for (auto x : sel_col) mu += x;
  // feasibility (Eq. 7) and König: |cover| = |matching|
  int64_t msize = 0;
  for (auto x : mr) msize += (x >= 0);
  for (int32_t u = 0; u < nr; ++u)
    for (int64_t k = ap[u]; k < ap[u + 1]; ++k)
      if (!sel_row[u] && !sel_col[adj[k]])
        throw Error(SHIRO_E_INTERNAL, "infeasible cover (Eq. 7)");
  if (mu != msize) throw Error(SHIRO_E_INTERNAL, "cover size != matching size (Koenig)");
  return mu;
}

}  // namespace shiro
