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
#include <cstdint>
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

}  // namespace

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
