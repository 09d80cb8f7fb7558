/*
 * oracle_core.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the SHIRO hot path
 * (arXiv 2512.20178).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header or constant with the CUDA product in paper_2512_20178_b200/.
 *
 * Two routines live here because they must run on full-size inputs:
 *
 *   oracle_spmm_f64      C = A*B by its plain definition (PAPER.md,
 *                        section II-A: "C = AB"; SPEC.md L54-57 fixes the
 *                        accumulation order: ascending column index within a
 *                        row).  fp64 accumulation over fp32 inputs.
 *
 *   oracle_dinic_cover   Minimum weighted vertex cover of one bipartite block
 *                        via the paper's flow network (PAPER.md L372-375,
 *                        section V-C2): s->i capacity w_row_i, j->t capacity
 *                        w_col_j, i->j capacity "infinite" (= sum of finite
 *                        capacities + 1), max flow by Dinic's
 *                        algorithm, cover read off the minimum
 *                        cut.  Two canonical cuts (reading R1):
 *                          rule 0 (row-max): S = vertices reachable from s in
 *                            the final residual graph; selected rows = rows
 *                            not in S (arc s->i cut), selected cols = cols in
 *                            S (arc j->t cut)  -- SPEC.md L196.
 *                          rule 1 (col-max): T = vertices that reach t in the
 *                            residual graph, S = complement; same read-off.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle_core.c -o liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* C[r, :] = sum_k A[r, k] * B[k, :]  for every requested row r.              */
/* row_ptr/col/val: CSR of the rows (global column ids into B).              */
/* rows == NULL means all nrows rows, output row r -> C[r].                  */
/* rows != NULL: output row t (0..nrows-1) is CSR row rows[t].               */
/* ------------------------------------------------------------------------ */
void oracle_spmm_f64(int64_t nrows, int64_t N, const int64_t *row_ptr,
                     const int32_t *col, const float *val, const float *B,
                     int64_t ldb, const int64_t *rows, double *C) {
  int64_t t;
#pragma omp parallel for schedule(dynamic, 64)
  for (t = 0; t < nrows; t++) {
    int64_t r = rows ? rows[t] : t;
    double *c = C + t * N;
    for (int64_t x = 0; x < N; x++) c[x] = 0.0;
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; k++) {
      double a = (double)val[k];
      const float *b = B + (int64_t)col[k] * ldb;
      for (int64_t x = 0; x < N; x++) c[x] += a * (double)b[x];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Dinic max flow on the bipartite cover network.                            */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t nv;      /* vertices: s=0, rows 1..nr, cols nr+1..nr+nc, t=nr+nc+1 */
  int64_t na;      /* arcs (each with a paired reverse arc: a ^ 1)           */
  int64_t *first;  /* CSR over tail vertex: arcs first[v]..first[v+1]-1      */
  int64_t *head;   /* head vertex of arc (by CSR slot)                        */
  int64_t *cap;    /* residual capacity of arc (by CSR slot)                  */
  int64_t *rev;    /* CSR slot of the reverse arc                             */
} net_t;

static void net_free(net_t *g) {
  free(g->first); free(g->head); free(g->cap); free(g->rev);
}

/* Build the network of PAPER.md L373. Returns 0 on success. */
static int net_build(net_t *g, int32_t nr, int32_t nc, int64_t ne,
                     const int32_t *er, const int32_t *ec,
                     const int64_t *w_row, const int64_t *w_col) {
  int64_t nv = (int64_t)nr + nc + 2, s = 0, t = (int64_t)nr + nc + 1;
  int64_t na = 2 * ((int64_t)nr + nc + ne);
  int64_t inf = 1, i;
  for (i = 0; i < nr; i++) inf += w_row[i];
  for (i = 0; i < nc; i++) inf += w_col[i];
  /* arcs listed as (tail, head, cap) pairs: forward then reverse */
  int64_t *tail = malloc(sizeof(int64_t) * na), *hd = malloc(sizeof(int64_t) * na);
  int64_t *cp = malloc(sizeof(int64_t) * na);
  if (!tail || !hd || !cp) return 1;
  int64_t a = 0;
#define ADD_ARC(u, v, c) do { tail[a] = (u); hd[a] = (v); cp[a] = (c); a++; \
                              tail[a] = (v); hd[a] = (u); cp[a] = 0; a++; } while (0)
  for (i = 0; i < nr; i++) ADD_ARC(s, 1 + i, w_row[i]);
  for (i = 0; i < ne; i++) ADD_ARC(1 + (int64_t)er[i], 1 + (int64_t)nr + ec[i], inf);
  for (i = 0; i < nc; i++) ADD_ARC(1 + (int64_t)nr + i, t, w_col[i]);
#undef ADD_ARC
  g->nv = nv; g->na = na;
  g->first = calloc(nv + 1, sizeof(int64_t));
  g->head = malloc(sizeof(int64_t) * na);
  g->cap = malloc(sizeof(int64_t) * na);
  g->rev = malloc(sizeof(int64_t) * na);
  int64_t *slot = malloc(sizeof(int64_t) * na), *fill = malloc(sizeof(int64_t) * nv);
  if (!g->first || !g->head || !g->cap || !g->rev || !slot || !fill) return 1;
  for (i = 0; i < na; i++) g->first[tail[i] + 1]++;
  for (i = 0; i < nv; i++) g->first[i + 1] += g->first[i];
  for (i = 0; i < nv; i++) fill[i] = g->first[i];
  for (i = 0; i < na; i++) slot[i] = fill[tail[i]]++;   /* stable: insertion order */
  for (i = 0; i < na; i++) {
    g->head[slot[i]] = hd[i];
    g->cap[slot[i]] = cp[i];
    g->rev[slot[i]] = slot[i ^ 1];
  }
  free(tail); free(hd); free(cp); free(slot); free(fill);
  return 0;
}

/* BFS level graph from s over arcs with residual capacity. */
static int bfs_levels(const net_t *g, int64_t s, int64_t t, int64_t *level,
                      int64_t *queue) {
  for (int64_t v = 0; v < g->nv; v++) level[v] = -1;
  int64_t qh = 0, qt = 0;
  level[s] = 0; queue[qt++] = s;
  while (qh < qt) {
    int64_t u = queue[qh++];
    for (int64_t a = g->first[u]; a < g->first[u + 1]; a++) {
      if (g->cap[a] > 0 && level[g->head[a]] < 0) {
        level[g->head[a]] = level[u] + 1;
        queue[qt++] = g->head[a];
      }
    }
  }
  return level[t] >= 0;
}

/* One blocking flow: repeated iterative DFS s->t along level+1 arcs with
 * current-arc pointers (Dinic 1970).  Returns the flow pushed. */
static int64_t blocking_flow(net_t *g, int64_t s, int64_t t, const int64_t *level,
                             int64_t *cur, int64_t *stack_arc) {
  int64_t total = 0;
  for (int64_t v = 0; v < g->nv; v++) cur[v] = g->first[v];
  for (;;) {
    /* find one augmenting path in the level graph */
    int64_t depth = 0, u = s;
    while (u != t) {
      int64_t a;
      for (a = cur[u]; a < g->first[u + 1]; a++) {
        int64_t v = g->head[a];
        if (g->cap[a] > 0 && level[v] == level[u] + 1) break;
      }
      cur[u] = a;
      if (a == g->first[u + 1]) {          /* dead end: retreat */
        if (depth == 0) return total;
        depth--;
        int64_t back = stack_arc[depth];
        u = g->head[g->rev[back]];          /* tail of the arc we came by */
        cur[u]++;                           /* that arc leads to a dead end */
        continue;
      }
      stack_arc[depth++] = a;
      u = g->head[a];
    }
    /* bottleneck and augment */
    int64_t f = INT64_MAX;
    for (int64_t d = 0; d < depth; d++)
      if (g->cap[stack_arc[d]] < f) f = g->cap[stack_arc[d]];
    for (int64_t d = 0; d < depth; d++) {
      g->cap[stack_arc[d]] -= f;
      g->cap[g->rev[stack_arc[d]]] += f;
    }
    total += f;
  }
}

/*
 * Minimum weighted vertex cover of the bipartite block with nr row vertices,
 * nc column vertices and ne edges (er[e], ec[e]) given as local vertex ids.
 * w_row / w_col: positive vertex weights (uniform = all ones).
 * rule: 0 = row-max canonical cut (s-reachable set), 1 = col-max (t-side).
 * Outputs sel_row[nr], sel_col[nc] in {0,1}; *flow = max-flow value.
 * Returns 0 on success, 1 on allocation failure, 2 if the read-off cover is
 * infeasible or its weight differs from the flow (must never happen).
 */
int oracle_dinic_cover(int32_t nr, int32_t nc, int64_t ne, const int32_t *er,
                       const int32_t *ec, const int64_t *w_row,
                       const int64_t *w_col, int32_t rule, uint8_t *sel_row,
                       uint8_t *sel_col, int64_t *flow) {
  net_t g;
  memset(&g, 0, sizeof g);
  if (net_build(&g, nr, nc, ne, er, ec, w_row, w_col)) return 1;
  int64_t s = 0, t = (int64_t)nr + nc + 1, f = 0;
  int64_t *level = malloc(sizeof(int64_t) * g.nv);
  int64_t *queue = malloc(sizeof(int64_t) * g.nv);
  int64_t *cur = malloc(sizeof(int64_t) * (g.nv + 1));
  int64_t *stk = malloc(sizeof(int64_t) * (g.nv + 1));
  uint8_t *mark = calloc(g.nv, 1);
  if (!level || !queue || !cur || !stk || !mark) return 1;
  while (bfs_levels(&g, s, t, level, queue)) f += blocking_flow(&g, s, t, level, cur, stk);
  *flow = f;

  int64_t qh = 0, qt = 0;
  if (rule == 0) {
    /* S = vertices reachable from s along arcs with residual capacity */
    mark[s] = 1; queue[qt++] = s;
    while (qh < qt) {
      int64_t u = queue[qh++];
      for (int64_t a = g.first[u]; a < g.first[u + 1]; a++)
        if (g.cap[a] > 0 && !mark[g.head[a]]) { mark[g.head[a]] = 1; queue[qt++] = g.head[a]; }
    }
    for (int32_t i = 0; i < nr; i++) sel_row[i] = !mark[1 + i];
    for (int32_t j = 0; j < nc; j++) sel_col[j] = mark[1 + (int64_t)nr + j];
  } else {
    /* T = vertices that reach t: walk arcs backwards. Arc u->v is residual
     * iff cap[slot(u->v)] > 0; from v, slot(u->v) = rev[slot(v->u)]. */
    mark[t] = 1; queue[qt++] = t;
    while (qh < qt) {
      int64_t v = queue[qh++];
      for (int64_t a = g.first[v]; a < g.first[v + 1]; a++) {
        int64_t u = g.head[a];
        if (g.cap[g.rev[a]] > 0 && !mark[u]) { mark[u] = 1; queue[qt++] = u; }
      }
    }
    for (int32_t i = 0; i < nr; i++) sel_row[i] = mark[1 + i];
    for (int32_t j = 0; j < nc; j++) sel_col[j] = !mark[1 + (int64_t)nr + j];
  }
  /* feasibility (Eq. 7) and max-flow = min-cut weight */
  int rc = 0;
  for (int64_t e = 0; e < ne; e++)
    if (!sel_row[er[e]] && !sel_col[ec[e]]) rc = 2;
  int64_t w = 0;
  for (int32_t i = 0; i < nr; i++) w += sel_row[i] ? w_row[i] : 0;
  for (int32_t j = 0; j < nc; j++) w += sel_col[j] ? w_col[j] : 0;
  if (w != f) rc = 2;
  free(level); free(queue); free(cur); free(stk); free(mark);
  net_free(&g);
  return rc;
}
