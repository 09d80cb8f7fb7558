// plan.cpp -- the offline phase of SHIRO's joint row/column strategy.
//
// PAPER.md L299-300 (section V-A, workflow steps 1-2): "Each process i
// analyzes the sparsity structure of its off-diagonal submatrices A^(i,j)
// ... solves a covering optimization problem to determine, for each nonzero
// in A^(i,j), whether to use row-based or column-based communication ...
// Process i retains the column-based portion and transfers the row-based
// portion to remote process j."  Steps P1-P4 of DESIGN.md:
//   P1 validate + split the owned rows into blocks by column owner,
//   P2 canonical minimum cover per block (cover.cpp), blocks in parallel,
//   P3 nonzero assignment (ROW if the row is selected, else COL; mirrored
//      under the col-max rule, R2),
//   P4 one-time exchange of (B-row list, C-row list, A_row) to the peer and
//      assembly of the per-iteration device operations.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstring>
#include <thread>

#include "shiro_internal.h"

namespace shiro {

namespace {

inline int owner_of(const int64_t *part, int P, int64_t id) {
  // largest p with part[p] <= id (part non-decreasing; empty blocks allowed)
  int lo = 0, hi = P;   // answer in [0, P)
  while (hi - lo > 1) {
    int mid = (lo + hi) / 2;
    if (part[mid] <= id) lo = mid; else hi = mid;
  }
  while (lo + 1 < P && part[lo + 1] <= id) ++lo;
  return lo;
}

template <typename F>
void parallel_for(int64_t n, F &&f) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  int64_t nt = std::min<int64_t>(n, hw);
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  std::atomic<int64_t> next{0};
  std::vector<Error> errs;
  std::mutex mu;
  for (int64_t t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (;;) {
        int64_t i = next.fetch_add(1);
        if (i >= n) break;
        try {
          f(i);
        } catch (const Error &e) {
          std::lock_guard<std::mutex> lk(mu);
          errs.push_back(e);
        }
      }
    });
  for (auto &x : th) x.join();
  if (!errs.empty()) throw errs.front();
}

struct MsgWriter {
  std::vector<int64_t> w;
  void put(int64_t x) { w.push_back(x); }
};

std::vector<char> to_bytes(const std::vector<int64_t> &w) {
  std::vector<char> b(w.size() * 8);
  if (!w.empty()) std::memcpy(b.data(), w.data(), b.size());
  return b;
}

}  // namespace

void validate_input(const PlanInput &in) {
  if (in.P < 1 || in.P > 64) throw Error(SHIRO_E_ARG, "nranks must be in 1..64");
  if (in.rank < 0 || in.rank >= in.P) throw Error(SHIRO_E_ARG, "rank out of range");
  if (in.g < 1 || in.P % in.g) throw Error(SHIRO_E_ARG, "group_size must divide nranks");
  if (in.N < 1 || in.N > 4096) throw Error(SHIRO_E_ARG, "N must be in 1..4096");
  if (in.n < 0 || in.n > 0x7fffffffLL) throw Error(SHIRO_E_ARG, "n must be in 0..2^31-1");
  if (!in.part) throw Error(SHIRO_E_ARG, "part is NULL");
  if (in.part[0] != 0 || in.part[in.P] != in.n)
    throw Error(SHIRO_E_PART, "part[0] must be 0 and part[P] must be n");
  for (int p = 0; p < in.P; ++p)
    if (in.part[p + 1] < in.part[p]) throw Error(SHIRO_E_PART, "part must be non-decreasing");
  const int64_t M = in.part[in.rank + 1] - in.part[in.rank];
  if (!in.row_ptr) throw Error(SHIRO_E_ARG, "row_ptr is NULL");
  if (in.row_ptr[0] != 0) throw Error(SHIRO_E_CSR, "row_ptr[0] must be 0");
  for (int64_t t = 0; t < M; ++t)
    if (in.row_ptr[t + 1] < in.row_ptr[t]) throw Error(SHIRO_E_CSR, "row_ptr not monotone");
  const int64_t nnz = in.row_ptr[M];
  if (nnz > 0 && (!in.col || !in.val)) throw Error(SHIRO_E_ARG, "col_idx/val is NULL");
  for (int64_t t = 0; t < M; ++t) {
    for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k) {
      const int64_t j = in.col[k];
      if (j < 0 || j >= in.n)
        throw Error(SHIRO_E_CSR, "column id out of range at local row " + std::to_string(t));
      if (k > in.row_ptr[t] && in.col[k - 1] >= j)
        throw Error(SHIRO_E_CSR, "columns not strictly increasing in local row " +
                                     std::to_string(t));
    }
  }
}

// -------------------------------------------------------------------------
// Phase 1 (owner side): covers of A^(r,q) for every q != r.
// -------------------------------------------------------------------------
Phase1 plan_phase1(const PlanInput &in) {
  const int P = in.P, r = in.rank;
  const int64_t lo = in.part[r], M = in.part[r + 1] - lo;
  const int64_t nnz = in.row_ptr[M];
  const bool colmax = in.flags & SHIRO_F_COVER_COLMAX;
  const bool mode_col = in.flags & SHIRO_F_MODE_COL;
  const bool mode_row = in.flags & SHIRO_F_MODE_ROW;
  const bool mode_block = in.flags & SHIRO_F_MODE_BLOCK;   // Eq. 1: whole B blocks
  Phase1 p1;
  p1.out.assign(P, {});
  p1.tag.assign(nnz, 0);
  p1.recv_b.assign(P, {});
  p1.recv_c.assign(P, {});
  p1.n_rows.assign(P, 0);
  p1.n_cols.assign(P, 0);
  p1.nnz_row.assign(P, 0);
  p1.ship_idx.assign(P, {});

  // owner of every nonzero's column; per-block nonzero index lists (CSR order)
  std::vector<int32_t> q_of(nnz);
  std::vector<int64_t> cnt(P + 1, 0);
  for (int64_t t = 0; t < M; ++t) {
    int q = 0;
    for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k) {
      const int64_t j = in.col[k];
      while (q + 1 < P && in.part[q + 1] <= j) ++q;   // columns ascending in a row
      q = (in.part[q] <= j && j < in.part[q + 1]) ? q : owner_of(in.part, P, j);
      q_of[k] = q;
      cnt[q + 1]++;
    }
  }
  for (int q = 0; q < P; ++q) cnt[q + 1] += cnt[q];
  std::vector<int64_t> idx(nnz), rowof(nnz), fill(cnt.begin(), cnt.end() - 1);
  for (int64_t t = 0; t < M; ++t)
    for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k) {
      idx[fill[q_of[k]]++] = k;
      rowof[k] = t;
    }

  std::vector<int> blocks;
  for (int q = 0; q < P; ++q)
    if (q != r && cnt[q + 1] > cnt[q]) blocks.push_back(q);

  parallel_for((int64_t)blocks.size(), [&](int64_t bi) {
    const int q = blocks[bi];
    const int64_t b0 = cnt[q], b1 = cnt[q + 1], ne = b1 - b0;
    const int64_t qlo = in.part[q], Kq = in.part[q + 1] - qlo;
    // rows: CSR order => local rows ascending; compress
    std::vector<int64_t> urow;          // local row ids t of Rows(A^(r,q))
    std::vector<int64_t> ap{0};
    std::vector<int32_t> adj(ne);
    std::vector<int32_t> cmap(Kq, -1);
    for (int64_t e = b0; e < b1; ++e) cmap[in.col[idx[e]] - qlo] = 0;
    std::vector<int64_t> ucol;          // global col ids of Cols(A^(r,q)), ascending
    for (int64_t x = 0; x < Kq; ++x)
      if (cmap[x] == 0) { cmap[x] = (int32_t)ucol.size(); ucol.push_back(qlo + x); }
    for (int64_t e = b0; e < b1; ++e) {
      const int64_t k = idx[e], t = rowof[k];
      if (urow.empty() || urow.back() != t) {
        if (!urow.empty()) ap.push_back(e - b0);
        urow.push_back(t);
      }
      adj[e - b0] = cmap[in.col[k] - qlo];
    }
    ap.push_back(ne);
    const int32_t nr = (int32_t)urow.size(), nc = (int32_t)ucol.size();
    std::vector<uint8_t> sel_r, sel_c;
    const bool joint = !mode_col && !mode_row && !mode_block;
    if (joint && in.w_row) {
      // weighted covers (Eqs. 4-8): vertex weights of the
      // block's rows (C rows of this rank) and columns (B rows of q)
      std::vector<int64_t> wr(nr), wc(nc);
      for (int32_t u = 0; u < nr; ++u) wr[u] = in.w_row[urow[u]];
      for (int32_t v = 0; v < nc; ++v) wc[v] = in.w_col[ucol[v]];
      block_cover_weighted(nr, nc, ap, adj, wr, wc, colmax, sel_r, sel_c);
    } else if (joint) {
      block_cover(nr, nc, ap, adj, colmax, sel_r, sel_c);
    }
    // SHIRO_F_COVER_BALANCE (R18): near-minimum all-rows cover -> all rows
    bool all_rows = false;
    if (joint && (in.flags & SHIRO_F_COVER_BALANCE)) {
      int64_t mu = 0;
      for (uint8_t x : sel_r) mu += x;
      for (uint8_t x : sel_c) mu += x;
      all_rows = nr <= mu + std::max<int64_t>(1, mu / 1000);
    }
    // assignment (P3)
    std::vector<uint8_t> row_used(nr, 0), col_used(nc, 0);
    int64_t nrow_nz = 0;
    for (int32_t u = 0; u < nr; ++u)
      for (int64_t e = ap[u]; e < ap[u + 1]; ++e) {
        const int32_t v = adj[e];
        bool is_row;
        if (mode_col || mode_block) is_row = false;
        else if (mode_row || all_rows) is_row = true;
        else if (!colmax) is_row = sel_r[u];
        else is_row = !sel_c[v];
        const int64_t k = idx[b0 + e];
        p1.tag[k] = is_row ? 1 : 2;
        if (is_row) { row_used[u] = 1; ++nrow_nz; }
        else col_used[v] = 1;
      }
    std::vector<int64_t> b_ids, c_ids;
    for (int32_t v = 0; v < nc; ++v)
      if (col_used[v] && !mode_block) b_ids.push_back(ucol[v]);
    if (mode_block)
      for (int64_t x = 0; x < Kq; ++x) b_ids.push_back(qlo + x);
    for (int32_t u = 0; u < nr; ++u)
      if (row_used[u]) c_ids.push_back(lo + urow[u]);
    if (joint && all_rows) {
      // balanced all-rows cover: every row carries its nonzeros, no column is sent
      for (int32_t u = 0; u < nr; ++u)
        if (!row_used[u]) throw Error(SHIRO_E_INTERNAL, "balanced cover: row unused");
      for (int32_t v = 0; v < nc; ++v)
        if (col_used[v]) throw Error(SHIRO_E_INTERNAL, "balanced cover: column used");
    } else if (joint) {
      // every selected vertex carries a private edge (minimality)
      for (int32_t u = 0; u < nr; ++u)
        if (sel_r[u] != row_used[u]) throw Error(SHIRO_E_INTERNAL, "selected row unused");
      for (int32_t v = 0; v < nc; ++v)
        if (sel_c[v] != col_used[v]) throw Error(SHIRO_E_INTERNAL, "selected col unused");
    }
    // message to q: header, b ids, c ids, per-c-row counts, A_row (col, val)
    MsgWriter m;
    m.put((int64_t)b_ids.size());
    m.put((int64_t)c_ids.size());
    m.put(nrow_nz);
    m.put(0);
    for (auto x : b_ids) m.put(x);
    for (auto x : c_ids) m.put(x);
    std::vector<int64_t> cols_w, vals_w, ship;
    for (int32_t u = 0; u < nr; ++u) {
      if (!row_used[u]) continue;
      int64_t c = 0;
      for (int64_t e = ap[u]; e < ap[u + 1]; ++e) {
        const int64_t k = idx[b0 + e];
        if (p1.tag[k] != 1) continue;
        ++c;
        ship.push_back(k);
        cols_w.push_back(in.col[k]);
        int32_t bits;
        std::memcpy(&bits, &in.val[k], 4);
        vals_w.push_back(bits);
      }
      m.put(c);
    }
    for (auto x : cols_w) m.put(x);
    for (auto x : vals_w) m.put(x);
    p1.out[q] = to_bytes(m.w);
    p1.recv_b[q] = std::move(b_ids);
    p1.recv_c[q] = std::move(c_ids);
    p1.n_rows[q] = nr;
    p1.n_cols[q] = nc;
    p1.nnz_row[q] = nrow_nz;
    p1.ship_idx[q] = std::move(ship);
  });
  // empty blocks still get an (empty) message so every peer can parse one
  for (int q = 0; q < P; ++q)
    if (q != r && p1.out[q].empty()) p1.out[q] = to_bytes({0, 0, 0, 0});
  return p1;
}

// -------------------------------------------------------------------------
// Phase 2: assemble lists, buffer layouts and the device operations.
// -------------------------------------------------------------------------
void plan_phase2(const PlanInput &in, Phase1 &p1, const std::vector<std::vector<char>> &in_msgs,
                 Plan &pl) {
  const int P = in.P, r = in.rank;
  const int64_t lo = in.part[r], M = in.part[r + 1] - lo;
  const int64_t nnz = in.row_ptr[M];
  const int N = in.N;
  pl.rank = r; pl.P = P; pl.g = in.g; pl.flags = in.flags; pl.n = in.n; pl.N = N;
  pl.part.assign(in.part, in.part + P + 1);
  pl.M = M;
  pl.send_b.assign(P, {}); pl.send_c.assign(P, {});
  pl.recv_b = std::move(p1.recv_b);
  pl.recv_c = std::move(p1.recv_c);

  // parse the incoming messages: what this rank sends to each peer p
  std::vector<std::vector<int64_t>> out_counts(P), out_cols(P);
  std::vector<std::vector<float>> out_vals(P);
  int64_t nnz_computed = 0;
  // value space of the refresh (N3): [local values || values received from
  // each peer, peers ascending, message order]
  pl.nnz_local = nnz;
  pl.ship_idx = std::move(p1.ship_idx);
  pl.recv_vals.assign(P, 0);
  std::vector<int64_t> vbase(P + 1, nnz);
  for (int p = 0; p < P; ++p) {
    if (p == r) continue;
    const auto &b = in_msgs[p];
    if (b.size() < 32 || b.size() % 8) throw Error(SHIRO_E_INTERNAL, "malformed plan message");
    const int64_t *w = reinterpret_cast<const int64_t *>(b.data());
    const int64_t nb = w[0], nc = w[1], nz = w[2];
    if ((int64_t)b.size() != 8 * (4 + nb + 2 * nc + 2 * nz))
      throw Error(SHIRO_E_INTERNAL, "plan message size mismatch");
    const int64_t *pb = w + 4, *pc = pb + nb, *pn = pc + nc, *pj = pn + nc, *pv = pj + nz;
    pl.send_b[p].assign(pb, pb + nb);
    pl.send_c[p].assign(pc, pc + nc);
    out_counts[p].assign(pn, pn + nc);
    out_cols[p].assign(pj, pj + nz);
    out_vals[p].resize(nz);
    for (int64_t k = 0; k < nz; ++k) {
      int32_t bits = (int32_t)pv[k];
      std::memcpy(&out_vals[p][k], &bits, 4);
    }
    for (auto x : pl.send_b[p])
      if (x < lo || x >= lo + M) throw Error(SHIRO_E_INTERNAL, "send_b id not owned");
    nnz_computed += nz;
    pl.recv_vals[p] = nz;
  }
  for (int p = 0; p < P; ++p) vbase[p + 1] = vbase[p] + pl.recv_vals[p];
  pl.nnz_recv_vals = nnz_computed;
  if (vbase[P] > 0x7fffffffLL) throw Error(SHIRO_E_ARG, "more than 2^31 values on one rank");

  // buffer layouts: per peer ascending, [B rows || C rows]
  pl.send_off.assign(P + 1, 0);
  pl.recv_off.assign(P + 1, 0);
  for (int p = 0; p < P; ++p) {
    pl.send_off[p + 1] = pl.send_off[p] + pl.send_b[p].size() + pl.send_c[p].size();
    pl.recv_off[p + 1] = pl.recv_off[p] + pl.recv_b[p].size() + pl.recv_c[p].size();
  }
  pl.send_rows = pl.send_off[P];
  pl.recv_rows = pl.recv_off[P];

  // K4 pack: send_buf[send_off[d] + k] = B_local[send_b[d][k] - lo]
  pl.pack_src.clear(); pl.pack_dst.clear();
  for (int d = 0; d < P; ++d)
    for (size_t k = 0; k < pl.send_b[d].size(); ++k) {
      pl.pack_src.push_back((int32_t)(pl.send_b[d][k] - lo));
      pl.pack_dst.push_back((int32_t)(pl.send_off[d] + k));
    }
  // K3 row-based partial SpMM: one CSR row per C row sent, output into send_buf
  HostCsr &ao = pl.A_out;
  ao = HostCsr();
  for (int d = 0; d < P; ++d) {
    int64_t pos = 0;
    for (size_t k = 0; k < pl.send_c[d].size(); ++k) {
      for (int64_t e = 0; e < out_counts[d][k]; ++e, ++pos) {
        ao.col.push_back((int32_t)(out_cols[d][pos] - lo));
        ao.val.push_back(out_vals[d][pos]);
        ao.vsrc.push_back((int32_t)(vbase[d] + pos));
      }
      ao.rp.push_back((int64_t)ao.col.size());
      ao.out_row.push_back((int32_t)(pl.send_off[d] + pl.send_b[d].size() + k));
    }
  }
  ao.nrows = (int64_t)ao.out_row.size();

  // K1 local SpMM on the diagonal block (all M rows, overwrite)
  HostCsr &ad = pl.A_diag;
  ad = HostCsr();
  ad.nrows = M;
  ad.rp.reserve(M + 1);
  int64_t n_local = 0, n_colb = 0, n_rowb = 0;
  for (int64_t t = 0; t < M; ++t) {
    for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k)
      if (p1.tag[k] == 0) {
        ad.col.push_back((int32_t)(in.col[k] - lo));
        ad.val.push_back(in.val[k]);
        ad.vsrc.push_back((int32_t)k);
      }
    ad.rp.push_back((int64_t)ad.col.size());
  }
  for (int64_t k = 0; k < nnz; ++k) {
    n_local += p1.tag[k] == 0;
    n_rowb += p1.tag[k] == 1;
    n_colb += p1.tag[k] == 2;
  }

  // K2 column-based remote SpMM over the receive buffer (compressed rows)
  std::vector<int64_t> owner_start(P + 1);
  for (int q = 0; q <= P; ++q) owner_start[q] = in.part[q];
  HostCsr &ac = pl.A_col;
  ac = HostCsr();
  std::vector<std::vector<int32_t>> colrow_cols(M);   // per local row: recv indices
  std::vector<std::vector<float>> colrow_vals(M);
  std::vector<std::vector<int32_t>> colrow_k(M);
  for (int64_t t = 0; t < M; ++t) {
    int q = 0;
    for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k) {
      if (p1.tag[k] != 2) continue;
      const int64_t j = in.col[k];
      while (q + 1 < P && in.part[q + 1] <= j) ++q;
      const auto &lb = pl.recv_b[q];
      auto itj = std::lower_bound(lb.begin(), lb.end(), j);
      if (itj == lb.end() || *itj != j) throw Error(SHIRO_E_INTERNAL, "col-based B row missing");
      colrow_cols[t].push_back((int32_t)(pl.recv_off[q] + (itj - lb.begin())));
      colrow_vals[t].push_back(in.val[k]);
      colrow_k[t].push_back((int32_t)k);
    }
    if (!colrow_cols[t].empty()) {
      ac.col.insert(ac.col.end(), colrow_cols[t].begin(), colrow_cols[t].end());
      ac.val.insert(ac.val.end(), colrow_vals[t].begin(), colrow_vals[t].end());
      ac.vsrc.insert(ac.vsrc.end(), colrow_k[t].begin(), colrow_k[t].end());
      ac.rp.push_back((int64_t)ac.col.size());
      ac.out_row.push_back((int32_t)t);
    }
  }
  ac.nrows = (int64_t)ac.out_row.size();

  // K5 scatter-add: per target row, its partial rows in the receive buffer
  // (sources ascending -> fixed summation order)
  std::vector<std::vector<int32_t>> part_src(M);
  for (int s = 0; s < P; ++s) {
    const int64_t base = pl.recv_off[s] + (int64_t)pl.recv_b[s].size();
    for (size_t k = 0; k < pl.recv_c[s].size(); ++k) {
      const int64_t t = pl.recv_c[s][k] - lo;
      if (t < 0 || t >= M) throw Error(SHIRO_E_INTERNAL, "recv_c id not owned");
      part_src[t].push_back((int32_t)(base + k));
    }
  }
  pl.sc_tgt.clear(); pl.sc_src.clear(); pl.sc_ptr.assign(1, 0);
  for (int64_t t = 0; t < M; ++t) {
    if (part_src[t].empty()) continue;
    pl.sc_tgt.push_back((int32_t)t);
    pl.sc_src.insert(pl.sc_src.end(), part_src[t].begin(), part_src[t].end());
    pl.sc_ptr.push_back((int64_t)pl.sc_src.size());
  }
  // fused K2+K5: per row, col-based entries then partials (weight 1)
  HostCsr &ar = pl.A_rem;
  ar = HostCsr();
  for (int64_t t = 0; t < M; ++t) {
    if (colrow_cols[t].empty() && part_src[t].empty()) continue;
    ar.col.insert(ar.col.end(), colrow_cols[t].begin(), colrow_cols[t].end());
    ar.val.insert(ar.val.end(), colrow_vals[t].begin(), colrow_vals[t].end());
    ar.vsrc.insert(ar.vsrc.end(), colrow_k[t].begin(), colrow_k[t].end());
    for (auto x : part_src[t]) { ar.col.push_back(x); ar.val.push_back(1.0f); ar.vsrc.push_back(-1); }
    ar.rp.push_back((int64_t)ar.col.size());
    ar.out_row.push_back((int32_t)t);
  }
  ar.nrows = (int64_t)ar.out_row.size();
  ar.src_bounds = pl.recv_off;     // receive-buffer segment of each source (per-unit waits)
  ad.hot_rows = M;                 // local rows read B_local (hot/cold L2 marks)
  ao.hot_rows = M;

  // local statistics
  shiro_info_t &I = pl.info;
  I.rank = r; I.nranks = P; I.group_size = in.g; I.N = N;
  I.n = in.n; I.m_local = M; I.nnz_local = nnz;
  I.nnz_diag = n_local; I.nnz_colbased = n_colb; I.nnz_rowbased_shipped = n_rowb;
  I.nnz_rowbased_computed = nnz_computed;
  for (int p = 0; p < P; ++p) {
    I.send_b_rows += pl.send_b[p].size();
    I.send_c_rows += pl.send_c[p].size();
    I.recv_b_rows += pl.recv_b[p].size();
    I.recv_c_rows += pl.recv_c[p].size();
  }
}

// -------------------------------------------------------------------------
// Global statistics: each rank contributes its share, summed over ranks.
// -------------------------------------------------------------------------
void plan_stats(const PlanInput &in, Plan &pl, const Alltoallv &xchg) {
  const int P = pl.P, r = pl.rank, g = pl.g;
  auto grp = [g](int x) { return x / g; };
  // these per-block numbers were consumed in phase 1; recompute from lists
  std::vector<int64_t> v(12, 0);
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const int64_t mu = pl.recv_b[q].size() + pl.recv_c[q].size();
    v[0] += mu;                                            // joint (as receiver)
    if (grp(q) != grp(r)) v[5] += mu;                      // flat inter
  }
  // hierarchical shares (hierarchical accounting)
  const int ngrp = P / g;
  for (int G = 0; G < ngrp; ++G) {
    if (G == grp(r)) continue;
    std::vector<int64_t> U, V;
    for (int p = G * g; p < G * g + g; ++p) {
      U.insert(U.end(), pl.send_b[p].begin(), pl.send_b[p].end());
      V.insert(V.end(), pl.recv_c[p].begin(), pl.recv_c[p].end());
    }
    std::sort(U.begin(), U.end());
    U.erase(std::unique(U.begin(), U.end()), U.end());
    std::sort(V.begin(), V.end());
    V.erase(std::unique(V.begin(), V.end()), V.end());
    v[6] += (int64_t)U.size() + (int64_t)V.size();         // col inter (sender) + row inter (receiver)
  }
  for (int p = 0; p < P; ++p) {
    if (p == r) continue;
    if (grp(p) == grp(r)) {
      v[7] += pl.send_b[p].size() + pl.send_c[p].size();   // same-group direct
    } else {
      const int rep_row = grp(r) * g + (p % g);
      if (rep_row != r) v[7] += pl.send_c[p].size();       // stage I row intra
      const int rep_col = grp(r) * g + (p % g);             // p plays the source q here
      if (rep_col != r) v[7] += pl.recv_b[p].size();       // stage II col intra (receiver)
    }
  }
  v[1] = pl.loc_cols;
  v[2] = pl.loc_rows;
  v[3] = pl.loc_block;
  v[4] = pl.loc_setup;
  v[8] = pl.send_rows;
  v[9] = pl.recv_rows;
  std::vector<std::vector<char>> send(P), recv(P);
  std::vector<char> mine(v.size() * 8);
  std::memcpy(mine.data(), v.data(), mine.size());
  for (int p = 0; p < P; ++p) send[p] = mine;
  xchg(send, recv);
  recv[r] = mine;
  shiro_info_t &I = pl.info;
  I.g_joint_rows = I.g_col_rows = I.g_row_rows = I.g_block_rows = I.g_setup_bytes = 0;
  I.g_flat_inter_rows = I.g_hier_inter_rows = I.g_hier_intra_rows = 0;
  I.g_max_send_rows = I.g_max_recv_rows = 0;
  for (int p = 0; p < P; ++p) {
    if (recv[p].size() != v.size() * 8) throw Error(SHIRO_E_INTERNAL, "stats message size");
    const int64_t *w = reinterpret_cast<const int64_t *>(recv[p].data());
    I.g_joint_rows += w[0];
    I.g_col_rows += w[1];
    I.g_row_rows += w[2];
    I.g_block_rows += w[3];
    I.g_setup_bytes += w[4];
    I.g_flat_inter_rows += w[5];
    I.g_hier_inter_rows += w[6];
    I.g_hier_intra_rows += w[7];
    I.g_max_send_rows = std::max(I.g_max_send_rows, w[8]);
    I.g_max_recv_rows = std::max(I.g_max_recv_rows, w[9]);
  }
  I.g_oblivious_rows = (int64_t)(P - 1) * pl.n;
  if (g == 1) { I.g_hier_inter_rows = I.g_flat_inter_rows; I.g_hier_intra_rows = 0; }
  (void)in;
}

}  // namespace shiro

namespace shiro {

// ---------------------------------------------------------------------------
// Transposed SpMM (GNN backward C = A^T G): with
// SHIRO_F_TRANSPOSE every rank passes its rows of A as usual; the entries are
// redistributed once (entry (i, j) goes to the owner of j as (j, i)) and the
// planner builds the joint plan of A^T, whose row blocks use the same
// partition.  The transposed rows are sorted by column, so A^T is a valid CSR.
// ---------------------------------------------------------------------------
std::vector<std::vector<char>> transpose_messages(const PlanInput &in) {
  const int P = in.P;
  const int64_t lo = in.part[in.rank], M = in.part[in.rank + 1] - lo;
  std::vector<std::vector<int64_t>> w(P);
  for (int64_t t = 0; t < M; ++t)
    for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k) {
      const int64_t j = in.col[k];
      int q = 0;
      while (in.part[q + 1] <= j) ++q;
      int32_t bits;
      std::memcpy(&bits, &in.val[k], 4);
      w[q].push_back(j);
      w[q].push_back(lo + t);
      w[q].push_back(bits);
    }
  std::vector<std::vector<char>> out(P);
  for (int q = 0; q < P; ++q) out[q] = to_bytes(w[q]);
  return out;
}

void transpose_assemble(const PlanInput &in, const std::vector<std::vector<char>> &msgs,
                        std::vector<int64_t> &rp, std::vector<int32_t> &col,
                        std::vector<float> &val, std::vector<int64_t> *perm) {
  const int64_t lo = in.part[in.rank], M = in.part[in.rank + 1] - lo;
  struct Ent { int32_t i; float v; int64_t src; };   // src: index over the messages in order
  std::vector<std::vector<Ent>> rows(M);
  int64_t gidx = 0;
  for (const auto &b : msgs) {
    const int64_t *w = reinterpret_cast<const int64_t *>(b.data());
    const int64_t n3 = (int64_t)b.size() / 24;
    for (int64_t e = 0; e < n3; ++e, ++gidx) {
      const int64_t j = w[3 * e], i = w[3 * e + 1];
      const int32_t bits = (int32_t)w[3 * e + 2];
      float v;
      std::memcpy(&v, &bits, 4);
      if (j < lo || j >= lo + M) throw Error(SHIRO_E_INTERNAL, "transpose: misrouted entry");
      rows[j - lo].push_back({(int32_t)i, v, gidx});
    }
  }
  rp.assign(1, 0);
  col.clear();
  val.clear();
  if (perm) perm->clear();
  for (int64_t t = 0; t < M; ++t) {
    std::sort(rows[t].begin(), rows[t].end(),
              [](const Ent &a, const Ent &b) { return a.i < b.i; });
    for (auto &e : rows[t]) {
      col.push_back(e.i);
      val.push_back(e.v);
      if (perm) perm->push_back(e.src);
    }
    rp.push_back((int64_t)col.size());
  }
}

// ---------------------------------------------------------------------------
// Value refresh (the plan is "reused across
// multiple SpMM operations with the same sparsity pattern"): the cover, lists
// and device layouts stay; only values move.  Each rank ships the new values
// of its row-based nonzeros to the column owner in the plan-time message
// order (one all-to-allv of 4 B per row-based nonzero), and assembles
// V = [own values || received values, peers ascending].  Transposed plans
// first redistribute the values exactly as the plan-time transpose did.
// ---------------------------------------------------------------------------
std::vector<std::vector<char>> refresh_ship(const Plan &pl, const float *lv) {
  std::vector<std::vector<char>> snd(pl.P);
  for (int q = 0; q < pl.P; ++q) {
    if (q == pl.rank) continue;
    const auto &ix = pl.ship_idx[q];
    snd[q].resize(ix.size() * 4);
    float *f = reinterpret_cast<float *>(snd[q].data());
    for (size_t e = 0; e < ix.size(); ++e) f[e] = lv[ix[e]];
  }
  return snd;
}

std::vector<float> refresh_assemble(const Plan &pl, const float *lv,
                                    const std::vector<std::vector<char>> &rcv) {
  std::vector<float> V;
  V.reserve(pl.nnz_local + pl.nnz_recv_vals);
  V.insert(V.end(), lv, lv + pl.nnz_local);
  for (int p = 0; p < pl.P; ++p) {
    if (p == pl.rank) continue;
    if ((int64_t)rcv[p].size() != 4 * pl.recv_vals[p])
      throw Error(SHIRO_E_INTERNAL, "refresh: value message size mismatch");
    const float *f = reinterpret_cast<const float *>(rcv[p].data());
    V.insert(V.end(), f, f + pl.recv_vals[p]);
  }
  return V;
}

std::vector<float> refresh_value_space(Plan &pl, const PlanInput &in, const float *val,
                                       const Alltoallv &xchg) {
  const int P = pl.P, r = pl.rank;
  std::vector<float> local;
  const float *lv = val;
  if (pl.flags & SHIRO_F_TRANSPOSE) {
    // the entries of this rank's rows of A, in transpose_messages order, to
    // the owner of each column; the receiver places them with tperm
    const int64_t lo = in.part[r], M = in.part[r + 1] - lo;
    std::vector<std::vector<char>> snd(P), rcv;
    std::vector<std::vector<float>> w(P);
    for (int64_t t = 0; t < M; ++t)
      for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k) {
        int q = 0;
        while (in.part[q + 1] <= in.col[k]) ++q;
        w[q].push_back(val[k]);
      }
    for (int q = 0; q < P; ++q) {
      snd[q].resize(w[q].size() * 4);
      if (!w[q].empty()) std::memcpy(snd[q].data(), w[q].data(), snd[q].size());
    }
    if (P > 1) xchg(snd, rcv);
    rcv.resize(P);
    rcv[r] = snd[r];
    std::vector<float> cat;
    for (int q = 0; q < P; ++q) {
      const float *f = reinterpret_cast<const float *>(rcv[q].data());
      cat.insert(cat.end(), f, f + rcv[q].size() / 4);
    }
    if ((int64_t)pl.tperm.size() != pl.nnz_local)
      throw Error(SHIRO_E_INTERNAL, "refresh: transposed value count mismatch");
    local.resize(pl.nnz_local);
    for (int64_t x = 0; x < pl.nnz_local; ++x) {
      if (pl.tperm[x] < 0 || pl.tperm[x] >= (int64_t)cat.size())
        throw Error(SHIRO_E_INTERNAL, "refresh: transposed index out of range");
      local[x] = cat[pl.tperm[x]];
    }
    lv = local.data();
  }
  std::vector<std::vector<char>> snd = refresh_ship(pl, lv), rcv;
  if (P > 1) xchg(snd, rcv);
  rcv.resize(P);
  return refresh_assemble(pl, lv, rcv);
}

}  // namespace shiro
