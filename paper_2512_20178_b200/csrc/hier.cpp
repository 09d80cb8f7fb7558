// hier.cpp -- hierarchical (two-stage) routing of the joint plan.
//
// PAPER.md section VI: the joint plan is separated into column-based (B
// rows) and row-based (partial C rows) traffic (L509-510).  Column traffic
// uses the three-step method "source group aggregation, inter-group transfer,
// intra-group distribution" (L516-517); row traffic uses "intra-group
// pre-aggregation of partial results, and inter-group transmission of
// aggregated data" (L519).  The two are scheduled as Algorithm 1 (L542-574,
// reading R13): Stage I = column inter-group fetch || row intra-group
// aggregation; Stage II = row inter-group transmission || column intra-group
// distribution.  Representatives (reading R12): B rows of owner q for group G
// go to the member of G with rank = q (mod g); partial C rows for destination
// p are aggregated by the member of the source group with rank = p (mod g).
// Same-group traffic goes directly in Stage I.
//
// Buffers of rank r (rows of N floats): R1 (Stage I receive) and R2 (Stage II
// receive), one segment per source rank, each segment = [B rows ascending ||
// C blocks by final destination ascending].  R1's segment from r itself holds
// r's own partials that r aggregates.  The final remote SpMM reads the
// concatenation [R1 || R2].
#include <algorithm>
#include <cstring>
#include <map>

#include "shiro_internal.h"

namespace shiro {

namespace {

std::vector<int64_t> sorted_union(const std::vector<const std::vector<int64_t> *> &parts) {
  std::vector<int64_t> u;
  for (auto *p : parts) u.insert(u.end(), p->begin(), p->end());
  std::sort(u.begin(), u.end());
  u.erase(std::unique(u.begin(), u.end()), u.end());
  return u;
}

int64_t index_of(const std::vector<int64_t> &v, int64_t x) {
  auto it = std::lower_bound(v.begin(), v.end(), x);
  if (it == v.end() || *it != x) throw Error(SHIRO_E_INTERNAL, "hierarchical plan: id not found");
  return it - v.begin();
}

void put_list(std::vector<int64_t> &w, int64_t tag, int64_t p, const std::vector<int64_t> &ids) {
  w.push_back(tag);
  w.push_back(p);
  w.push_back((int64_t)ids.size());
  w.insert(w.end(), ids.begin(), ids.end());
}

}  // namespace

// Round A messages: the lists a representative needs from its sources.
//   tag 1 (to rep_col(r, G) for every other group G): send_b[r][p] for p in G
//   tag 2 (to same-group member a): send_c[r][p] for p outside the group
//         with p = a (mod g) (a aggregates them)
std::vector<std::vector<char>> hier_meta_messages(const Plan &pl) {
  const int P = pl.P, g = pl.g, me = pl.rank, G0 = me / g;
  std::vector<std::vector<char>> out(P);
  for (int d = 0; d < P; ++d) {
    if (d == me) continue;
    std::vector<int64_t> w;
    const int Gd = d / g;
    if (Gd != G0 && d == Gd * g + me % g)
      for (int p = Gd * g; p < Gd * g + g; ++p) put_list(w, 1, p, pl.send_b[p]);
    if (Gd == G0)
      for (int p = 0; p < P; ++p)
        if (p / g != G0 && p % g == d % g) put_list(w, 2, p, pl.send_c[p]);
    out[d].resize(w.size() * 8);
    if (!w.empty()) std::memcpy(out[d].data(), w.data(), out[d].size());
  }
  return out;
}

void hier_build(const PlanInput &in, const Phase1 &p1, Plan &pl,
                const std::vector<std::vector<char>> &meta) {
  const int P = pl.P, g = pl.g, me = pl.rank, G0 = me / g;
  const int64_t lo = pl.part[me], M = pl.M;
  Route &R = pl.route;
  R = Route();
  R.active = true;
  auto grp = [g](int x) { return x / g; };
  auto in_g0 = [&](int x) { return grp(x) == G0; };
  // ---- decode round-A lists -------------------------------------------------
  // fwd[q][p] = send_b[q][p] (q outside, q = me mod g, p in G0)
  // agg[m][p] = send_c[m][p] (m in G0, p outside, p = me mod g)
  std::map<std::pair<int, int>, std::vector<int64_t>> fwd, agg;
  for (int s = 0; s < P; ++s) {
    if (s == me) continue;
    const auto &b = meta[s];
    const int64_t *w = reinterpret_cast<const int64_t *>(b.data());
    const int64_t nw = (int64_t)b.size() / 8;
    for (int64_t i = 0; i < nw;) {
      const int64_t tag = w[i], p = w[i + 1], n = w[i + 2];
      std::vector<int64_t> ids(w + i + 3, w + i + 3 + n);
      if (tag == 1) fwd[{s, (int)p}] = std::move(ids);
      else agg[{s, (int)p}] = std::move(ids);
      i += 3 + n;
    }
  }
  for (int p = 0; p < P; ++p)
    if (!in_g0(p) && p % g == me % g) agg[{me, p}] = pl.send_c[p];
  auto aggl = [&](int m, int p) -> const std::vector<int64_t> & {
    static const std::vector<int64_t> empty;
    auto it = agg.find({m, p});
    return it == agg.end() ? empty : it->second;
  };
  auto fwdl = [&](int q, int p) -> const std::vector<int64_t> & {
    static const std::vector<int64_t> empty;
    auto it = fwd.find({q, p});
    return it == fwd.end() ? empty : it->second;
  };
  // destinations outside G0 that member a aggregates for: p = a (mod g)
  auto agg_dests = [&](int a) {
    std::vector<int> v;
    for (int p = 0; p < P; ++p)
      if (!in_g0(p) && p % g == a % g) v.push_back(p);
    return v;
  };
  // U(q, G0) for q outside G0 with q = me (mod g)
  std::map<int, std::vector<int64_t>> U;
  for (int q = 0; q < P; ++q)
    if (!in_g0(q) && q % g == me % g) {
      std::vector<const std::vector<int64_t> *> parts;
      for (int p = G0 * g; p < G0 * g + g; ++p) parts.push_back(&fwdl(q, p));
      U[q] = sorted_union(parts);
    }
  // V(G, me) for every other group G (aggregated by G*g + me%g)
  std::map<int, std::vector<int64_t>> Vin;
  for (int G = 0; G < P / g; ++G) {
    if (G == G0) continue;
    std::vector<const std::vector<int64_t> *> parts;
    for (int m = G * g; m < G * g + g; ++m) parts.push_back(&pl.recv_c[m]);
    Vin[G * g + me % g] = sorted_union(parts);
  }
  // ---- R1 layout: segment per source --------------------------------------
  // seg content and row offsets, in list format (B ids, then C blocks by final)
  R.h_send[0].assign(P, {}); R.h_send[1].assign(P, {});
  R.h_recv[0].assign(P, {}); R.h_recv[1].assign(P, {});
  R.r1_off.assign(P + 1, 0);
  R.r2_off.assign(P + 1, 0);
  // position maps inside my R1 for the consumers
  std::map<int, int64_t> r1_b_base;                       // B part of seg(s)
  std::map<std::pair<int, int>, int64_t> r1_c_base;       // C block (s, final) start
  for (int s = 0; s < P; ++s) {
    R.r1_off[s + 1] = R.r1_off[s];
    std::vector<int64_t> &L = R.h_recv[0][s];
    int64_t pos = 0;
    auto add_c = [&](int fin, const std::vector<int64_t> &ids) {
      r1_c_base[{s, fin}] = R.r1_off[s] + pos;
      L.insert(L.end(), ids.begin(), ids.end());
      pos += (int64_t)ids.size();
    };
    if (s == me) {
      for (int p : agg_dests(me)) add_c(p, aggl(me, p));
    } else if (in_g0(s)) {
      r1_b_base[s] = R.r1_off[s];
      L = pl.recv_b[s];
      pos = (int64_t)L.size();
      std::vector<int> fins = agg_dests(me);
      fins.push_back(me);
      std::sort(fins.begin(), fins.end());
      for (int f : fins) add_c(f, f == me ? pl.recv_c[s] : aggl(s, f));
    } else if (s % g == me % g) {
      r1_b_base[s] = R.r1_off[s];
      L = U[s];
      pos = (int64_t)L.size();
    }
    R.r1_off[s + 1] = R.r1_off[s] + pos;
  }
  if (!R.h_recv[0][me].empty()) R.h_recv[0][me].clear();   // self segment is not "received"
  R.r1_rows = R.r1_off[P];
  // ---- R2 layout -------------------------------------------------------------
  std::map<std::pair<int, int>, int64_t> r2_fwd_base;     // (s, q) -> start of recv_b[q] from s
  std::map<int, int64_t> r2_agg_base;                     // s -> start of V from s
  for (int s = 0; s < P; ++s) {
    R.r2_off[s + 1] = R.r2_off[s];
    if (s == me) continue;
    std::vector<int64_t> &L = R.h_recv[1][s];
    int64_t pos = 0;
    if (in_g0(s)) {
      for (int q = 0; q < P; ++q)
        if (!in_g0(q) && q % g == s % g) {
          r2_fwd_base[{s, q}] = R.r2_off[s] + pos;
          L.insert(L.end(), pl.recv_b[q].begin(), pl.recv_b[q].end());
          pos += (int64_t)pl.recv_b[q].size();
        }
    } else if (s % g == me % g) {
      r2_agg_base[s] = R.r2_off[s];
      L = Vin[s];
      pos = (int64_t)L.size();
    }
    R.r2_off[s + 1] = R.r2_off[s] + pos;
  }
  R.r2_rows = R.r2_off[P];
  // ---- Stage I producers ------------------------------------------------------
  // lists in the sender's view (what I write into d's R1 seg(me))
  for (int d = 0; d < P; ++d) {
    if (d == me) continue;
    std::vector<int64_t> &L = R.h_send[0][d];
    if (in_g0(d)) {
      L = pl.send_b[d];
      // C blocks by final ascending: d itself and the outside p = d (mod g)
      std::vector<int> fins = agg_dests(d);
      fins.push_back(d);
      std::sort(fins.begin(), fins.end());
      for (int f : fins) L.insert(L.end(), pl.send_c[f].begin(), pl.send_c[f].end());
    } else if (d == grp(d) * g + me % g) {
      std::vector<const std::vector<int64_t> *> parts;
      for (int p = grp(d) * g; p < grp(d) * g + g; ++p) parts.push_back(&pl.send_b[p]);
      L = sorted_union(parts);
    }
  }
  // pack rows (B_local -> peer R1 seg(me), B part at pos k)
  for (int d = 0; d < P; ++d) {
    if (d == me) continue;
    std::vector<int64_t> bl;
    if (in_g0(d)) bl = pl.send_b[d];
    else if (d == grp(d) * g + me % g) bl = R.h_send[0][d];
    for (size_t k = 0; k < bl.size(); ++k) {
      R.s1_pack_src.push_back((int32_t)(bl[k] - lo));
      R.s1_pack_dst.push_back(Dest{d, 0, (int64_t)k});
    }
  }
  // partial rows: A_out rows of destination p (pl.A_out is in p-ascending
  // order, k ascending), routed to p (same group) or to the aggregator
  {
    int64_t row = 0;
    for (int p = 0; p < P; ++p) {
      for (size_t k = 0; k < pl.send_c[p].size(); ++k, ++row) {
        Dest dst{};
        if (p == me) throw Error(SHIRO_E_INTERNAL, "partial to self");
        if (in_g0(p)) {
          // p's R1 seg(me): after B rows, C blocks by final ascending; block p
          int64_t pos = (int64_t)pl.send_b[p].size();
          std::vector<int> fins = agg_dests(p);
          fins.push_back(p);
          std::sort(fins.begin(), fins.end());
          for (int f : fins) {
            if (f == p) break;
            pos += (int64_t)pl.send_c[f].size();
          }
          dst = Dest{p, 0, pos + (int64_t)k};
        } else {
          const int a = G0 * g + p % g;
          int64_t pos = 0;
          if (a == me) {
            // own R1 self segment: blocks by p ascending
            for (int f : agg_dests(me)) {
              if (f == p) break;
              pos += (int64_t)pl.send_c[f].size();
            }
            dst = Dest{me, 0, pos + (int64_t)k};
          } else {
            pos = (int64_t)pl.send_b[a].size();
            std::vector<int> fins = agg_dests(a);
            fins.push_back(a);
            std::sort(fins.begin(), fins.end());
            for (int f : fins) {
              if (f == p) break;
              pos += (int64_t)pl.send_c[f].size();
            }
            dst = Dest{a, 0, pos + (int64_t)k};
          }
        }
        R.s1_part_dst.push_back(dst);
      }
    }
    if (row != pl.A_out.nrows) throw Error(SHIRO_E_INTERNAL, "A_out row count mismatch");
    R.s1_part = pl.A_out;      // same CSR (cols local B), destinations differ
  }
  // ---- Stage II producers --------------------------------------------------------
  for (int d = 0; d < P; ++d) {
    if (d == me) continue;
    std::vector<int64_t> &L = R.h_send[1][d];
    if (in_g0(d)) {
      for (int q = 0; q < P; ++q)
        if (!in_g0(q) && q % g == me % g) {
          const auto &ids = fwdl(q, d);
          for (size_t k = 0; k < ids.size(); ++k) {
            R.s2_fwd_src.push_back((int32_t)(r1_b_base[q] + index_of(U[q], ids[k])));
            R.s2_fwd_dst.push_back(Dest{d, 1, (int64_t)L.size()});
            L.push_back(ids[k]);
          }
        }
    } else if (d % g == me % g) {
      // aggregated partials V(G0, d): unit-weight SpMM over my R1
      std::vector<const std::vector<int64_t> *> parts;
      for (int m = G0 * g; m < G0 * g + g; ++m) parts.push_back(&aggl(m, d));
      const std::vector<int64_t> V = sorted_union(parts);
      for (size_t k = 0; k < V.size(); ++k) {
        for (int m = G0 * g; m < G0 * g + g; ++m) {   // member order ascending
          const auto &ml = aggl(m, d);
          auto it = std::lower_bound(ml.begin(), ml.end(), V[k]);
          if (it == ml.end() || *it != V[k]) continue;
          R.s2_agg.col.push_back((int32_t)(r1_c_base.at({m, d}) + (it - ml.begin())));
          R.s2_agg.val.push_back(1.0f);
        }
        R.s2_agg.rp.push_back((int64_t)R.s2_agg.col.size());
        R.s2_agg_dst.push_back(Dest{d, 1, (int64_t)k});
        L.push_back(V[k]);
      }
    }
  }
  R.s2_agg.nrows = (int64_t)R.s2_agg_dst.size();
  // identity out_row: bounds row groups to 2*LPR rows (per-row output pointers)
  for (int64_t t = 0; t < R.s2_agg.nrows; ++t) R.s2_agg.out_row.push_back((int32_t)t);
  // ---- final remote SpMM over [R1 || R2] ------------------------------------------
  // COL entries by B-row location, then unit-weight partials
  struct FinEnt { int32_t pos; float v; int32_t k; };   // k: value-space index (-1 = unit)
  std::vector<std::vector<FinEnt>> rows(M);
  for (int64_t t = 0; t < M; ++t) {
    for (int64_t k = in.row_ptr[t]; k < in.row_ptr[t + 1]; ++k) {
      if (p1.tag[k] != 2) continue;
      const int64_t j = in.col[k];
      int q = 0;
      while (pl.part[q + 1] <= j) ++q;
      int64_t pos;
      if (in_g0(q)) pos = r1_b_base.at(q) + index_of(pl.recv_b[q], j);
      else if (q % g == me % g) pos = r1_b_base.at(q) + index_of(U[q], j);
      else {
        const int s = G0 * g + q % g;
        pos = R.r1_rows + r2_fwd_base.at({s, q}) + index_of(pl.recv_b[q], j);
      }
      rows[t].push_back({(int32_t)pos, in.val[k], (int32_t)k});
    }
  }
  for (int s = 0; s < P; ++s) {
    if (s == me) continue;
    if (in_g0(s)) {
      const int64_t base = r1_c_base.at({s, me});
      for (size_t k = 0; k < pl.recv_c[s].size(); ++k)
        rows[pl.recv_c[s][k] - lo].push_back({(int32_t)(base + k), 1.0f, -1});
    } else if (s % g == me % g) {
      const auto &V = Vin[s];
      for (size_t k = 0; k < V.size(); ++k)
        rows[V[k] - lo].push_back({(int32_t)(R.r1_rows + r2_agg_base.at(s) + k), 1.0f, -1});
    }
  }
  for (int64_t t = 0; t < M; ++t) {
    if (rows[t].empty()) continue;
    for (auto &e : rows[t]) {
      R.fin.col.push_back(e.pos);
      R.fin.val.push_back(e.v);
      R.fin.vsrc.push_back(e.k);
    }
    R.fin.rp.push_back((int64_t)R.fin.col.size());
    R.fin.out_row.push_back((int32_t)t);
  }
  R.fin.nrows = (int64_t)R.fin.out_row.size();
}

}  // namespace shiro
