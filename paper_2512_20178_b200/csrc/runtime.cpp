// runtime.cpp -- device upload, executor, transports and the C ABI.
//
// Per-iteration flow of the flat joint plan (workflow
// steps 3-5; DESIGN.md rows E1-E6), on the caller's stream s0 and an internal
// communication stream s1:
//   s0: K4 pack B rows -> send_buf      (E1, "prepares required B rows")
//   s0: K3 A_out * B   -> send_buf      (E2, "computes partial C results")
//   s0: record ev_packed
//   s1: wait ev_packed; NCCL grouped send/recv per peer (E3, all-to-allv)
//   s0: K1 C = A_diag * B               (E4, overlapped with E3)
//   s0: wait ev_recvd
//   s0: K2 C += A_col * recv_B          (E5)
//   s0: K5 C += sum of recv partials     (E6)   [default: K2+K5 in one pass; SHIRO_F_SPLIT_RECV: two launches]
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>

#include "shiro_internal.h"

namespace shiro {

Plan::~Plan() {
  if (!loopback_view) {
    for (auto &g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    p2p_release(*this);
    hier_release(*this);
    if (comm) ncclCommDestroy(comm);
    if (ev_packed) cudaEventDestroy(ev_packed);
    if (ev_recvd) cudaEventDestroy(ev_recvd);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (arena) cudaFree(arena);
    if (stage) cudaFree(stage);
    if (stage2) cudaFree(stage2);
    if (vspace) cudaFree(vspace);
    if (merged_ops) cudaFree(merged_ops);
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t e : {ev_in[k], ev_comp[k], ev_out[k]})
        if (e) cudaEventDestroy(e);
    if (h2d_s) cudaStreamDestroy(h2d_s);
    if (d2h_s) cudaStreamDestroy(d2h_s);
    for (auto &e : prof)
      if (e) cudaEventDestroy(e);
  }
}

namespace {

// ---------------------------------------------------------------- arena
struct Arena {
  struct Item { size_t off; const void *src; size_t bytes; };
  std::vector<Item> items;
  size_t total = 0;
  size_t reserve(size_t bytes, const void *src = nullptr) {
    size_t off = (total + 255) & ~size_t(255);
    total = off + bytes;
    items.push_back({off, src, bytes});
    return off;
  }
};

template <typename T>
size_t put(Arena &ar, const std::vector<T> &v) {
  return ar.reserve(v.size() * sizeof(T), v.empty() ? nullptr : v.data());
}

// Work decomposition of one SpMM op (plan time).  Rows with more than L
// nonzeros (power-law hubs) become chunk tasks of L nonzeros; every other row
// belongs to a row group: a run of consecutive short rows with at most L
// nonzeros and kMaxGroupRows rows (2*LPR when an out_row map is used),
// streamed by one lane group; a per-nonzero byte holds the row offset inside
// the group.
// Unit size L: 256 nonzeros for large ops; smaller ops use smaller units so
// that the launch still has ~W waves of one-warp CTAs (32 per SM).  A lane
// group walks its unit serially, ~1 memory round trip per U = 4 gathers, so
// when an op fits in about one wave its time is the longest unit's chain of
// round trips: small ops (the remote SpMM and the per-rank producers of c2 at
// P >= 2) need short units.  L = nnz / (SMs * 32 * W), W = 4 (SHIRO_WAVES),
// rounded down to a multiple of 8, clamped to [8, 256] (SHIRO_CHUNK_MIN /
// SHIRO_CHUNK override; c2 at P = 1 lands at 56-64, c3/c4 at 256).
constexpr int32_t kChunk = 256;

int32_t unit_size(int64_t nnz) {
  static const int32_t fixed = getenv("SHIRO_CHUNK") ? atoi(getenv("SHIRO_CHUNK")) : 0;
  static const int32_t lmin = getenv("SHIRO_CHUNK_MIN") ? std::max(1, atoi(getenv("SHIRO_CHUNK_MIN"))) : 8;
  static const int32_t waves = getenv("SHIRO_WAVES") ? std::max(1, atoi(getenv("SHIRO_WAVES"))) : 4;
  if (fixed > 0) return fixed;
  int64_t L = nnz / ((int64_t)num_sms() * 32 * waves);
  L = (L / 8) * 8;
  return (int32_t)std::max<int64_t>(lmin, std::min<int64_t>(kChunk, L));
}
constexpr int32_t kMaxGroupRows = 64;

struct SplitHost {
  int32_t L = 0x7fffffff;
  std::vector<int32_t> task_long, long_row, long_first{0};
  std::vector<RowGroup> groups;
  std::vector<uint8_t> roff;
  std::vector<int2> cv;
  std::vector<uint64_t> unit_src;   // per unit (tasks, then groups): source mask
  std::vector<int32_t> vsrc;        // refresh map in cv order (two-phase ops permute)
  std::vector<int64_t> long_mid;    // two-phase ops: first remote nonzero of each long row
  std::vector<int32_t> hot_ids;     // compact hot buffer: its source rows (slot order)
  std::vector<int32_t> hot_dst;     // ... and their slots 0..H-1 (k_pack destinations)
  bool hot = false;
};

int64_t env_mb(const char *name, int64_t dflt) {
  const char *e = getenv(name);
  return e ? atoll(e) : dflt;
}

// Hot/cold L2 marks (kHotBit): when an op's source rows are far larger than
// L2, the most referenced source rows (column degree >= 2, highest first, up
// to SHIRO_HOT_MB of rows) are marked so that their gathers are L2
// evict_last and every other gather evict_first.
// The most referenced source rows of an op (column degree >= 2, highest
// first, ties by id) up to `budget` bytes of rows, when its source rows are
// more than SHIRO_HOT_MIN_MB (default 96 MB, i.e. far from L2-resident).
std::vector<int32_t> select_hot(const HostCsr &c, int N, int64_t budget) {
  const int64_t rowb = (int64_t)N * 4;
  const int64_t min_src = env_mb("SHIRO_HOT_MIN_MB", 96) << 20;
  if (c.hot_rows <= 0 || budget <= 0 || c.hot_rows * rowb <= min_src || c.nnz() == 0) return {};
  std::vector<int32_t> deg(c.hot_rows, 0);
  for (int32_t j : c.col)
    if (j >= 0 && j < c.hot_rows) deg[j]++;
  std::vector<int32_t> ids;
  for (int32_t j = 0; j < (int32_t)c.hot_rows; ++j)
    if (deg[j] >= 2) ids.push_back(j);
  const size_t H = std::min<size_t>(ids.size(), (size_t)(budget / rowb));
  std::partial_sort(ids.begin(), ids.begin() + H, ids.end(), [&](int32_t a, int32_t b) {
    return deg[a] != deg[b] ? deg[a] > deg[b] : a < b;
  });
  ids.resize(H);
  return ids;
}

void mark_hot(const HostCsr &c, int N, SplitHost &s) {
  const std::vector<int32_t> ids = select_hot(c, N, env_mb("SHIRO_HOT_MB", 0) << 20);
  if (ids.empty()) return;
  std::vector<uint8_t> hot(c.hot_rows, 0);
  for (int32_t j : ids) hot[j] = 1;
  for (int64_t k = 0; k < c.nnz(); ++k)
    if (c.col[k] >= 0 && c.col[k] < c.hot_rows && hot[c.col[k]]) s.cv[k].x |= kHotBit;
  s.hot = true;
}

// Compact hot buffer (SHIRO_HOTBUF_MB, single-source ops only): the hot
// source rows are copied each step into a contiguous buffer (one k_pack of
// hot_ids) that the op reads as its second source -- column j of a hot row
// becomes hot_rows + slot -- so an address-based L2 policy (the in-kernel
// evict_last of HINT 4, or a persisting access-policy window) covers exactly
// them, and the hot gathers share few pages.
void make_hotbuf(const HostCsr &c, int N, SplitHost &s) {
  if (s.hot || !c.mid.empty() || !c.src_bounds.empty() || !c.out_row.empty() || c.ptr_rows) return;
  s.hot_ids = select_hot(c, N, env_mb("SHIRO_HOTBUF_MB", 0) << 20);
  if (s.hot_ids.empty()) return;
  if (c.hot_rows + (int64_t)s.hot_ids.size() > 0x7fffffffLL) {   // ids stay int32
    s.hot_ids.clear();
    return;
  }
  std::vector<int32_t> slot(c.hot_rows, -1);
  for (size_t i = 0; i < s.hot_ids.size(); ++i) slot[s.hot_ids[i]] = (int32_t)i;
  for (int64_t k = 0; k < c.nnz(); ++k) {
    const int32_t j = c.col[k];
    if (j >= 0 && j < c.hot_rows && slot[j] >= 0) s.cv[k].x = (int32_t)(c.hot_rows + slot[j]);
  }
}

SplitHost make_split(const HostCsr &c, int N) {
  SplitHost s;
  s.cv.resize(c.nnz());
  for (int64_t k = 0; k < c.nnz(); ++k) {
    const float v = c.val.empty() ? 1.0f : c.val[k];
    int bits;
    std::memcpy(&bits, &v, 4);
    s.cv[k] = make_int2(c.col[k], bits);
  }
  int lpr, wv, vpl;
  if (!spmm_vec_shape(N, &lpr, &wv, &vpl)) return s;   // generic path: row per warp
  mark_hot(c, N, s);
  make_hotbuf(c, N, s);
  s.L = unit_size(c.nnz());
  s.roff.assign(c.nnz(), 0);
  const int64_t max_rows = (c.out_row.empty() && !c.ptr_rows) ? kMaxGroupRows
                                                              : std::min(kMaxGroupRows, 2 * lpr);
  auto deg = [&](int64_t r) { return c.rp[r + 1] - c.rp[r]; };
  // hub threshold: rows longer than H become chunk tasks; a row of L < deg <= H
  // is a unit of its own (no chunk reduction for moderately long rows)
  static const int64_t hmin = getenv("SHIRO_HUB_MIN") ? atoi(getenv("SHIRO_HUB_MIN")) : 64;
  const int64_t H = std::max<int64_t>(s.L, hmin);
  int64_t t = 0;
  while (t < c.nrows) {
    if (deg(t) > H) {
      const int32_t lr = (int32_t)s.long_row.size();
      s.long_row.push_back((int32_t)t);
      // chunk length ~max(H, sqrt(deg)): balances the serial walk of one chunk
      // against the in-order reduction of the chunk partials (both ~latency-bound)
      const int64_t clen = std::max<int64_t>(H, (int64_t)std::sqrt((double)deg(t)));
      const int64_t nch = (deg(t) + clen - 1) / clen;
      for (int64_t k = 0; k < nch; ++k) s.task_long.push_back(lr);
      s.long_first.push_back((int32_t)s.task_long.size());
      ++t;
      continue;
    }
    const int64_t r0 = t;
    int64_t sum = 0;
    while (t < c.nrows && deg(t) <= H && t - r0 < max_rows && (t == r0 || sum + deg(t) <= s.L)) {
      for (int64_t k = c.rp[t]; k < c.rp[t + 1]; ++k) s.roff[k] = (uint8_t)(t - r0);
      sum += deg(t);
      ++t;
    }
    s.groups.push_back(RowGroup{c.rp[r0], c.rp[t], c.rp[t], (int32_t)r0, (int32_t)t});
  }
  if (!c.mid.empty()) {
    // two-phase op: inside each group, every row's local part (row order),
    // then every row's remote part (row order); kmid between them
    if ((int64_t)c.mid.size() != c.nrows) throw Error(SHIRO_E_INTERNAL, "two-phase map size");
    s.vsrc = c.vsrc;
    std::vector<int2> tcv;
    std::vector<uint8_t> troff;
    std::vector<int32_t> tvs;
    for (RowGroup &g : s.groups) {
      tcv.clear(); troff.clear(); tvs.clear();
      for (int ph = 0; ph < 2; ++ph) {
        if (ph == 1) g.kmid = g.k0 + (int64_t)tcv.size();
        for (int32_t r = g.r0; r < g.r1; ++r) {
          const int64_t a = ph == 0 ? c.rp[r] : c.rp[r] + c.mid[r];
          const int64_t b = ph == 0 ? c.rp[r] + c.mid[r] : c.rp[r + 1];
          for (int64_t k = a; k < b; ++k) {
            tcv.push_back(s.cv[k]);
            troff.push_back(s.roff[k]);
            if (!s.vsrc.empty()) tvs.push_back(s.vsrc[k]);
          }
        }
      }
      std::copy(tcv.begin(), tcv.end(), s.cv.begin() + g.k0);
      std::copy(troff.begin(), troff.end(), s.roff.begin() + g.k0);
      if (!s.vsrc.empty()) std::copy(tvs.begin(), tvs.end(), s.vsrc.begin() + g.k0);
    }
    for (int32_t t : s.long_row) s.long_mid.push_back(c.rp[t] + c.mid[t]);
  }
  if (!c.src_bounds.empty()) {
    // per-unit source masks (fused exchange consumer): the sources whose
    // receive-buffer segments the unit's nonzeros read
    const auto &b = c.src_bounds;
    if (b.size() > 65) throw Error(SHIRO_E_INTERNAL, "source masks need P <= 64");
    auto mask_of = [&](int64_t k0, int64_t k1) {
      uint64_t m = 0;
      for (int64_t k = k0; k < k1; ++k) {
        const int64_t x = c.col[k];
        if (x < b[0]) continue;                     // local source row (B_local)
        const int src = (int)(std::upper_bound(b.begin(), b.end(), x) - b.begin()) - 1;
        if (src < 0 || src >= (int)b.size() - 1) throw Error(SHIRO_E_INTERNAL, "source of column");
        m |= 1ull << src;
      }
      return m;
    };
    for (size_t i = 0; i < s.task_long.size(); ++i) {
      const int32_t lr = s.task_long[i];
      const int64_t t0 = s.long_row[lr];
      const int64_t f = s.long_first[lr], nch = s.long_first[lr + 1] - f;
      const int64_t rb = c.rp[t0], re = c.rp[t0 + 1];
      const int64_t clen = (re - rb + nch - 1) / nch;    // as in the kernel
      const int64_t kb = rb + ((int64_t)i - f) * clen, ke = std::min(re, kb + clen);
      s.unit_src.push_back(mask_of(kb, ke));
    }
    for (const RowGroup &g : s.groups) s.unit_src.push_back(mask_of(g.k0, g.k1));
  }
  return s;
}

struct SpmmLayout {
  size_t rp, cv, roff, out, tl, lrow, lfirst, cnt, scratch, grp, usrc, vsrc, lmid, hsrc, hdst, hbuf;
  SplitHost sp;
  bool has_out, has_usrc, has_vsrc;
};

SpmmLayout layout_spmm(Arena &ar, const HostCsr &c, int N) {
  SpmmLayout L;
  L.sp = make_split(c, N);
  L.rp = put(ar, c.rp);
  L.cv = put(ar, L.sp.cv);
  L.roff = put(ar, L.sp.roff);
  L.has_out = !c.out_row.empty();
  L.out = put(ar, c.out_row);
  L.tl = put(ar, L.sp.task_long);
  L.lrow = put(ar, L.sp.long_row);
  L.lfirst = put(ar, L.sp.long_first);
  L.grp = put(ar, L.sp.groups);
  L.cnt = ar.reserve(L.sp.long_row.size() * sizeof(int32_t));          // zeroed
  L.scratch = ar.reserve(L.sp.task_long.size() * (size_t)N * sizeof(float));
  L.has_usrc = !L.sp.unit_src.empty();
  L.usrc = put(ar, L.sp.unit_src);
  L.has_vsrc = !c.vsrc.empty();
  if (L.has_vsrc && (int64_t)c.vsrc.size() != c.nnz())
    throw Error(SHIRO_E_INTERNAL, "refresh map size");
  L.vsrc = put(ar, L.sp.vsrc.empty() ? c.vsrc : L.sp.vsrc);
  L.lmid = put(ar, L.sp.long_mid);
  // (the arena keeps pointers to the host vectors until upload: they live in L.sp)
  L.sp.hot_dst.resize(L.sp.hot_ids.size());
  for (size_t i = 0; i < L.sp.hot_dst.size(); ++i) L.sp.hot_dst[i] = (int32_t)i;
  L.hsrc = put(ar, L.sp.hot_ids);
  L.hdst = put(ar, L.sp.hot_dst);
  L.hbuf = ar.reserve(L.sp.hot_ids.size() * (size_t)N * sizeof(float));
  return L;
}

DevSpmm bind_spmm(char *base, const SpmmLayout &L, const HostCsr &c, int N) {
  DevSpmm d;
  SpmmArgs &a = d.a;
  a.nrows = c.nrows;
  a.rp = reinterpret_cast<const int64_t *>(base + L.rp);
  a.cv = reinterpret_cast<const int2 *>(base + L.cv);
  a.roff = reinterpret_cast<const uint8_t *>(base + L.roff);
  a.out_row = L.has_out ? reinterpret_cast<const int32_t *>(base + L.out) : nullptr;
  a.N = N;
  a.L = L.sp.L;
  a.n_tasks = (int32_t)L.sp.task_long.size();
  a.n_groups = (int32_t)L.sp.groups.size();
  a.groups = reinterpret_cast<const RowGroup *>(base + L.grp);
  a.task_long = reinterpret_cast<const int32_t *>(base + L.tl);
  a.long_row = reinterpret_cast<const int32_t *>(base + L.lrow);
  a.long_first = reinterpret_cast<const int32_t *>(base + L.lfirst);
  a.long_counter = reinterpret_cast<int32_t *>(base + L.cnt);
  a.scratch = reinterpret_cast<float *>(base + L.scratch);
  a.hot = L.sp.hot ? 1 : 0;
  a.unit_src = L.has_usrc ? reinterpret_cast<const uint64_t *>(base + L.usrc) : nullptr;
  d.nnz = c.nnz();
  d.vsrc = L.has_vsrc ? reinterpret_cast<const int32_t *>(base + L.vsrc) : nullptr;
  a.long_mid = c.mid.empty() ? nullptr : reinterpret_cast<const int64_t *>(base + L.lmid);
  if (!L.sp.hot_ids.empty()) {
    d.hot.n = (int64_t)L.sp.hot_ids.size();
    d.hot.src = reinterpret_cast<const int32_t *>(base + L.hsrc);
    d.hot.dst = reinterpret_cast<const int32_t *>(base + L.hdst);
    d.hot_buf = reinterpret_cast<float *>(base + L.hbuf);
    d.hot_base = c.hot_rows;
    a.hot = 2;
  }
  return d;
}

}  // namespace

// SHIRO_DBUF=0 keeps one receive buffer and the CONSUMED round trip
bool dbuf_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("SHIRO_DBUF");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

void plan_upload(Plan &pl, cudaStream_t s) {
  SHIRO_CK(cudaGetDevice(&pl.device));
  // measurement knob: L2 set-aside for persisting (evict_last) lines
  if (const char *e = getenv("SHIRO_PERSIST_MB")) {
    const size_t mb = (size_t)atoll(e);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, mb << 20);
    cudaGetLastError();
  }
  Arena ar;
  const int N = pl.N;
  const size_t o_send = ar.reserve((size_t)pl.send_rows * N * sizeof(float));
  const size_t o_recv = ar.reserve((size_t)pl.recv_rows * N * sizeof(float));
  // second receive buffer for the double-buffered fused exchange
  const bool want2 = pl.P > 1 && !(pl.flags & SHIRO_F_XCHG_NCCL) && dbuf_enabled();
  const size_t o_recv2 = want2 ? ar.reserve((size_t)pl.recv_rows * N * sizeof(float)) : 0;
  // fused-exchange flags: ready[P], consumed[P], err, ep_sig, ep_wait,
  // done_ctr (IPC-exported with the arena)
  const size_t o_flags = ar.reserve((2 * (size_t)pl.P + 4) * sizeof(int32_t));
  const bool fused = !(pl.flags & SHIRO_F_SPLIT_RECV);
  SpmmLayout l_diag = layout_spmm(ar, pl.A_diag, N);
  SpmmLayout l_out = layout_spmm(ar, pl.A_out, N);
  HostCsr empty;
  SpmmLayout l_col = layout_spmm(ar, fused ? empty : pl.A_col, N);
  SpmmLayout l_rem = layout_spmm(ar, fused ? pl.A_rem : empty, N);
  const size_t o_ps = put(ar, pl.pack_src), o_pd = put(ar, pl.pack_dst);
  const size_t o_st = put(ar, pl.sc_tgt), o_sp = put(ar, pl.sc_ptr), o_ss = put(ar, pl.sc_src);
  pl.arena_bytes = std::max<size_t>(ar.total, 256);
  SHIRO_CK(cudaMalloc(&pl.arena, pl.arena_bytes));
  SHIRO_CK(cudaMemsetAsync(pl.arena, 0, pl.arena_bytes, s));
  char *base = static_cast<char *>(pl.arena);
  for (const auto &it : ar.items)
    if (it.src && it.bytes)
      SHIRO_CK(cudaMemcpyAsync(base + it.off, it.src, it.bytes, cudaMemcpyHostToDevice, s));
  SHIRO_CK(cudaStreamSynchronize(s));
  pl.send_buf = reinterpret_cast<float *>(base + o_send);
  pl.recv_buf = reinterpret_cast<float *>(base + o_recv);
  pl.xflags = reinterpret_cast<int32_t *>(base + o_flags);
  pl.recv_buf_off = (int64_t)o_recv;
  if (want2) {
    pl.recv_buf2 = reinterpret_cast<float *>(base + o_recv2);
    pl.recv_buf2_off = (int64_t)o_recv2;
  }
  pl.flags_off = (int64_t)o_flags;
  pl.d_diag = bind_spmm(base, l_diag, pl.A_diag, N);
  pl.d_out = bind_spmm(base, l_out, pl.A_out, N);
  pl.d_col = bind_spmm(base, l_col, fused ? empty : pl.A_col, N);
  pl.d_rem = bind_spmm(base, l_rem, fused ? pl.A_rem : empty, N);
  pl.d_pack.n = (int64_t)pl.pack_src.size();
  pl.d_pack.src = reinterpret_cast<const int32_t *>(base + o_ps);
  pl.d_pack.dst = reinterpret_cast<const int32_t *>(base + o_pd);
  pl.d_scatter.nt = (int64_t)pl.sc_tgt.size();
  pl.d_scatter.tgt = reinterpret_cast<const int32_t *>(base + o_st);
  pl.d_scatter.ptr = reinterpret_cast<const int64_t *>(base + o_sp);
  pl.d_scatter.src = reinterpret_cast<const int32_t *>(base + o_ss);
  pl.d_scatter.nsrc = (int64_t)pl.sc_src.size();
  pl.refresh_ops = {&pl.d_diag, &pl.d_out, &pl.d_col, &pl.d_rem};
  pl.info.dev_bytes = (int64_t)pl.arena_bytes;
  // per-op algorithmic work (before the host images are dropped)
  auto distinct = [](const std::vector<int32_t> &ids) {
    if (ids.empty()) return (int64_t)0;
    std::vector<int32_t> v(ids);
    std::sort(v.begin(), v.end());
    return (int64_t)(std::unique(v.begin(), v.end()) - v.begin());
  };
  auto op = [&](int i, const HostCsr &c) {
    pl.info.op_nnz[i] = c.nnz();
    pl.info.op_rows[i] = c.nrows;
    pl.info.op_src_rows[i] = distinct(c.col);
  };
  op(SHIRO_OP_LOCAL, pl.A_diag);
  op(SHIRO_OP_PARTIAL, pl.A_out);
  op(SHIRO_OP_REMOTE, fused ? pl.A_rem : pl.A_col);
  pl.info.op_nnz[SHIRO_OP_SCATTER] = fused ? 0 : (int64_t)pl.sc_src.size();
  pl.info.op_rows[SHIRO_OP_SCATTER] = fused ? 0 : (int64_t)pl.sc_tgt.size();
  pl.info.op_src_rows[SHIRO_OP_SCATTER] = fused ? 0 : (int64_t)pl.sc_src.size();
  pl.info.op_nnz[SHIRO_OP_PACK] = (int64_t)pl.pack_src.size();
  pl.info.op_rows[SHIRO_OP_PACK] = (int64_t)pl.pack_src.size();
  pl.info.op_src_rows[SHIRO_OP_PACK] = distinct(pl.pack_src);
  if (!pl.loopback_view) {
    SHIRO_CK(cudaStreamCreateWithFlags(&pl.comm_stream, cudaStreamNonBlocking));
    SHIRO_CK(cudaEventCreateWithFlags(&pl.ev_packed, cudaEventDisableTiming));
    SHIRO_CK(cudaEventCreateWithFlags(&pl.ev_recvd, cudaEventDisableTiming));
  }
}

// Host images are dropped once every device image has been built.
void plan_drop_host(Plan &pl) {
  pl.A_diag = HostCsr(); pl.A_out = HostCsr(); pl.A_col = HostCsr(); pl.A_rem = HostCsr();
  std::vector<int32_t>().swap(pl.pack_src);
  std::vector<int32_t>().swap(pl.pack_dst);
  std::vector<int32_t>().swap(pl.sc_tgt);
  std::vector<int32_t>().swap(pl.sc_src);
  std::vector<int64_t>(1, 0).swap(pl.sc_ptr);
  pl.route.s1_part = HostCsr(); pl.route.s2_agg = HostCsr(); pl.route.fin = HostCsr();
}

// Fused producer op of the fused exchange: one SpMM launch whose rows are
// (1) the packed B rows (one unit-weight nonzero each, K4) and (2) the
// row-based partial rows (A_out, K3), both stored at peer addresses; with
// `with_local` (hierarchical Stage I) also (3) the local rows (A_diag, K1)
// stored into C (tagged row index).  The flat exchange runs K1 as its own
// launch concurrently with this one (exec_p2p).
static bool prod_ops_exist(const Plan &pl) { return pl.prod_ops != nullptr; }

void upload_prod(Plan &pl, const std::vector<int32_t> &pack_src,
                 const std::vector<uint64_t> &pack_addr, const std::vector<uint64_t> &part_addr,
                 bool with_local, const std::vector<uint64_t> *pack_addr2,
                 const std::vector<uint64_t> *part_addr2) {
  HostCsr c;
  c.ptr_rows = true;
  c.hot_rows = pl.M;
  std::vector<uint64_t> outp, outp2;
  const bool two = pack_addr2 && part_addr2;
  const int64_t np = (int64_t)pack_src.size();
  const bool refresh = !pl.A_out.vsrc.empty() || !pl.A_diag.vsrc.empty();
  if (prod_ops_exist(pl)) { cudaFree(pl.prod_ops); pl.prod_ops = nullptr; }
  auto pack_row = [&](int64_t i) {
    c.col.push_back(pack_src[i]);
    c.val.push_back(1.0f);
    if (refresh) c.vsrc.push_back(-1);
    c.rp.push_back((int64_t)c.col.size());
    outp.push_back(pack_addr[i]);
    if (two) outp2.push_back((*pack_addr2)[i]);
  };
  auto append = [&](const HostCsr &a, int64_t t) {
    for (int64_t k = a.rp[t]; k < a.rp[t + 1]; ++k) {
      c.col.push_back(a.col[k]);
      c.val.push_back(a.val[k]);
      if (refresh) c.vsrc.push_back(a.vsrc.empty() ? -1 : a.vsrc[k]);
    }
    c.rp.push_back((int64_t)c.col.size());
  };
  auto part_row = [&](int64_t t) {
    append(pl.A_out, t);
    outp.push_back(part_addr[t]);
    if (two) outp2.push_back((*part_addr2)[t]);
  };
  // Flat exchange: the rows for peer d are the send_b[d] pack rows and the
  // send_c[d] partial rows (both lists peer-ascending).  Every rank visits
  // its peers in its own rotated order rank+1, rank+2, ... so that at any
  // moment the P producers store into P different receivers instead of all
  // into the same one (incast on one GPU's NVLink ports); the destinations
  // are per-row addresses, so the order is free.
  int64_t nb = 0, nc = 0;
  for (int d = 0; d < pl.P; ++d) { nb += (int64_t)pl.send_b[d].size(); nc += (int64_t)pl.send_c[d].size(); }
  if (!with_local && nb == np && nc == pl.A_out.nrows && pl.P > 1) {
    std::vector<int64_t> b0(pl.P + 1, 0), c0(pl.P + 1, 0);
    for (int d = 0; d < pl.P; ++d) {
      b0[d + 1] = b0[d] + (int64_t)pl.send_b[d].size();
      c0[d + 1] = c0[d] + (int64_t)pl.send_c[d].size();
    }
    for (int k = 1; k < pl.P; ++k) {
      const int d = (pl.rank + k) % pl.P;
      for (int64_t i = b0[d]; i < b0[d + 1]; ++i) pack_row(i);
      for (int64_t t = c0[d]; t < c0[d + 1]; ++t) part_row(t);
    }
  } else {
    for (int64_t i = 0; i < np; ++i) pack_row(i);
    for (int64_t t = 0; t < pl.A_out.nrows; ++t) part_row(t);
  }
  if (with_local)
    for (int64_t t = 0; t < pl.A_diag.nrows; ++t) {
      append(pl.A_diag, t);
      outp.push_back((1ull << 63) | (uint64_t)t);       // local row of C
      if (two) outp2.push_back((1ull << 63) | (uint64_t)t);
    }
  c.nrows = (int64_t)outp.size();
  Arena ar;
  SpmmLayout L = layout_spmm(ar, c, pl.N);
  const size_t o_ptr = put(ar, outp);
  const size_t o_ptr2 = two ? put(ar, outp2) : 0;
  SHIRO_CK(cudaMalloc(&pl.prod_ops, std::max<size_t>(ar.total, 256)));
  SHIRO_CK(cudaMemset(pl.prod_ops, 0, std::max<size_t>(ar.total, 256)));
  char *base = static_cast<char *>(pl.prod_ops);
  for (const auto &it : ar.items)
    if (it.src && it.bytes)
      SHIRO_CK(cudaMemcpy(base + it.off, it.src, it.bytes, cudaMemcpyHostToDevice));
  pl.d_prod = bind_spmm(base, L, c, pl.N);
  pl.d_prod.a.out_ptr = reinterpret_cast<float *const *>(base + o_ptr);
  pl.prod_out_ptr[0] = pl.d_prod.a.out_ptr;
  pl.prod_out_ptr[1] = two ? reinterpret_cast<float *const *>(base + o_ptr2) : nullptr;
  pl.refresh_ops.push_back(&pl.d_prod);
  pl.info.dev_bytes += (int64_t)ar.total;
  // the producer launch carries pack + partial (+ local); its work replaces
  // those ops in the per-op statistics
  std::vector<int32_t> src(c.col);
  std::sort(src.begin(), src.end());
  const int64_t nsrc = (int64_t)(std::unique(src.begin(), src.end()) - src.begin());
  const int slot = with_local ? SHIRO_OP_LOCAL : SHIRO_OP_PARTIAL;
  pl.info.op_nnz[slot] = c.nnz();
  pl.info.op_rows[slot] = c.nrows;
  pl.info.op_src_rows[slot] = nsrc;
  pl.info.op_nnz[SHIRO_OP_PACK] = pl.info.op_rows[SHIRO_OP_PACK] = pl.info.op_src_rows[SHIRO_OP_PACK] = 0;
  if (with_local) {
    pl.info.op_nnz[SHIRO_OP_PARTIAL] = pl.info.op_rows[SHIRO_OP_PARTIAL] = 0;
    pl.info.op_src_rows[SHIRO_OP_PARTIAL] = 0;
  }
}

// Two-phase consumer of the fused exchange: every local
// row t, its diagonal nonzeros (columns in B_local) then its A_rem entries
// (column-based entries and unit-weight partials, columns shifted by M into
// the receive buffer); mid[t] = number of diagonal nonzeros.  Overwrite, one
// store per row in phase A, read-modify-write in phase B only for rows with
// remote entries.
void upload_merged(Plan &pl) {
  const int64_t M = pl.M;
  const HostCsr &ad = pl.A_diag, &ar = pl.A_rem;
  std::vector<int64_t> rem_of(M, -1);
  for (int64_t i = 0; i < ar.nrows; ++i) rem_of[ar.out_row[i]] = i;
  const bool refresh = !ad.vsrc.empty();
  HostCsr cx;
  cx.nrows = M;
  cx.mid.resize(M);
  cx.col.reserve(ad.nnz() + ar.nnz());
  for (int64_t t = 0; t < M; ++t) {
    for (int64_t k = ad.rp[t]; k < ad.rp[t + 1]; ++k) {
      cx.col.push_back(ad.col[k]);
      cx.val.push_back(ad.val[k]);
      if (refresh) cx.vsrc.push_back(ad.vsrc[k]);
    }
    cx.mid[t] = (int32_t)(ad.rp[t + 1] - ad.rp[t]);
    if (const int64_t i = rem_of[t]; i >= 0)
      for (int64_t k = ar.rp[i]; k < ar.rp[i + 1]; ++k) {
        cx.col.push_back((int32_t)(M + ar.col[k]));
        cx.val.push_back(ar.val[k]);
        if (refresh) cx.vsrc.push_back(ar.vsrc.empty() ? -1 : ar.vsrc[k]);
      }
    cx.rp.push_back((int64_t)cx.col.size());
  }
  for (int64_t b : pl.recv_off) cx.src_bounds.push_back(M + b);   // per-unit source masks
  if (M + pl.recv_rows > 0x7fffffffLL)
    throw Error(SHIRO_E_ARG, "two-phase consumer: more than 2^31 source rows");
  Arena ar2;
  SpmmLayout L = layout_spmm(ar2, cx, pl.N);
  const size_t units = L.sp.task_long.size() + L.sp.groups.size();
  const size_t o_def = ar2.reserve(std::max<size_t>(1, units) * sizeof(int32_t));   // deferred list
  const size_t o_ctr = ar2.reserve(2 * sizeof(int32_t));                            // defer_n, work_ctr
  if (pl.merged_ops) cudaFree(pl.merged_ops);
  SHIRO_CK(cudaMalloc(&pl.merged_ops, std::max<size_t>(ar2.total, 256)));
  SHIRO_CK(cudaMemset(pl.merged_ops, 0, std::max<size_t>(ar2.total, 256)));
  char *base = static_cast<char *>(pl.merged_ops);
  for (const auto &it : ar2.items)
    if (it.src && it.bytes)
      SHIRO_CK(cudaMemcpy(base + it.off, it.src, it.bytes, cudaMemcpyHostToDevice));
  pl.d_cx = bind_spmm(base, L, cx, pl.N);
  pl.d_cx.a.defer_list = reinterpret_cast<int32_t *>(base + o_def);
  pl.d_cx.a.defer_n = reinterpret_cast<int32_t *>(base + o_ctr);
  pl.d_cx.a.work_ctr = reinterpret_cast<int32_t *>(base + o_ctr) + 1;
  pl.refresh_ops.push_back(&pl.d_cx);
  pl.info.dev_bytes += (int64_t)ar2.total;
  // the consumer carries the local (K1) and remote (K2 + K5) work of a step
  std::vector<int32_t> src(cx.col);
  std::sort(src.begin(), src.end());
  pl.info.op_nnz[SHIRO_OP_LOCAL] = ad.nnz();
  pl.info.op_rows[SHIRO_OP_LOCAL] = M;
  pl.info.op_nnz[SHIRO_OP_REMOTE] = cx.nnz();
  pl.info.op_rows[SHIRO_OP_REMOTE] = M;
  pl.info.op_src_rows[SHIRO_OP_REMOTE] = (int64_t)(std::unique(src.begin(), src.end()) - src.begin());
  pl.merged = true;
}

// N3 value refresh on the device: upload V, then rewrite the value half of
// every op's (column, value) pairs through its map.
void refresh_device(Plan &pl, const std::vector<float> &V, cudaStream_t s) {
  if (!pl.arena) throw Error(SHIRO_E_ARG, "plan has no device state (SHIRO_F_HOST_ONLY)");
  const size_t bytes = std::max<size_t>(1, V.size()) * sizeof(float);
  if (!pl.vspace) SHIRO_CK(cudaMalloc(&pl.vspace, (size_t)std::max<int64_t>(1, pl.nnz_local + pl.nnz_recv_vals) * sizeof(float)));
  if ((int64_t)V.size() != pl.nnz_local + pl.nnz_recv_vals)
    throw Error(SHIRO_E_INTERNAL, "refresh: value space size");
  if (!V.empty()) SHIRO_CK(cudaMemcpyAsync(pl.vspace, V.data(), bytes, cudaMemcpyHostToDevice, s));
  for (DevSpmm *d : pl.refresh_ops)
    if (d->vsrc && d->nnz)
      launch_refresh(d->nnz, d->vsrc, pl.vspace, const_cast<int2 *>(d->a.cv), s);
  if (pl.route.active) {
    Route &R = pl.route;
    for (DevSpmm *d : {&R.d_part, &R.d_agg, &R.d_fin})
      if (d->vsrc && d->nnz)
        launch_refresh(d->nnz, d->vsrc, pl.vspace, const_cast<int2 *>(d->a.cv), s);
  }
  SHIRO_CK(cudaGetLastError());
  SHIRO_CK(cudaStreamSynchronize(s));   // V (host) may go away after the call
}

namespace {

// SHIRO_HOTBUF_WIN=1: a persisting L2 access-policy window over the compact
// hot buffer around its op's launch (measurement knob)
bool hotbuf_window() {
  static const int v = getenv("SHIRO_HOTBUF_WIN") ? atoi(getenv("SHIRO_HOTBUF_WIN")) : 0;
  return v == 1;
}

int64_t run_spmm(const DevSpmm &d, const float *X0, int64_t n0, const float *X1, float *Y,
                 bool accumulate, cudaStream_t s) {
  if (d.a.nrows == 0) return 0;
  SpmmArgs a = d.a;
  a.X0 = X0; a.n0 = n0; a.X1 = X1; a.Y = Y;
  int64_t n = 0;
  if (d.hot.n) {   // compact hot buffer: this step's hot rows of X0, then the op reads it as X1
    if (X1 || n0 != d.hot_base) throw Error(SHIRO_E_INTERNAL, "hot buffer op with a second source");
    n += launch_pack(d.hot.n, d.hot.src, d.hot.dst, X0, d.hot_buf, a.N, s);
    a.X1 = d.hot_buf;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    SHIRO_CK(cudaStreamIsCapturing(s, &cap));
    if (hotbuf_window() && cap == cudaStreamCaptureStatusNone) {   // direct launches only
      cudaStreamAttrValue v = {};
      v.accessPolicyWindow.base_ptr = d.hot_buf;
      v.accessPolicyWindow.num_bytes = (size_t)d.hot.n * a.N * sizeof(float);
      v.accessPolicyWindow.hitRatio = 1.0f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      SHIRO_CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
      n += launch_spmm(a, accumulate, s);
      v.accessPolicyWindow.num_bytes = 0;
      SHIRO_CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
      return n;
    }
  }
  return n + launch_spmm(a, accumulate, s);
}

// E1 + E2: fill the send buffer from B
int64_t stage_send(Plan &pl, const float *B, cudaStream_t s) {
  int64_t n = 0;
  n += launch_pack(pl.d_pack.n, pl.d_pack.src, pl.d_pack.dst, B, pl.send_buf, pl.N, s);
  n += run_spmm(pl.d_out, B, pl.M, nullptr, pl.send_buf, false, s);
  return n;
}

// E5 + E6: consume the receive buffer
int64_t stage_recv(Plan &pl, float *C, cudaStream_t s) {
  int64_t n = 0;
  if (!(pl.flags & SHIRO_F_SPLIT_RECV)) {
    n += run_spmm(pl.d_rem, pl.recv_buf, pl.recv_rows, nullptr, C, true, s);
  } else {
    n += run_spmm(pl.d_col, pl.recv_buf, pl.recv_rows, nullptr, C, true, s);
    n += launch_scatter_add(pl.d_scatter.nt, pl.d_scatter.tgt, pl.d_scatter.ptr, pl.d_scatter.src,
                            pl.recv_buf, C, pl.N, s);
  }
  return n;
}

int64_t stage_local(Plan &pl, const float *B, float *C, cudaStream_t s) {
  if (pl.M == 0) return 0;
  return run_spmm(pl.d_diag, B, pl.M, nullptr, C, false, s);
}

}  // namespace

void exec_flat(Plan &pl, const float *B, float *C, cudaStream_t s) {
  // profiling events: 0 start | 1 after pack | 2 after partial | 3,4 exchange
  // (comm stream) | 5 local start | 6 local end | 7 after remote | 8 end
  auto rec = [&](int i, cudaStream_t st) {
    if (pl.prof_on) SHIRO_CK(cudaEventRecord(pl.prof[i], st));
  };
  int64_t launches = 0;
  if (pl.P == 1) {
    rec(5, s);
    launches += stage_local(pl, B, C, s);
    rec(6, s);
    pl.last_launches = launches;
    pl.prof_used = 1;
    return;
  }
  const bool overlap = !(pl.flags & SHIRO_F_NO_OVERLAP);
  rec(0, s);
  launches += launch_pack(pl.d_pack.n, pl.d_pack.src, pl.d_pack.dst, B, pl.send_buf, pl.N, s);
  rec(1, s);
  launches += run_spmm(pl.d_out, B, pl.M, nullptr, pl.send_buf, false, s);
  rec(2, s);
  SHIRO_CK(cudaEventRecord(pl.ev_packed, s));
  SHIRO_CK(cudaStreamWaitEvent(pl.comm_stream, pl.ev_packed, 0));
  rec(3, pl.comm_stream);
  SHIRO_NCK(ncclGroupStart());
  for (int k = 1; k < pl.P; ++k) {
    // ring-shifted peer order: same schedule on every rank
    const int d = (pl.rank + k) % pl.P, src = (pl.rank - k + pl.P) % pl.P;
    const int64_t ns = pl.send_off[d + 1] - pl.send_off[d];
    const int64_t nr = pl.recv_off[src + 1] - pl.recv_off[src];
    if (ns) SHIRO_NCK(ncclSend(pl.send_buf + pl.send_off[d] * pl.N, (size_t)(ns * pl.N), ncclFloat,
                               d, pl.comm, pl.comm_stream));
    if (nr) SHIRO_NCK(ncclRecv(pl.recv_buf + pl.recv_off[src] * pl.N, (size_t)(nr * pl.N),
                               ncclFloat, src, pl.comm, pl.comm_stream));
  }
  SHIRO_NCK(ncclGroupEnd());
  rec(4, pl.comm_stream);
  SHIRO_CK(cudaEventRecord(pl.ev_recvd, pl.comm_stream));
  if (overlap) {
    rec(5, s);
    launches += stage_local(pl, B, C, s);
    rec(6, s);
  }
  SHIRO_CK(cudaStreamWaitEvent(s, pl.ev_recvd, 0));
  if (!overlap) {
    rec(5, s);
    launches += stage_local(pl, B, C, s);
    rec(6, s);
  }
  if (!(pl.flags & SHIRO_F_SPLIT_RECV)) {
    launches += run_spmm(pl.d_rem, pl.recv_buf, pl.recv_rows, nullptr, C, true, s);
    rec(7, s);
  } else {
    launches += run_spmm(pl.d_col, pl.recv_buf, pl.recv_rows, nullptr, C, true, s);
    rec(7, s);
    launches += launch_scatter_add(pl.d_scatter.nt, pl.d_scatter.tgt, pl.d_scatter.ptr,
                                   pl.d_scatter.src, pl.recv_buf, C, pl.N, s);
  }
  rec(8, s);
  pl.last_launches = launches;
  pl.prof_used = 2;
}

// ---------------------------------------------------------------------------
// Hierarchical routing: device images, destination resolution, executor.
// ---------------------------------------------------------------------------
void hier_upload(Plan &pl) {
  Route &R = pl.route;
  const int N = pl.N, P = pl.P;
  Arena ab;
  const size_t o_rb = ab.reserve((size_t)(R.r1_rows + R.r2_rows) * N * sizeof(float));
  const size_t o_fl = ab.reserve((3 * (size_t)P + 2) * sizeof(int32_t));
  SHIRO_CK(cudaMalloc(&R.arena, std::max<size_t>(ab.total, 256)));
  SHIRO_CK(cudaMemset(R.arena, 0, std::max<size_t>(ab.total, 256)));
  char *bb = static_cast<char *>(R.arena);
  R.rb = reinterpret_cast<float *>(bb + o_rb);
  R.xflags = reinterpret_cast<int32_t *>(bb + o_fl);
  R.rb_off = (int64_t)o_rb;
  R.flags_off = (int64_t)o_fl;
  Arena ar;
  SpmmLayout lp = layout_spmm(ar, R.s1_part, N);
  SpmmLayout lg = layout_spmm(ar, R.s2_agg, N);
  SpmmLayout lf = layout_spmm(ar, R.fin, N);
  const size_t o_p1 = put(ar, R.s1_pack_src), o_fw = put(ar, R.s2_fwd_src);
  SHIRO_CK(cudaMalloc(&R.ops, std::max<size_t>(ar.total, 256)));
  SHIRO_CK(cudaMemset(R.ops, 0, std::max<size_t>(ar.total, 256)));
  char *base = static_cast<char *>(R.ops);
  for (const auto &it : ar.items)
    if (it.src && it.bytes)
      SHIRO_CK(cudaMemcpy(base + it.off, it.src, it.bytes, cudaMemcpyHostToDevice));
  R.d_part = bind_spmm(base, lp, R.s1_part, N);
  R.d_agg = bind_spmm(base, lg, R.s2_agg, N);
  R.d_fin = bind_spmm(base, lf, R.fin, N);
  R.d_pack1.n = (int64_t)R.s1_pack_src.size();
  R.d_pack1.src = reinterpret_cast<const int32_t *>(base + o_p1);
  R.d_fwd.n = (int64_t)R.s2_fwd_src.size();
  R.d_fwd.src = reinterpret_cast<const int32_t *>(base + o_fw);
  pl.info.dev_bytes += (int64_t)(ab.total + ar.total);
}

void hier_resolve(Plan &pl, const std::function<char *(int, int)> &seg,
                  const std::function<int32_t *(int, int)> &flag) {
  Route &R = pl.route;
  const int P = pl.P, me = pl.rank;
  const int64_t rowb = (int64_t)pl.N * sizeof(float);
  std::vector<uint64_t> v;
  auto add = [&](const std::vector<Dest> &ds) {
    for (const Dest &d : ds) v.push_back((uint64_t)(seg(d.rank, d.buf) + d.pos * rowb));
  };
  add(R.s1_pack_dst);
  add(R.s1_part_dst);
  add(R.s2_fwd_dst);
  add(R.s2_agg_dst);
  const size_t n_rows = v.size();
  for (int k = 0; k < 3; ++k)
    for (int d = 0; d < P; ++d)
      if (d != me) v.push_back((uint64_t)flag(d, k * P + me));
  if (R.ptrs) cudaFree(R.ptrs);
  SHIRO_CK(cudaMalloc(&R.ptrs, std::max<size_t>(8, v.size() * 8)));
  if (!v.empty()) SHIRO_CK(cudaMemcpy(R.ptrs, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
  uint64_t *a = static_cast<uint64_t *>(R.ptrs);
  size_t o = 0;
  R.pack1_dstp = reinterpret_cast<float *const *>(a + o); o += R.s1_pack_dst.size();
  R.d_part.a.out_ptr = reinterpret_cast<float *const *>(a + o); o += R.s1_part_dst.size();
  R.fwd_dstp = reinterpret_cast<float *const *>(a + o); o += R.s2_fwd_dst.size();
  R.d_agg.a.out_ptr = reinterpret_cast<float *const *>(a + o); o += R.s2_agg_dst.size();
  if (o != n_rows) throw Error(SHIRO_E_INTERNAL, "route pointer count");
  R.ready1_ptrs = reinterpret_cast<int32_t *const *>(a + o); o += P - 1;
  R.ready2_ptrs = reinterpret_cast<int32_t *const *>(a + o); o += P - 1;
  R.consumed_ptrs = reinterpret_cast<int32_t *const *>(a + o);
  // own flags never block
  std::vector<int32_t> f(3 * P + 2, 0);
  f[me] = f[P + me] = f[2 * P + me] = 0x7fffffff;
  SHIRO_CK(cudaMemcpy(R.xflags, f.data(), f.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  // Stage I producers + local rows as one launch (same as the flat fused exchange)
  const size_t n1 = R.s1_pack_dst.size(), n2 = R.s1_part_dst.size();
  upload_prod(pl, R.s1_pack_src, std::vector<uint64_t>(v.begin(), v.begin() + n1),
              std::vector<uint64_t>(v.begin() + n1, v.begin() + n1 + n2), true);
}

// stage 1: B rows and partial C rows -> R1 (peers and self); stage 2: forward
// B rows and pre-aggregated partials R1 -> R2 (peers); stage 3: final remote
// SpMM over [R1 || R2] into C.
int64_t hier_stage(Plan &pl, int stage, const float *B, float *C, cudaStream_t s) {
  Route &R = pl.route;
  int64_t n = 0;
  if (stage == 1) {
    n += launch_pack_ptr(R.d_pack1.n, R.d_pack1.src, R.pack1_dstp, B, pl.N, s);
    n += run_spmm(R.d_part, B, pl.M, nullptr, nullptr, false, s);
  } else if (stage == 2) {
    n += launch_pack_ptr(R.d_fwd.n, R.d_fwd.src, R.fwd_dstp, R.rb, pl.N, s);
    n += run_spmm(R.d_agg, R.rb, R.r1_rows, nullptr, nullptr, false, s);
  } else {
    n += run_spmm(R.d_fin, R.rb, R.r1_rows + R.r2_rows, nullptr, C, true, s);
  }
  return n;
}

void exec_hier(Plan &pl, const float *B, float *C, cudaStream_t s) {
  if (*pl.err_host) throw Error(SHIRO_E_PEER, "hierarchical exchange: a peer did not signal in time");
  Route &R = pl.route;
  auto rec = [&](int i) {
    if (pl.prof_on) SHIRO_CK(cudaEventRecord(pl.prof[i], s));
  };
  const int P = pl.P;
  int32_t *err = R.xflags + 3 * P, *ep = R.xflags + 3 * P + 1;   // device epoch e-1
  int64_t n = 0;
  rec(0);
  n += launch_wait(R.xflags + 2 * P, P, ep, 0, err, pl.wait_timeout_ns, s);   // CONSUMED >= e-1
  // Stage I producers (B-row unions, partial rows -> R1 of peers/self) and
  // the local rows (K1 -> C) in one launch
  n += run_spmm(pl.d_prod, B, pl.M, nullptr, C, false, s);
  rec(1);
  n += launch_signal(R.ready1_ptrs, P - 1, ep, 1, false, s);
  rec(2);
  n += launch_wait(R.xflags, P, ep, 1, err, pl.wait_timeout_ns, s);
  rec(3);
  n += hier_stage(pl, 2, B, C, s);                        // Stage II producers
  n += launch_signal(R.ready2_ptrs, P - 1, ep, 1, false, s);
  rec(4);
  n += launch_wait(R.xflags + P, P, ep, 1, err, pl.wait_timeout_ns, s);
  rec(5);
  n += hier_stage(pl, 3, B, C, s);                        // final remote SpMM
  rec(6);
  n += launch_signal(R.consumed_ptrs, P - 1, ep, 1, true, s);   // ... and advance the epoch
  SHIRO_CK(cudaMemcpyAsync(pl.err_host, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  pl.last_launches = n;
  pl.prof_used = 4;
}

// Fused exchange (SHIRO_F_XCHG_NCCL unset, P > 1): K4/K3 store rows straight
// into the peers' receive buffers over NVLink; flags order the producer and
// consumer sides (p2p.cu).  No staging copy, no NCCL kernel.  One step:
//
//   s_hi (high priority):  [wait CONSUMED >= e-1, single buffer only]
//                          producer: K4 pack + K3 partial SpMM -> peers' buffers
//                          signal READY = e at every peer
//   s    (caller's stream): K1 local SpMM -> C       (concurrently with s_hi)
//                          K2+K5 remote SpMM, C += A_rem * recv: each work
//                          unit waits only for the READY flags of the sources
//                          its nonzeros read (rows of a peer
//                          are consumed as soon as they land); the last warp
//                          also waits for every peer before the step ends
//                          [signal CONSUMED = e, single buffer only]
//   join s_hi -> s.
//
// Double buffering (default): step e's rows land in the peers' buffer e mod
// 2.  A peer read that buffer last in its remote SpMM of step e-2, which
// completed before its step e-1 forked its producer and READY(e-1) -- and
// this rank's step e-1 ended only after READY(e-1) from every peer.  So no
// CONSUMED round trip.  The producer runs on a high-priority stream: CTAs of
// the remote SpMM that spin on a late peer can never keep this GPU's own
// producer from being scheduled.  Epochs: ep_sig (advanced by the READY
// signal) and ep_wait (advanced by the remote SpMM's last warp) live in
// device memory, so the whole step is one replayable CUDA graph.
// Consumer wait of the fused exchange.  Default: one k_wait launch for every
// peer's READY, then the remote SpMM with read-only (L1-cached) loads.
// SHIRO_INKERNEL_WAIT=1: per-source consumption -- every remote work unit
// waits (in the kernel) only for the READY of the sources it reads.  Measured
// on 2 and 4 B200 (profiles/r2m4b_*, r2m2e_*): on one NVSwitch box the peers'
// rows land within microseconds of each other (balanced producers, rotated
// peer order), so the per-unit acquires cost more than they overlap (c2/P=4
// 0.0695 vs 0.0654 ms, c3 1.214 vs 1.184, c4 0.802 vs 0.798).
bool inkernel_wait_enabled() {
  const char *e = getenv("SHIRO_INKERNEL_WAIT");   // read per step (cheap)
  return e && e[0] == '1';
}

// The split consumer is used with the in-kernel waits, the fused K2+K5 and a
// vector width (the WAIT kernel); otherwise local SpMM -> k_wait -> remote.
// Opt-in (SHIRO_CX=1) until its spin-free variant exists: with its warps
// spinning in phase B, the consumer can occupy every SM slot before the
// GPU's own producer has finished, and two GPUs then wait on each other
// (seen on 2 x B200; one GPU shared by two processes time-slices and hides it).
bool merged_enabled(const Plan &pl) {
  const char *e = getenv("SHIRO_CX");     // read at plan time
  int lpr, wv, vpl;
  return e && e[0] == '1' && inkernel_wait_enabled() && !(pl.flags & SHIRO_F_SPLIT_RECV) &&
         spmm_vec_shape(pl.N, &lpr, &wv, &vpl);
}

void exec_p2p(Plan &pl, const float *B, float *C, cudaStream_t s) {
  if (*pl.err_host) throw Error(SHIRO_E_PEER, "fused exchange: a peer did not signal in time");
  auto rec = [&](int i, cudaStream_t st) {
    if (pl.prof_on) SHIRO_CK(cudaEventRecord(pl.prof[i], st));
  };
  const int P = pl.P;
  int32_t *err = pl.xflags + 2 * P, *ep_sig = err + 1, *ep_wait = err + 2;
  int64_t launches = 0;
  const int par = pl.dbuf ? pl.step_parity : 0;
  float *rb = par ? pl.recv_buf2 : pl.recv_buf;
  if (pl.merged) {
    // two-phase consumer: producer (s_hi) || CX stage 1 (s: every unit's K1
    // part, its K2 + K5 part too if its sources are READY already, else the
    // unit is deferred); after this GPU's producer + READY: CX stage 2 (the
    // deferred units, with per-source waits) -- no warp spins before the join
    rec(0, s);
    SHIRO_CK(cudaEventRecord(pl.ev_fork, s));
    SHIRO_CK(cudaStreamWaitEvent(pl.s_hi, pl.ev_fork, 0));
    if (!pl.dbuf)
      launches += launch_wait(pl.xflags + P, P, ep_sig, 0, err, pl.wait_timeout_ns, pl.s_hi);
    DevSpmm prod = pl.d_prod;
    prod.a.out_ptr = pl.prod_out_ptr[par];
    launches += run_spmm(prod, B, pl.M, nullptr, C, false, pl.s_hi);
    rec(1, pl.s_hi);
    launches += launch_signal(pl.ready_ptrs, P - 1, ep_sig, 1, true, pl.s_hi);
    rec(2, pl.s_hi);
    SHIRO_CK(cudaEventRecord(pl.ev_join, pl.s_hi));
    if (pl.d_cx.a.n_groups + pl.d_cx.a.n_tasks > 0) {
      DevSpmm cx = pl.d_cx;
      cx.a.ready = pl.xflags;
      cx.a.wait_epoch = ep_wait;
      cx.a.wait_err = err;
      cx.a.wait_timeout_ns = pl.wait_timeout_ns;
      cx.a.cx_stage = 1;
      launches += run_spmm(cx, B, pl.M, rb, C, false, s);
      rec(3, s);
      SHIRO_CK(cudaStreamWaitEvent(s, pl.ev_join, 0));
      cx.a.cx_stage = 2;
      launches += run_spmm(cx, B, pl.M, rb, C, false, s);
      SHIRO_CK(cudaMemsetAsync(pl.d_cx.a.defer_n, 0, 2 * sizeof(int32_t), s));   // re-arm
    } else {
      rec(3, s);
      SHIRO_CK(cudaStreamWaitEvent(s, pl.ev_join, 0));
    }
    // step-end barrier (READY from every peer) and the epoch advance
    launches += launch_wait(pl.xflags, P, ep_wait, 1, err, pl.wait_timeout_ns, s, true);
    rec(4, s);
    if (!pl.dbuf) launches += launch_signal(pl.consumed_ptrs, P - 1, ep_wait, 0, false, s);
    rec(5, s);
    SHIRO_CK(cudaMemcpyAsync(pl.err_host, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    pl.last_launches = launches;
    pl.prof_used = 5;
    return;
  }
  // fork: the producer branch
  rec(0, s);
  SHIRO_CK(cudaEventRecord(pl.ev_fork, s));
  SHIRO_CK(cudaStreamWaitEvent(pl.s_hi, pl.ev_fork, 0));
  if (!pl.dbuf)   // single buffer: every peer consumed my rows of step e-1
    launches += launch_wait(pl.xflags + P, P, ep_sig, 0, err, pl.wait_timeout_ns, pl.s_hi);
  DevSpmm prod = pl.d_prod;
  prod.a.out_ptr = pl.prod_out_ptr[par];
  launches += run_spmm(prod, B, pl.M, nullptr, C, false, pl.s_hi);
  rec(1, pl.s_hi);
  launches += launch_signal(pl.ready_ptrs, P - 1, ep_sig, 1, true, pl.s_hi);
  rec(2, pl.s_hi);
  SHIRO_CK(cudaEventRecord(pl.ev_join, pl.s_hi));
  // consumer branch: K1 (concurrent with the producer branch); then, once
  // this GPU's own producer and READY signal are done (so no spinning
  // consumer warp can hold an SM slot its producer needs), the remote SpMM
  // whose units each wait only for the sources they read
  launches += stage_local(pl, B, C, s);
  rec(3, s);
  SHIRO_CK(cudaStreamWaitEvent(s, pl.ev_join, 0));
  int lpr_, w_, vpl_;
  const bool split = pl.flags & SHIRO_F_SPLIT_RECV;
  if (inkernel_wait_enabled() && !split && pl.d_rem.a.n_groups + pl.d_rem.a.n_tasks > 0 &&
      spmm_vec_shape(pl.N, &lpr_, &w_, &vpl_)) {
    DevSpmm rem = pl.d_rem;
    rem.a.ready = pl.xflags;
    rem.a.wait_epoch = ep_wait;
    rem.a.wait_err = err;
    rem.a.wait_timeout_ns = pl.wait_timeout_ns;
    launches += run_spmm(rem, rb, pl.recv_rows, nullptr, C, true, s);
    // step-end barrier (READY from every peer) and the epoch advance
    launches += launch_wait(pl.xflags, P, ep_wait, 1, err, pl.wait_timeout_ns, s, true);
  } else {
    launches += launch_wait(pl.xflags, P, ep_wait, 1, err, pl.wait_timeout_ns, s, true);
    if (!split) {
      launches += run_spmm(pl.d_rem, rb, pl.recv_rows, nullptr, C, true, s);
    } else {
      launches += run_spmm(pl.d_col, rb, pl.recv_rows, nullptr, C, true, s);
      launches += launch_scatter_add(pl.d_scatter.nt, pl.d_scatter.tgt, pl.d_scatter.ptr,
                                     pl.d_scatter.src, rb, C, pl.N, s);
    }
  }
  rec(4, s);
  if (!pl.dbuf) launches += launch_signal(pl.consumed_ptrs, P - 1, ep_wait, 0, false, s);
  rec(5, s);
  SHIRO_CK(cudaMemcpyAsync(pl.err_host, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  pl.last_launches = launches;
  pl.prof_used = 3;
}

void exec_plan(Plan &pl, const float *B, float *C, cudaStream_t s) {
  if (pl.route.active && pl.P > 1) exec_hier(pl, B, C, s);
  else if (pl.p2p) exec_p2p(pl, B, C, s);
  else exec_flat(pl, B, C, s);
}

}  // namespace shiro

// ===========================================================================
// C ABI
// ===========================================================================
using namespace shiro;

struct shiro_plan_s {
  bool loopback = false;
  std::unique_ptr<Plan> single;                 // distributed: this rank
  std::vector<std::unique_ptr<Plan>> ranks;     // loopback: all virtual ranks
  std::vector<std::unique_ptr<shiro_plan_s>> views;
  Plan *view = nullptr;                         // borrowed rank view
  int64_t last_launches = 0;
  // loopback value refresh: planned-matrix value offset of each virtual rank
  // and (SHIRO_F_TRANSPOSE) the entry permutation A -> A^T
  std::vector<int64_t> lb_val_off, lb_tperm;
  int64_t lb_nnz = 0;
  Plan &rank_plan() { return view ? *view : *single; }
};

namespace {

thread_local std::string g_last_error;

// A step is captured into a CUDA graph (and replayed while B, C, the stream
// and the profiling state are unchanged) for the paths whose launches have
// static arguments: P = 1, the fused exchange and the hierarchical schedule
// (their epochs live on the device).  Not on the legacy default stream (it
// cannot be captured), not for the NCCL exchange; SHIRO_GRAPH=0 disables.
bool graph_eligible(const Plan &pl, cudaStream_t s) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("SHIRO_GRAPH");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  if (!env || s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread) return false;
  if (pl.prof_on) return false;      // stage events need direct launches
  return pl.P == 1 || pl.p2p || pl.route.active;
}

void launch_graph(Plan &pl, const float *B, float *C, cudaStream_t s) {
  if (pl.err_host && *pl.err_host)
    throw Error(SHIRO_E_PEER, "fused exchange: a peer did not signal in time");
  const int par = pl.dbuf ? pl.step_parity : 0;
  Plan::GraphSlot *hit = nullptr;
  for (auto &c : pl.graphs)
    if (c.exec && c.parity == par && c.B == B && c.C == C && c.s == s && c.prof == pl.prof_on)
      hit = &c;
  Plan::GraphSlot &g = hit ? *hit : pl.graphs[pl.graph_next++ % 4];
  if (!hit) {
    if (g.exec) {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    SHIRO_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t cg = nullptr;
    try {
      exec_plan(pl, B, C, s);
    } catch (...) {
      cudaStreamEndCapture(s, &cg);
      if (cg) cudaGraphDestroy(cg);
      throw;
    }
    SHIRO_CK(cudaStreamEndCapture(s, &cg));
    const cudaError_t ie = cudaGraphInstantiate(&g.exec, cg, 0);
    cudaGraphDestroy(cg);
    SHIRO_CK(ie);
    g.parity = par;
    g.B = B;
    g.C = C;
    g.s = s;
    g.prof = pl.prof_on;
    g.launches = pl.last_launches;
  }
  SHIRO_CK(cudaGraphLaunch(g.exec, s));
  pl.last_launches = g.launches;
}

// One step through the graph or direct launches; advances the step parity
// of the double-buffered exchange (every rank calls in the same order).
void run_step(Plan &pl, const float *B, float *C, cudaStream_t s) {
  if (graph_eligible(pl, s)) launch_graph(pl, B, C, s);
  else exec_plan(pl, B, C, s);
  if (pl.dbuf) pl.step_parity ^= 1;
}

int fail(const Error &e) {
  g_last_error = e.msg;
  return e.code;
}

template <typename F>
int guarded(F &&f) {
  try {
    g_last_error.clear();
    f();
    return SHIRO_OK;
  } catch (const Error &e) {
    return fail(e);
  } catch (const std::bad_alloc &) {
    return fail(Error(SHIRO_E_OOM, "host allocation failed"));
  } catch (const std::exception &e) {
    return fail(Error(SHIRO_E_INTERNAL, e.what()));
  }
}

// NCCL all-to-allv of host byte segments (plan time only): sizes first.
void nccl_host_alltoallv(ncclComm_t comm, int P, int rank, cudaStream_t s,
                         const std::vector<std::vector<char>> &send,
                         std::vector<std::vector<char>> &recv) {
  std::vector<int64_t> ssz(P, 0), rsz(P, 0);
  for (int p = 0; p < P; ++p) ssz[p] = p == rank ? 0 : (int64_t)send[p].size();
  int64_t *d_sz = nullptr;
  SHIRO_CK(cudaMalloc(&d_sz, 2 * P * sizeof(int64_t)));
  SHIRO_CK(cudaMemcpyAsync(d_sz, ssz.data(), P * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  SHIRO_NCK(ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    if (p == rank) continue;
    SHIRO_NCK(ncclSend(d_sz + p, 8, ncclChar, p, comm, s));
    SHIRO_NCK(ncclRecv(d_sz + P + p, 8, ncclChar, p, comm, s));
  }
  SHIRO_NCK(ncclGroupEnd());
  SHIRO_CK(cudaMemcpyAsync(rsz.data(), d_sz + P, P * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SHIRO_CK(cudaStreamSynchronize(s));
  SHIRO_CK(cudaFree(d_sz));
  rsz[rank] = 0;
  std::vector<int64_t> so(P + 1, 0), ro(P + 1, 0);
  for (int p = 0; p < P; ++p) { so[p + 1] = so[p] + ssz[p]; ro[p + 1] = ro[p] + rsz[p]; }
  char *d_buf = nullptr;
  SHIRO_CK(cudaMalloc(&d_buf, std::max<int64_t>(1, so[P] + ro[P])));
  for (int p = 0; p < P; ++p)
    if (ssz[p]) SHIRO_CK(cudaMemcpyAsync(d_buf + so[p], send[p].data(), ssz[p],
                                         cudaMemcpyHostToDevice, s));
  SHIRO_NCK(ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    if (p == rank) continue;
    if (ssz[p]) SHIRO_NCK(ncclSend(d_buf + so[p], ssz[p], ncclChar, p, comm, s));
    if (rsz[p]) SHIRO_NCK(ncclRecv(d_buf + so[P] + ro[p], rsz[p], ncclChar, p, comm, s));
  }
  SHIRO_NCK(ncclGroupEnd());
  recv.assign(P, {});
  for (int p = 0; p < P; ++p) {
    recv[p].resize(rsz[p]);
    if (rsz[p]) SHIRO_CK(cudaMemcpyAsync(recv[p].data(), d_buf + so[P] + ro[p], rsz[p],
                                         cudaMemcpyDeviceToHost, s));
  }
  SHIRO_CK(cudaStreamSynchronize(s));
  SHIRO_CK(cudaFree(d_buf));
}

// Caller-provided host transport (e.g. gloo): sizes first, then payload.
void callback_alltoallv(shiro_alltoallv_fn fn, void *ctx, int P, int rank,
                        const std::vector<std::vector<char>> &send,
                        std::vector<std::vector<char>> &recv) {
  std::vector<int64_t> ssz(P, 0), rsz(P, 0), eight(P, 8);
  for (int p = 0; p < P; ++p) ssz[p] = p == rank ? 0 : (int64_t)send[p].size();
  eight[rank] = 8;
  if (fn(ctx, ssz.data(), eight.data(), rsz.data(), eight.data()) != 0)
    throw Error(SHIRO_E_TRANSPORT, "host transport failed (sizes)");
  rsz[rank] = 0;
  std::vector<char> sb, rb;
  int64_t rt = 0;
  for (int p = 0; p < P; ++p) {
    if (p != rank) sb.insert(sb.end(), send[p].begin(), send[p].end());
    rt += rsz[p];
  }
  ssz[rank] = 0;
  rb.resize(std::max<int64_t>(rt, 1));
  if (sb.empty()) sb.resize(1);
  if (fn(ctx, sb.data(), ssz.data(), rb.data(), rsz.data()) != 0)
    throw Error(SHIRO_E_TRANSPORT, "host transport failed (payload)");
  recv.assign(P, {});
  int64_t o = 0;
  for (int p = 0; p < P; ++p) {
    recv[p].assign(rb.begin() + o, rb.begin() + o + rsz[p]);
    o += rsz[p];
  }
}

// Status agreement before any payload exchange (every rank learns every
// rank's validation status).
int agree_status(const Alltoallv &x, int P, int rank, int mine) {
  std::vector<std::vector<char>> send(P), recv;
  for (int p = 0; p < P; ++p) {
    send[p].resize(4);
    std::memcpy(send[p].data(), &mine, 4);
  }
  x(send, recv);
  int worst = mine;
  for (int p = 0; p < P; ++p) {
    if (p == rank) continue;
    int v = 0;
    if (recv[p].size() == 4) std::memcpy(&v, recv[p].data(), 4);
    if (v != 0 && worst == 0) worst = SHIRO_E_PEER;
  }
  return worst;
}

void fill_block_stats(const Phase1 &p1, const PlanInput &in, Plan &pl) {
  int64_t cols = 0, rows = 0, block = 0, setup = 0;
  for (int q = 0; q < in.P; ++q) {
    if (q == in.rank || p1.n_cols[q] == 0) continue;
    cols += p1.n_cols[q];
    rows += p1.n_rows[q];
    block += in.part[q + 1] - in.part[q];
    setup += 8 * p1.nnz_row[q];
  }
  pl.loc_cols = cols;
  pl.loc_rows = rows;
  pl.loc_block = block;
  pl.loc_setup = setup;
}

}  // namespace

extern "C" {

const char *shiro_last_error(void) { return g_last_error.c_str(); }

int shiro_get_unique_id(void *id128) {
  return guarded([&] {
    if (!id128) throw Error(SHIRO_E_ARG, "id buffer is NULL");
    ncclUniqueId id;
    SHIRO_NCK(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId must be 128 bytes");
    std::memcpy(id128, &id, 128);
  });
}

static int plan_impl(const shiro_dist_t *d, int64_t n, const int64_t *part,
                     const int64_t *row_ptr, const int32_t *col_idx, const float *val, int32_t N,
                     const int64_t *w_row, const int64_t *w_col, void *stream, shiro_plan_t *out) {
  if (out) *out = nullptr;
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    if (!d || !out) throw Error(SHIRO_E_ARG, "dist/out is NULL");
    const bool host_only = d->flags & SHIRO_F_HOST_ONLY;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PlanInput in{d->rank, d->nranks, d->group_size, d->flags, n, part, row_ptr, col_idx, val, N};
    if ((w_row == nullptr) != (w_col == nullptr))
      throw Error(SHIRO_E_ARG, "w_row and w_col must both be given or both be NULL");
    in.w_row = w_row;
    in.w_col = w_col;
    if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks)
      throw Error(SHIRO_E_ARG, "bad rank/nranks");
    auto h = std::make_unique<shiro_plan_s>();
    h->single = std::make_unique<Plan>();
    Plan &pl = *h->single;
    // transport
    Alltoallv xchg;
    if (d->nranks > 1) {
      if (d->host_xchg) {
        xchg = [&](const std::vector<std::vector<char>> &snd, std::vector<std::vector<char>> &rcv) {
          callback_alltoallv(d->host_xchg, d->host_xchg_ctx, d->nranks, d->rank, snd, rcv);
        };
      }
      // NCCL communicator: needed for the NCCL exchange or as the plan-time
      // transport; skipped when a host transport is given and the fused
      // exchange (IPC peer stores, no NCCL) carries the data
      const bool need_nccl = !d->host_xchg || (d->flags & SHIRO_F_XCHG_NCCL) ||
                             (!host_only && d->nccl_id);
      if (need_nccl) {
        if (!d->nccl_id) throw Error(SHIRO_E_ARG, "nccl_id is NULL with nranks > 1");
        ncclUniqueId id;
        std::memcpy(&id, d->nccl_id, 128);
        SHIRO_NCK(ncclCommInitRank(&pl.comm, d->nranks, id, d->rank));
        if (!d->host_xchg) {
          ncclComm_t comm = pl.comm;
          int P = d->nranks, r = d->rank;
          xchg = [comm, P, r, s](const std::vector<std::vector<char>> &snd,
                                 std::vector<std::vector<char>> &rcv) {
            nccl_host_alltoallv(comm, P, r, s, snd, rcv);
          };
        }
      }
    } else {
      xchg = [](const std::vector<std::vector<char>> &snd, std::vector<std::vector<char>> &rcv) {
        rcv.assign(snd.size(), {});
      };
    }
    // P1: validate, then agree on the status across ranks
    int st = 0;
    std::string msg;
    try {
      validate_input(in);
    } catch (const Error &e) {
      st = e.code;
      msg = e.msg;
    }
    if (d->nranks > 1) {
      int agreed = agree_status(xchg, d->nranks, d->rank, st);
      if (agreed != 0) throw Error(st ? st : agreed, st ? msg : "another rank failed validation");
    } else if (st) {
      throw Error(st, msg);
    }
    // SHIRO_F_TRANSPOSE: plan A^T instead of A (one distributed transpose)
    std::vector<int64_t> t_rp;
    std::vector<int32_t> t_col;
    std::vector<float> t_val;
    if (d->flags & SHIRO_F_TRANSPOSE) {
      std::vector<std::vector<char>> tmsg = transpose_messages(in), trecv;
      xchg(tmsg, trecv);
      trecv.resize(d->nranks);
      trecv[d->rank] = tmsg[d->rank];
      transpose_assemble(in, trecv, t_rp, t_col, t_val, &pl.tperm);
      in.row_ptr = t_rp.data();
      in.col = t_col.data();
      in.val = t_val.data();
    }
    // P2-P3
    Phase1 p1 = plan_phase1(in);
    // P4: one-time exchange of lists + A_row
    std::vector<std::vector<char>> in_msgs;
    xchg(p1.out, in_msgs);
    in_msgs.resize(d->nranks);
    plan_phase2(in, p1, in_msgs, pl);
    const bool hier = d->group_size > 1 && d->nranks > 1;
    if (hier) {
      if (d->flags & SHIRO_F_XCHG_NCCL)
        throw Error(SHIRO_E_ARG, "the hierarchical schedule uses the fused NVLink exchange");
      std::vector<std::vector<char>> meta;
      xchg(hier_meta_messages(pl), meta);
      meta.resize(d->nranks);
      hier_build(in, p1, pl, meta);
    }
    fill_block_stats(p1, in, pl);
    plan_stats(in, pl, xchg);
    if (!host_only) {
      plan_upload(pl, s);
      if (hier) {
        hier_upload(pl);
        hier_p2p_setup(pl, xchg);
      } else if (d->nranks > 1 && !(d->flags & SHIRO_F_XCHG_NCCL)) {
        p2p_setup(pl, xchg);   // collective: every rank agrees on p2p or not
        if (!pl.p2p && !pl.comm)
          throw Error(SHIRO_E_ARG, "fused exchange unavailable and no nccl_id for the NCCL exchange");
      }
      plan_drop_host(pl);
    }
    // transport of later value refreshes (N3): the caller's host transport
    // (must outlive the plan) or the plan's NCCL communicator
    if (d->nranks > 1) {
      if (d->host_xchg) {
        shiro_alltoallv_fn fn = d->host_xchg;
        void *ctx = d->host_xchg_ctx;
        const int P = d->nranks, r = d->rank;
        pl.refresh_xchg = [fn, ctx, P, r](const std::vector<std::vector<char>> &snd,
                                          std::vector<std::vector<char>> &rcv) {
          callback_alltoallv(fn, ctx, P, r, snd, rcv);
        };
      } else if (pl.comm) {
        ncclComm_t comm = pl.comm;
        const int P = d->nranks, r = d->rank;
        cudaStream_t cs = pl.comm_stream;
        pl.refresh_xchg = [comm, P, r, cs](const std::vector<std::vector<char>> &snd,
                                           std::vector<std::vector<char>> &rcv) {
          nccl_host_alltoallv(comm, P, r, cs, snd, rcv);
        };
      }
    }
    pl.info.plan_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
  });
}

int shiro_plan(const shiro_dist_t *d, int64_t n, const int64_t *part, const int64_t *row_ptr,
               const int32_t *col_idx, const float *val, int32_t N, void *stream,
               shiro_plan_t *out) {
  return plan_impl(d, n, part, row_ptr, col_idx, val, N, nullptr, nullptr, stream, out);
}

int shiro_plan_weighted(const shiro_dist_t *d, int64_t n, const int64_t *part,
                        const int64_t *row_ptr, const int32_t *col_idx, const float *val, int32_t N,
                        const int64_t *w_row, const int64_t *w_col, void *stream,
                        shiro_plan_t *out) {
  if (!w_row || !w_col) {
    if (out) *out = nullptr;
    return guarded([&] { throw Error(SHIRO_E_ARG, "w_row / w_col is NULL"); });
  }
  return plan_impl(d, n, part, row_ptr, col_idx, val, N, w_row, w_col, stream, out);
}

int shiro_plan_update_values(shiro_plan_t plan, const int64_t *row_ptr, const int32_t *col_idx,
                             const float *val, void *stream) {
  return guarded([&] {
    if (!plan || plan->loopback || plan->view) throw Error(SHIRO_E_ARG, "not a distributed plan");
    Plan &pl = *plan->single;
    if (!pl.arena) throw Error(SHIRO_E_ARG, "plan was built with SHIRO_F_HOST_ONLY");
    if (pl.nnz_local > 0 && !val) throw Error(SHIRO_E_ARG, "val is NULL");
    if ((pl.flags & SHIRO_F_TRANSPOSE) && (!row_ptr || (pl.M > 0 && !col_idx)))
      throw Error(SHIRO_E_ARG, "transposed plans need row_ptr and col_idx");
    if (pl.P > 1 && !pl.refresh_xchg) throw Error(SHIRO_E_ARG, "plan has no refresh transport");
    auto t0 = std::chrono::steady_clock::now();
    PlanInput in{pl.rank, pl.P, pl.g, pl.flags, pl.n, pl.part.data(), row_ptr, col_idx, val, pl.N};
    std::vector<float> V = refresh_value_space(pl, in, val, pl.refresh_xchg);
    refresh_device(pl, V, static_cast<cudaStream_t>(stream));
    pl.refresh_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    pl.info.refresh_seconds = pl.refresh_seconds;
  });
}

static int plan_loopback_impl(int32_t nranks, int32_t group_size, uint32_t flags, int64_t n,
                              const int64_t *part, const int64_t *row_ptr,
                              const int32_t *col_idx, const float *val, int32_t N,
                              const int64_t *w_row, const int64_t *w_col, void *stream,
                              shiro_plan_t *out) {
  if (out) *out = nullptr;
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    if (!out || !part || !row_ptr) throw Error(SHIRO_E_ARG, "NULL argument");
    if (nranks < 1 || nranks > 64) throw Error(SHIRO_E_ARG, "nranks must be in 1..64");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool host_only = flags & SHIRO_F_HOST_ONLY;
    const int P = nranks;
    auto h = std::make_unique<shiro_plan_s>();
    h->loopback = true;
    std::vector<PlanInput> ins(P);
    std::vector<int64_t> lb_t_rp;      // full A^T for SHIRO_F_TRANSPOSE
    std::vector<int32_t> lb_t_col;
    std::vector<float> lb_t_val;
    std::vector<std::vector<int64_t>> rps(P);
    for (int r = 0; r < P; ++r) {
      PlanInput in{r, P, group_size, flags, n, part, nullptr, nullptr, nullptr, N};
      if ((w_row == nullptr) != (w_col == nullptr))
        throw Error(SHIRO_E_ARG, "w_row and w_col must both be given or both be NULL");
      in.w_row = w_row ? w_row + part[r] : nullptr;
      in.w_col = w_col;
      if (part[0] != 0 || part[P] != n) throw Error(SHIRO_E_PART, "part[0]/part[P] mismatch");
      if (r == 0 && (flags & SHIRO_F_TRANSPOSE)) {
        // full A^T on the host (validated as A first)
        PlanInput all{0, 1, 1, 0, n, nullptr, row_ptr, col_idx, val, N};
        const int64_t part1[2] = {0, n};
        all.part = part1;
        validate_input(all);
        std::vector<std::vector<char>> one = transpose_messages(all);
        transpose_assemble(all, one, lb_t_rp, lb_t_col, lb_t_val, &h->lb_tperm);
        row_ptr = lb_t_rp.data();
        col_idx = lb_t_col.data();
        val = lb_t_val.data();
      }
      for (int p = 0; p < P; ++p)
        if (part[p + 1] < part[p]) throw Error(SHIRO_E_PART, "part must be non-decreasing");
      const int64_t lo = part[r], hi = part[r + 1], base = row_ptr[lo];
      if (r == 0) { h->lb_val_off.assign(P + 1, 0); h->lb_nnz = row_ptr[n]; }
      h->lb_val_off[r] = base;
      h->lb_val_off[r + 1] = row_ptr[hi];
      rps[r].resize(hi - lo + 1);
      for (int64_t t = lo; t <= hi; ++t) rps[r][t - lo] = row_ptr[t] - base;
      in.row_ptr = rps[r].data();
      in.col = col_idx ? col_idx + base : nullptr;
      in.val = val ? val + base : nullptr;
      validate_input(in);
      ins[r] = in;
    }
    std::vector<Phase1> p1(P);
    for (int r = 0; r < P; ++r) p1[r] = plan_phase1(ins[r]);
    // in-process exchange: message r -> q lands at q from r
    std::vector<std::vector<std::vector<char>>> inbox(P, std::vector<std::vector<char>>(P));
    for (int r = 0; r < P; ++r)
      for (int q = 0; q < P; ++q)
        if (q != r) inbox[q][r] = p1[r].out[q];
    for (int r = 0; r < P; ++r) {
      h->ranks.push_back(std::make_unique<Plan>());
      Plan &pl = *h->ranks.back();
      pl.loopback_view = false;
      plan_phase2(ins[r], p1[r], inbox[r], pl);
      fill_block_stats(p1[r], ins[r], pl);
    }
    const bool hier = group_size > 1 && P > 1;
    if (hier) {
      std::vector<std::vector<std::vector<char>>> mbox(P, std::vector<std::vector<char>>(P));
      for (int r = 0; r < P; ++r) {
        auto out_m = hier_meta_messages(*h->ranks[r]);
        for (int q = 0; q < P; ++q)
          if (q != r) mbox[q][r] = std::move(out_m[q]);
      }
      for (int r = 0; r < P; ++r) hier_build(ins[r], p1[r], *h->ranks[r], mbox[r]);
    }
    // stats exchange among virtual ranks: run plan_stats sequentially with a
    // transport that serves precomputed vectors (two passes)
    std::vector<std::vector<char>> shares(P);
    for (int r = 0; r < P; ++r) {
      Alltoallv cap = [&, r](const std::vector<std::vector<char>> &snd,
                             std::vector<std::vector<char>> &rcv) {
        shares[r] = snd[(r + 1) % P];
        rcv.assign(P, {});
        for (int p = 0; p < P; ++p) rcv[p] = snd[(r + 1) % P];
      };
      plan_stats(ins[r], *h->ranks[r], cap);
    }
    for (int r = 0; r < P; ++r) {
      Alltoallv serve = [&](const std::vector<std::vector<char>> &,
                            std::vector<std::vector<char>> &rcv) {
        rcv.assign(P, {});
        for (int p = 0; p < P; ++p) rcv[p] = shares[p];
      };
      plan_stats(ins[r], *h->ranks[r], serve);
    }
    for (int r = 0; r < P; ++r) {
      Plan &pl = *h->ranks[r];
      if (!host_only) {
        plan_upload(pl, s);
        if (hier) hier_upload(pl);
      }
      pl.info.plan_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (hier && !host_only) {
      // same-device "peers": destinations are the other virtual ranks' buffers
      for (int r = 0; r < P; ++r) {
        Plan &pl = *h->ranks[r];
        auto seg = [&, r](int d, int buf) -> char * {
          Route &D = h->ranks[d]->route;
          const int64_t row = (buf == 0) ? D.r1_off[r] : D.r1_rows + D.r2_off[r];
          return reinterpret_cast<char *>(D.rb) + row * (int64_t)pl.N * (int64_t)sizeof(float);
        };
        auto flag = [&](int d, int i) -> int32_t * { return h->ranks[d]->route.xflags + i; };
        hier_resolve(pl, seg, flag);
      }
    } else if (!host_only && P > 1 && !(flags & SHIRO_F_XCHG_NCCL)) {
      // fused producer launch with same-device destinations (the kernels of
      // the NVLink path); SHIRO_F_XCHG_NCCL keeps the staged copy exchange
      for (int r = 0; r < P; ++r) {
        Plan &pl = *h->ranks[r];
        const int64_t rowb = (int64_t)pl.N * sizeof(float);
        std::vector<uint64_t> dstp, outp;
        for (int d = 0; d < P; ++d) {
          if (d == r) continue;
          Plan &D = *h->ranks[d];
          char *base = reinterpret_cast<char *>(D.recv_buf) + D.recv_off[r] * rowb;
          for (size_t k = 0; k < pl.send_b[d].size(); ++k)
            dstp.push_back((uint64_t)(base + (int64_t)k * rowb));
          const int64_t nb = (int64_t)pl.send_b[d].size();
          for (size_t k = 0; k < pl.send_c[d].size(); ++k)
            outp.push_back((uint64_t)(base + (nb + (int64_t)k) * rowb));
        }
        upload_prod(pl, pl.pack_src, dstp, outp, false);
        if (merged_enabled(pl)) upload_merged(pl);
        pl.p2p = true;      // marks the pointer-routed path (no flags in loopback)
      }
    }
    if (!host_only)
      for (int r = 0; r < P; ++r) plan_drop_host(*h->ranks[r]);
    *out = h.release();
  });
}

int shiro_plan_loopback(int32_t nranks, int32_t group_size, uint32_t flags, int64_t n,
                        const int64_t *part, const int64_t *row_ptr, const int32_t *col_idx,
                        const float *val, int32_t N, void *stream, shiro_plan_t *out) {
  return plan_loopback_impl(nranks, group_size, flags, n, part, row_ptr, col_idx, val, N, nullptr,
                            nullptr, stream, out);
}

int shiro_plan_loopback_weighted(int32_t nranks, int32_t group_size, uint32_t flags, int64_t n,
                                 const int64_t *part, const int64_t *row_ptr,
                                 const int32_t *col_idx, const float *val, int32_t N,
                                 const int64_t *w_row, const int64_t *w_col, void *stream,
                                 shiro_plan_t *out) {
  if (!w_row || !w_col) {
    if (out) *out = nullptr;
    return guarded([&] { throw Error(SHIRO_E_ARG, "w_row / w_col is NULL"); });
  }
  return plan_loopback_impl(nranks, group_size, flags, n, part, row_ptr, col_idx, val, N, w_row,
                            w_col, stream, out);
}

int shiro_plan_update_values_loopback(shiro_plan_t plan, const float *val, void *stream) {
  return guarded([&] {
    if (!plan || !plan->loopback || plan->view) throw Error(SHIRO_E_ARG, "not a loopback plan");
    if (plan->lb_nnz > 0 && !val) throw Error(SHIRO_E_ARG, "val is NULL");
    const int P = (int)plan->ranks.size();
    for (auto &p : plan->ranks)
      if (!p->arena) throw Error(SHIRO_E_ARG, "plan was built with SHIRO_F_HOST_ONLY");
    auto t0 = std::chrono::steady_clock::now();
    std::vector<float> tv;
    const float *pv = val;
    if (!plan->lb_tperm.empty() || (plan->ranks[0]->flags & SHIRO_F_TRANSPOSE)) {
      tv.resize(plan->lb_nnz);
      for (int64_t x = 0; x < plan->lb_nnz; ++x) tv[x] = val[plan->lb_tperm[x]];
      pv = tv.data();
    }
    // in-process exchange of the row-based values, then every rank's V
    std::vector<std::vector<std::vector<char>>> out(P);
    for (int r = 0; r < P; ++r) out[r] = refresh_ship(*plan->ranks[r], pv + plan->lb_val_off[r]);
    for (int r = 0; r < P; ++r) {
      std::vector<std::vector<char>> rcv(P);
      for (int q = 0; q < P; ++q)
        if (q != r) rcv[q] = out[q][r];
      std::vector<float> V = refresh_assemble(*plan->ranks[r], pv + plan->lb_val_off[r], rcv);
      refresh_device(*plan->ranks[r], V, static_cast<cudaStream_t>(stream));
    }
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto &p : plan->ranks) { p->refresh_seconds = sec; p->info.refresh_seconds = sec; }
  });
}

int shiro_plan_rank(shiro_plan_t plan, int32_t r, shiro_plan_t *out) {
  return guarded([&] {
    if (!plan || !out) throw Error(SHIRO_E_ARG, "NULL argument");
    if (!plan->loopback) {
      if (r != plan->single->rank) throw Error(SHIRO_E_ARG, "not this rank");
      *out = plan;
      return;
    }
    if (r < 0 || r >= (int)plan->ranks.size()) throw Error(SHIRO_E_ARG, "rank out of range");
    if (plan->views.empty())
      for (auto &p : plan->ranks) {
        auto v = std::make_unique<shiro_plan_s>();
        v->view = p.get();
        plan->views.push_back(std::move(v));
      }
    *out = plan->views[r].get();
  });
}

int shiro_spmm(shiro_plan_t plan, const float *B_p, float *C_p, void *stream) {
  return guarded([&] {
    if (!plan || plan->loopback || plan->view) throw Error(SHIRO_E_ARG, "not a distributed plan");
    Plan &pl = *plan->single;
    if (!pl.arena) throw Error(SHIRO_E_ARG, "plan was built with SHIRO_F_HOST_ONLY");
    if (pl.M > 0 && (!B_p || !C_p)) throw Error(SHIRO_E_ARG, "B/C is NULL");
    if (pl.comm) {
      ncclResult_t as = ncclSuccess;
      ncclCommGetAsyncError(pl.comm, &as);
      if (as != ncclSuccess && as != ncclInProgress)
        throw Error(SHIRO_E_NCCL, std::string("asynchronous NCCL error: ") + ncclGetErrorString(as));
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    run_step(pl, B_p, C_p, s);
    SHIRO_CK(cudaGetLastError());
    plan->last_launches = pl.last_launches;
  });
}

int shiro_spmm_host(shiro_plan_t plan, const float *B_host, float *C_host, void *stream) {
  return guarded([&] {
    if (!plan || plan->loopback || plan->view) throw Error(SHIRO_E_ARG, "not a distributed plan");
    Plan &pl = *plan->single;
    if (!pl.arena) throw Error(SHIRO_E_ARG, "plan was built with SHIRO_F_HOST_ONLY");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)pl.M * pl.N * sizeof(float);
    if (!pl.stage && bytes) SHIRO_CK(cudaMalloc(&pl.stage, 2 * bytes));   // once per plan
    float *dB = pl.stage, *dC = pl.stage ? pl.stage + (size_t)pl.M * pl.N : nullptr;
    if (bytes) SHIRO_CK(cudaMemcpyAsync(dB, B_host, bytes, cudaMemcpyHostToDevice, s));
    run_step(pl, dB, dC, s);
    if (bytes) SHIRO_CK(cudaMemcpyAsync(C_host, dC, bytes, cudaMemcpyDeviceToHost, s));
    SHIRO_CK(cudaStreamSynchronize(s));
    if (pl.err_host && *pl.err_host)
      throw Error(SHIRO_E_PEER, "fused exchange: a peer did not signal in time (C is invalid)");
    plan->last_launches = pl.last_launches;
  });
}

int shiro_spmm_host_batch(shiro_plan_t plan, int64_t nb, const float *const *B_host,
                          float *const *C_host, void *stream) {
  return guarded([&] {
    if (!plan || plan->loopback || plan->view) throw Error(SHIRO_E_ARG, "not a distributed plan");
    if (nb < 0 || (nb > 0 && (!B_host || !C_host))) throw Error(SHIRO_E_ARG, "bad batch");
    Plan &pl = *plan->single;
    if (!pl.arena) throw Error(SHIRO_E_ARG, "plan was built with SHIRO_F_HOST_ONLY");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)pl.M * pl.N * sizeof(float);
    if (!pl.stage2 && bytes) SHIRO_CK(cudaMalloc(&pl.stage2, 4 * bytes));   // two slots of B, C
    if (!pl.h2d_s) {
      SHIRO_CK(cudaStreamCreateWithFlags(&pl.h2d_s, cudaStreamNonBlocking));
      SHIRO_CK(cudaStreamCreateWithFlags(&pl.d2h_s, cudaStreamNonBlocking));
      for (int k = 0; k < 2; ++k)
        for (cudaEvent_t *e : {&pl.ev_in[k], &pl.ev_comp[k], &pl.ev_out[k]})
          SHIRO_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    const size_t elems = (size_t)pl.M * pl.N;
    auto dB = [&](int k) { return pl.stage2 ? pl.stage2 + (2 * k) * elems : nullptr; };
    auto dC = [&](int k) { return pl.stage2 ? pl.stage2 + (2 * k + 1) * elems : nullptr; };
    // Double-buffered pipeline over the batch: item i uses slot k = i mod 2.
    // The upload of B[i] waits only for SpMM i-2 (the last reader of slot k),
    // so it overlaps SpMM i-1; SpMM i waits for its upload and for the
    // download of C[i-2] (the last reader of dC[k]); the download of C[i]
    // overlaps SpMM i+1 and the upload of B[i+2] (PCIe is full duplex).
    // Steady state per item: max(H2D, SpMM, D2H) instead of their sum.
    for (int k = 0; k < 2; ++k) {
      SHIRO_CK(cudaEventRecord(pl.ev_comp[k], s));
      SHIRO_CK(cudaEventRecord(pl.ev_out[k], s));
    }
    int64_t launches = 0;
    for (int64_t i = 0; i < nb; ++i) {
      const int k = (int)(i & 1);
      SHIRO_CK(cudaStreamWaitEvent(pl.h2d_s, pl.ev_comp[k], 0));
      if (bytes) SHIRO_CK(cudaMemcpyAsync(dB(k), B_host[i], bytes, cudaMemcpyHostToDevice, pl.h2d_s));
      SHIRO_CK(cudaEventRecord(pl.ev_in[k], pl.h2d_s));
      SHIRO_CK(cudaStreamWaitEvent(s, pl.ev_in[k], 0));
      SHIRO_CK(cudaStreamWaitEvent(s, pl.ev_out[k], 0));
      run_step(pl, dB(k), dC(k), s);
      launches += pl.last_launches;
      SHIRO_CK(cudaEventRecord(pl.ev_comp[k], s));
      SHIRO_CK(cudaStreamWaitEvent(pl.d2h_s, pl.ev_comp[k], 0));
      if (bytes) SHIRO_CK(cudaMemcpyAsync(C_host[i], dC(k), bytes, cudaMemcpyDeviceToHost, pl.d2h_s));
      SHIRO_CK(cudaEventRecord(pl.ev_out[k], pl.d2h_s));
    }
    for (int k = 0; k < 2; ++k) SHIRO_CK(cudaStreamWaitEvent(s, pl.ev_out[k], 0));
    SHIRO_CK(cudaStreamSynchronize(s));
    if (pl.err_host && *pl.err_host)
      throw Error(SHIRO_E_PEER, "fused exchange: a peer did not signal in time (C is invalid)");
    plan->last_launches = launches;
  });
}

int shiro_spmm_loopback(shiro_plan_t plan, const float *B, float *C, void *stream) {
  return guarded([&] {
    if (!plan || !plan->loopback) throw Error(SHIRO_E_ARG, "not a loopback plan");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int P = (int)plan->ranks.size();
    int64_t launches = 0;
    for (auto &p : plan->ranks)
      if (!p->arena) throw Error(SHIRO_E_ARG, "plan was built with SHIRO_F_HOST_ONLY");
    const int N = plan->ranks[0]->N;
    auto Bp = [&](int r) { return B + plan->ranks[r]->part[r] * N; };
    auto Cp = [&](int r) { return C + plan->ranks[r]->part[r] * N; };
    if (P == 1) {
      launches += stage_local(*plan->ranks[0], Bp(0), Cp(0), s);
    } else if (plan->ranks[0]->route.active) {
      for (int r = 0; r < P; ++r) {
        Plan &pl = *plan->ranks[r];
        launches += run_spmm(pl.d_prod, Bp(r), pl.M, nullptr, Cp(r), false, s);   // Stage I + K1
      }
      for (int r = 0; r < P; ++r) launches += hier_stage(*plan->ranks[r], 2, Bp(r), Cp(r), s);
      for (int r = 0; r < P; ++r) launches += hier_stage(*plan->ranks[r], 3, Bp(r), Cp(r), s);
    } else if (plan->ranks[0]->p2p) {
      // fused producer launches (peer rows), then each rank's local SpMM and
      // receives
      for (int r = 0; r < P; ++r) {
        Plan &pl = *plan->ranks[r];
        launches += run_spmm(pl.d_prod, Bp(r), pl.M, nullptr, Cp(r), false, s);
      }
      for (int r = 0; r < P; ++r) {
        Plan &pl = *plan->ranks[r];
        if (pl.merged) {   // two-phase consumer over [B_local || receive buffer]
          launches += run_spmm(pl.d_cx, Bp(r), pl.M, pl.recv_buf, Cp(r), false, s);
        } else {
          launches += stage_local(pl, Bp(r), Cp(r), s);
          launches += stage_recv(pl, Cp(r), s);
        }
      }
    } else {
      for (int r = 0; r < P; ++r) launches += stage_send(*plan->ranks[r], Bp(r), s);
      // exchange: device copies send(s -> r) into recv(r from s)
      for (int r = 0; r < P; ++r) {
        Plan &dst = *plan->ranks[r];
        for (int src = 0; src < P; ++src) {
          if (src == r) continue;
          Plan &sp = *plan->ranks[src];
          const int64_t rows = sp.send_off[r + 1] - sp.send_off[r];
          if (rows != dst.recv_off[src + 1] - dst.recv_off[src])
            throw Error(SHIRO_E_INTERNAL, "loopback segment size mismatch");
          if (rows)
            SHIRO_CK(cudaMemcpyAsync(dst.recv_buf + dst.recv_off[src] * N,
                                     sp.send_buf + sp.send_off[r] * N,
                                     (size_t)rows * N * sizeof(float), cudaMemcpyDeviceToDevice, s));
        }
      }
      for (int r = 0; r < P; ++r) {
        launches += stage_local(*plan->ranks[r], Bp(r), Cp(r), s);
        launches += stage_recv(*plan->ranks[r], Cp(r), s);
      }
    }
    SHIRO_CK(cudaGetLastError());
    plan->last_launches = launches;
  });
}

int shiro_free(shiro_plan_t plan) {
  return guarded([&] {
    if (!plan) return;
    if (plan->view) throw Error(SHIRO_E_ARG, "cannot free a borrowed rank view");
    delete plan;
  });
}

int shiro_plan_info(shiro_plan_t plan, shiro_info_t *out) {
  return guarded([&] {
    if (!plan || !out) throw Error(SHIRO_E_ARG, "NULL argument");
    if (plan->loopback) {
      *out = plan->ranks[0]->info;
      int64_t dev = 0;
      for (auto &p : plan->ranks) dev += p->info.dev_bytes;
      out->dev_bytes = dev;
      return;
    }
    *out = plan->rank_plan().info;
  });
}

int shiro_plan_list(shiro_plan_t plan, int32_t peer, int32_t kind, int64_t *buf, int64_t cap,
                    int64_t *len) {
  return guarded([&] {
    if (!plan || !len) throw Error(SHIRO_E_ARG, "NULL argument");
    if (plan->loopback && !plan->view) throw Error(SHIRO_E_ARG, "use shiro_plan_rank first");
    Plan &pl = plan->rank_plan();
    if (peer < 0 || peer >= pl.P) throw Error(SHIRO_E_ARG, "peer out of range");
    const std::vector<int64_t> *v = nullptr;
    switch (kind) {
      case SHIRO_LIST_SEND_B: v = &pl.send_b[peer]; break;
      case SHIRO_LIST_SEND_C: v = &pl.send_c[peer]; break;
      case SHIRO_LIST_RECV_B: v = &pl.recv_b[peer]; break;
      case SHIRO_LIST_RECV_C: v = &pl.recv_c[peer]; break;
      case SHIRO_LIST_H1_SEND: case SHIRO_LIST_H2_SEND:
      case SHIRO_LIST_H1_RECV: case SHIRO_LIST_H2_RECV: {
        if (!pl.route.active) throw Error(SHIRO_E_ARG, "not a hierarchical plan");
        const int st = (kind == SHIRO_LIST_H1_SEND || kind == SHIRO_LIST_H1_RECV) ? 0 : 1;
        const bool snd = kind == SHIRO_LIST_H1_SEND || kind == SHIRO_LIST_H2_SEND;
        v = snd ? &pl.route.h_send[st][peer] : &pl.route.h_recv[st][peer];
        break;
      }
      default: throw Error(SHIRO_E_ARG, "unknown list kind");
    }
    *len = (int64_t)v->size();
    if (buf) std::memcpy(buf, v->data(), sizeof(int64_t) * std::min<int64_t>(cap, *len));
  });
}

int shiro_profile(shiro_plan_t plan, int32_t enable) {
  return guarded([&] {
    if (!plan || plan->loopback || plan->view) throw Error(SHIRO_E_ARG, "not a distributed plan");
    Plan &pl = *plan->single;
    if (enable && !pl.prof[0])
      for (auto &e : pl.prof) SHIRO_CK(cudaEventCreate(&e));
    pl.prof_on = enable != 0;
    pl.prof_used = 0;
  });
}

int shiro_stage_times(shiro_plan_t plan, double *ms) {
  return guarded([&] {
    if (!plan || !ms || plan->loopback || plan->view) throw Error(SHIRO_E_ARG, "bad argument");
    Plan &pl = *plan->single;
    for (int i = 0; i < SHIRO_NUM_STAGES; ++i) ms[i] = 0.0;
    if (!pl.prof_on || !pl.prof_used) throw Error(SHIRO_E_ARG, "no profiled call");
    auto el = [&](int a, int b) {
      float t = 0.f;
      SHIRO_CK(cudaEventSynchronize(pl.prof[b]));
      SHIRO_CK(cudaEventElapsedTime(&t, pl.prof[a], pl.prof[b]));
      return (double)t;
    };
    if (pl.prof_used == 1) {
      ms[SHIRO_STAGE_LOCAL] = ms[SHIRO_STAGE_TOTAL] = el(5, 6);
      return;
    }
    if (pl.prof_used == 4) {   // hierarchical: LOCAL = Stage I + K1 launch, PARTIAL = Stage II
      ms[SHIRO_STAGE_LOCAL] = el(0, 1);
      ms[SHIRO_STAGE_PACK] = el(1, 2);
      ms[SHIRO_STAGE_EXCHANGE] = el(2, 3) + el(4, 5);
      ms[SHIRO_STAGE_PARTIAL] = el(3, 4);
      ms[SHIRO_STAGE_REMOTE] = el(5, 6);
      ms[SHIRO_STAGE_TOTAL] = el(0, 6);
      return;
    }
    if (pl.prof_used == 5) {
      // two-phase consumer (SHIRO_CX=1): PARTIAL = producer (K4 + K3 ->
      // peers), EXCHANGE = its READY signal, LOCAL = CX stage 1 (every K1
      // part plus the K2 + K5 parts already READY; concurrent with the
      // producer, from the step's start), REMOTE = stage 2 (deferred units)
      ms[SHIRO_STAGE_PARTIAL] = el(0, 1);
      ms[SHIRO_STAGE_EXCHANGE] = el(1, 2);
      ms[SHIRO_STAGE_LOCAL] = el(0, 3);
      ms[SHIRO_STAGE_REMOTE] = el(3, 4);
      ms[SHIRO_STAGE_TOTAL] = el(0, 5);
      return;
    }
    if (pl.prof_used == 3) {
      // fused exchange, the same schedule as the timed (graph) step:
      // PARTIAL = the producer launch (K4 pack + K3 partials -> peers, on the
      // high-priority branch), EXCHANGE = its READY signal, LOCAL = K1
      // (concurrent with the producer), REMOTE = the consumer from the end of
      // K1, including its per-source waits
      ms[SHIRO_STAGE_PARTIAL] = el(0, 1);
      ms[SHIRO_STAGE_EXCHANGE] = el(1, 2);
      ms[SHIRO_STAGE_LOCAL] = el(0, 3);
      ms[SHIRO_STAGE_REMOTE] = el(3, 4);
      ms[SHIRO_STAGE_TOTAL] = el(0, 5);
      return;
    }
    ms[SHIRO_STAGE_PACK] = el(0, 1);
    ms[SHIRO_STAGE_PARTIAL] = el(1, 2);
    ms[SHIRO_STAGE_EXCHANGE] = el(3, 4);
    ms[SHIRO_STAGE_LOCAL] = el(5, 6);
    if (pl.flags & SHIRO_F_NO_OVERLAP) {
      ms[SHIRO_STAGE_REMOTE] = el(6, 7);
    } else {
      // remote starts when both the local SpMM and the exchange are done
      const double t_local_end = el(0, 6), t_x_end = el(0, 4);
      ms[SHIRO_STAGE_REMOTE] = el(0, 7) - std::max(t_local_end, t_x_end);
    }
    ms[SHIRO_STAGE_SCATTER] = el(7, 8);
    ms[SHIRO_STAGE_TOTAL] = el(0, 8);
  });
}

int64_t shiro_last_launches(shiro_plan_t plan) { return plan ? plan->last_launches : -1; }

}  // extern "C"
