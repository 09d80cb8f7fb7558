// p2p_host.cpp -- setup of the fused NVLink exchange (collective, plan time).
//
// Every rank exports its plan arena (receive buffer + flags) with
// cudaIpcGetMemHandle and sends to each peer the handle, the byte offsets of
// its receive buffer and flags inside the arena, and the row offset at which
// that peer's rows land in its receive buffer (recv_off).  Each rank then
// opens the peers' arenas and precomputes, for every row it sends, the
// peer-mapped destination address: K4 (pack) and K3 (row-based partial SpMM)
// store straight into the receivers' buffers over NVLink -- the exchange is
// fused into the producing kernels (workflow steps 3-4).
// If any rank fails to map a peer, every rank keeps the NCCL exchange.
#include <climits>
#include <cstring>

#include "shiro_internal.h"

namespace shiro {

namespace {

struct PeerMsg {
  cudaIpcMemHandle_t handle;
  int64_t recv_buf_off, flags_off, recv_row_off, recv_buf2_off;
};

template <typename T>
std::vector<char> bytes_of(const T &x) {
  std::vector<char> b(sizeof(T));
  std::memcpy(b.data(), &x, sizeof(T));
  return b;
}

}  // namespace

void p2p_release(Plan &pl) {
  for (void *b : pl.peer_base)
    if (b) cudaIpcCloseMemHandle(b);
  pl.peer_base.clear();
  if (pl.p2p_arena) cudaFree(pl.p2p_arena);
  pl.p2p_arena = nullptr;
  if (pl.prod_ops) cudaFree(pl.prod_ops);
  pl.prod_ops = nullptr;
  if (pl.err_host) cudaFreeHost(pl.err_host);
  pl.err_host = nullptr;
  if (pl.s_hi) cudaStreamDestroy(pl.s_hi);
  if (pl.ev_fork) cudaEventDestroy(pl.ev_fork);
  if (pl.ev_join) cudaEventDestroy(pl.ev_join);
  pl.s_hi = nullptr;
  pl.ev_fork = pl.ev_join = nullptr;
  pl.p2p = false;
}

void p2p_setup(Plan &pl, const Alltoallv &xchg) {
  const int P = pl.P, me = pl.rank;
  const int64_t rowb = (int64_t)pl.N * sizeof(float);
  // 1. export
  cudaIpcMemHandle_t h;
  int status = cudaIpcGetMemHandle(&h, pl.arena) == cudaSuccess ? 0 : 1;
  std::vector<std::vector<char>> send(P), recv;
  for (int d = 0; d < P; ++d) {
    PeerMsg m{h, pl.recv_buf_off, pl.flags_off, pl.recv_off[d], pl.recv_buf2_off};
    send[d] = bytes_of(m);
  }
  xchg(send, recv);
  // 2. open the peers' arenas
  pl.peer_base.assign(P, nullptr);
  std::vector<PeerMsg> pm(P);
  for (int d = 0; d < P && status == 0; ++d) {
    if (d == me) continue;
    if (recv[d].size() != sizeof(PeerMsg)) { status = 1; break; }
    std::memcpy(&pm[d], recv[d].data(), sizeof(PeerMsg));
    void *base = nullptr;
    if (cudaIpcOpenMemHandle(&base, pm[d].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      status = 1;
      break;
    }
    pl.peer_base[d] = base;
  }
  // 3. agree: all ranks use the fused exchange or none does
  std::vector<std::vector<char>> st_send(P, bytes_of(status)), st_recv;
  xchg(st_send, st_recv);
  int any = status;
  for (int d = 0; d < P; ++d)
    if (d != me && st_recv[d].size() == sizeof(int)) {
      int v;
      std::memcpy(&v, st_recv[d].data(), sizeof(int));
      any |= v;
    }
  if (any) {
    p2p_release(pl);
    return;   // NCCL exchange stays in place
  }
  // 4. destination addresses of every row this rank sends
  auto peer_recv = [&](int d) {
    return reinterpret_cast<char *>(pl.peer_base[d]) + pm[d].recv_buf_off;
  };
  // double buffering needs a second receive buffer on every rank; each rank
  // sees every peer's choice (recv_buf2_off < 0 = none), so all ranks agree
  // on the protocol even if SHIRO_DBUF differs between them
  bool dbuf = pl.recv_buf2_off >= 0;
  for (int d = 0; d < P; ++d)
    if (d != me && pm[d].recv_buf2_off < 0) dbuf = false;
  std::vector<uint64_t> dstp, outp, dstp2, outp2, rdy, cons;
  for (int d = 0; d < P; ++d) {
    if (d == me) continue;
    char *base = peer_recv(d) + pm[d].recv_row_off * rowb;
    char *base2 = dbuf ? reinterpret_cast<char *>(pl.peer_base[d]) + pm[d].recv_buf2_off +
                             pm[d].recv_row_off * rowb
                       : nullptr;
    for (size_t k = 0; k < pl.send_b[d].size(); ++k) {
      dstp.push_back((uint64_t)(base + (int64_t)k * rowb));
      if (dbuf) dstp2.push_back((uint64_t)(base2 + (int64_t)k * rowb));
    }
    const int64_t nb = (int64_t)pl.send_b[d].size();
    for (size_t k = 0; k < pl.send_c[d].size(); ++k) {
      outp.push_back((uint64_t)(base + (nb + (int64_t)k) * rowb));
      if (dbuf) outp2.push_back((uint64_t)(base2 + (nb + (int64_t)k) * rowb));
    }
    char *fl = reinterpret_cast<char *>(pl.peer_base[d]) + pm[d].flags_off;
    rdy.push_back((uint64_t)(fl + sizeof(int32_t) * me));
    cons.push_back((uint64_t)(fl + sizeof(int32_t) * (P + me)));
  }
  if ((int64_t)outp.size() != pl.d_out.a.nrows || (int64_t)dstp.size() != pl.d_pack.n)
    throw Error(SHIRO_E_INTERNAL, "fused exchange: row count mismatch");
  // K4 + K3 as one pointer-routed launch (one destination table per buffer)
  if (dbuf) upload_prod(pl, pl.pack_src, dstp, outp, false, &dstp2, &outp2);
  else upload_prod(pl, pl.pack_src, dstp, outp, false);
  pl.dbuf = dbuf;
  pl.step_parity = 0;
  const size_t n_all = rdy.size() + cons.size();
  SHIRO_CK(cudaMalloc(&pl.p2p_arena, std::max<size_t>(1, n_all) * sizeof(uint64_t)));
  uint64_t *a = static_cast<uint64_t *>(pl.p2p_arena);
  std::vector<uint64_t> all;
  all.insert(all.end(), rdy.begin(), rdy.end());
  all.insert(all.end(), cons.begin(), cons.end());
  if (!all.empty())
    SHIRO_CK(cudaMemcpy(a, all.data(), all.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  pl.ready_ptrs = reinterpret_cast<int32_t *const *>(a);
  pl.consumed_ptrs = reinterpret_cast<int32_t *const *>(a + rdy.size());
  // 5. local flags: own entries never block (INT_MAX), the rest start at 0
  std::vector<int32_t> f(2 * P + 4, 0);
  f[me] = INT_MAX;
  f[P + me] = INT_MAX;
  SHIRO_CK(cudaMemcpy(pl.xflags, f.data(), f.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  SHIRO_CK(cudaMallocHost(&pl.err_host, sizeof(int32_t)));
  *pl.err_host = 0;
  if (const char *e = getenv("SHIRO_P2P_TIMEOUT_MS")) pl.wait_timeout_ns = atoll(e) * 1000000LL;
  pl.epoch = 0;
  // the producer branch of a step runs on the highest-priority stream:
  // pending producer CTAs are dispatched before the consumer's (whose warps
  // may spin on a late peer), so a consumer can never starve its own GPU's
  // producer
  int lo_prio = 0, hi_prio = 0;
  SHIRO_CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  SHIRO_CK(cudaStreamCreateWithPriority(&pl.s_hi, cudaStreamNonBlocking, hi_prio));
  if (merged_enabled(pl)) upload_merged(pl);
  SHIRO_CK(cudaEventCreateWithFlags(&pl.ev_fork, cudaEventDisableTiming));
  SHIRO_CK(cudaEventCreateWithFlags(&pl.ev_join, cudaEventDisableTiming));
  pl.p2p = true;
  // every rank's flags are initialised before any peer signals into them
  std::vector<std::vector<char>> bar_send(P, bytes_of(0)), bar_recv;
  SHIRO_CK(cudaDeviceSynchronize());
  xchg(bar_send, bar_recv);
}

}  // namespace shiro

namespace shiro {

// ---------------------------------------------------------------------------
// Hierarchical routing over NVLink: export the route arena (R1 || R2, flags),
// exchange (handle, offsets of R1/R2/flags, and where the receiver placed
// each sender's R1 and R2 segments), map the peers, resolve destinations.
// ---------------------------------------------------------------------------
namespace {
struct HierMsg {
  cudaIpcMemHandle_t handle;
  int64_t rb_off, flags_off, r1_rows, seg1, seg2;
};
}  // namespace

void hier_release(Plan &pl) {
  Route &R = pl.route;
  for (void *b : R.peer_base)
    if (b) cudaIpcCloseMemHandle(b);
  R.peer_base.clear();
  if (R.ptrs) cudaFree(R.ptrs);
  if (R.ops) cudaFree(R.ops);
  if (R.arena) cudaFree(R.arena);
  R.ptrs = R.ops = R.arena = nullptr;
}

void hier_p2p_setup(Plan &pl, const Alltoallv &xchg) {
  Route &R = pl.route;
  const int P = pl.P, me = pl.rank;
  cudaIpcMemHandle_t h;
  int status = cudaIpcGetMemHandle(&h, R.arena) == cudaSuccess ? 0 : 1;
  std::vector<std::vector<char>> send(P), recv;
  for (int d = 0; d < P; ++d) {
    HierMsg m{h, R.rb_off, R.flags_off, R.r1_rows, R.r1_off[d], R.r2_off[d]};
    send[d] = bytes_of(m);
  }
  xchg(send, recv);
  R.peer_base.assign(P, nullptr);
  std::vector<HierMsg> hm(P);
  for (int d = 0; d < P && status == 0; ++d) {
    if (d == me) continue;
    if (recv[d].size() != sizeof(HierMsg)) { status = 1; break; }
    std::memcpy(&hm[d], recv[d].data(), sizeof(HierMsg));
    void *base = nullptr;
    if (cudaIpcOpenMemHandle(&base, hm[d].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      status = 1;
      break;
    }
    R.peer_base[d] = base;
  }
  std::vector<std::vector<char>> st_send(P, bytes_of(status)), st_recv;
  xchg(st_send, st_recv);
  int any = status;
  for (int d = 0; d < P; ++d)
    if (d != me && st_recv[d].size() == sizeof(int)) {
      int v;
      std::memcpy(&v, st_recv[d].data(), sizeof(int));
      any |= v;
    }
  if (any) throw Error(SHIRO_E_CUDA, "hierarchical mode needs CUDA IPC peer mappings");
  const int64_t rowb = (int64_t)pl.N * sizeof(float);
  hm[me] = HierMsg{h, R.rb_off, R.flags_off, R.r1_rows, R.r1_off[me], R.r2_off[me]};
  auto seg = [&](int d, int buf) -> char * {
    char *base = (d == me) ? static_cast<char *>(R.arena) : static_cast<char *>(R.peer_base[d]);
    const int64_t row = (buf == 0) ? hm[d].seg1 : hm[d].r1_rows + hm[d].seg2;
    return base + hm[d].rb_off + row * rowb;
  };
  auto flag = [&](int d, int i) -> int32_t * {
    char *base = (d == me) ? static_cast<char *>(R.arena) : static_cast<char *>(R.peer_base[d]);
    return reinterpret_cast<int32_t *>(base + hm[d].flags_off) + i;
  };
  hier_resolve(pl, seg, flag);
  SHIRO_CK(cudaMallocHost(&pl.err_host, sizeof(int32_t)));
  *pl.err_host = 0;
  if (const char *e = getenv("SHIRO_P2P_TIMEOUT_MS")) pl.wait_timeout_ns = atoll(e) * 1000000LL;
  pl.epoch = 0;
  std::vector<std::vector<char>> bar_send(P, bytes_of(0)), bar_recv;
  SHIRO_CK(cudaDeviceSynchronize());
  xchg(bar_send, bar_recv);
}

}  // namespace shiro
