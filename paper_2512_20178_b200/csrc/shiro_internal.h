// shiro_internal.h -- host-side structures of the planner and executor.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../../include/shiro.h"
#include "kernels.h"

namespace shiro {

struct Error {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
};

#define SHIRO_CK(x)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw ::shiro::Error(e_ == cudaErrorMemoryAllocation ? SHIRO_E_OOM : SHIRO_E_CUDA, \
                           std::string(#x) + ": " + cudaGetErrorString(e_));             \
  } while (0)

#define SHIRO_NCK(x)                                                                     \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess)                                                               \
      throw ::shiro::Error(SHIRO_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// canonical block cover (cover.cpp); returns mu
int64_t block_cover(int32_t nr, int32_t nc, const std::vector<int64_t> &ap,
                    const std::vector<int32_t> &adj, bool colmax, std::vector<uint8_t> &sel_row,
                    std::vector<uint8_t> &sel_col);


// weighted canonical block cover (cover.cpp): exact minimum
// weight cover by max flow on the paper's network
int64_t block_cover_weighted(int32_t nr, int32_t nc, const std::vector<int64_t> &ap,
                             const std::vector<int32_t> &adj, const std::vector<int64_t> &w_row,
                             const std::vector<int64_t> &w_col, bool colmax,
                             std::vector<uint8_t> &sel_row, std::vector<uint8_t> &sel_col);

// Host CSR of one SpMM op.  out_row empty = identity.
struct HostCsr {
  int64_t nrows = 0;
  std::vector<int64_t> rp{0};
  std::vector<int32_t> col;
  std::vector<float> val;       // empty = all ones
  std::vector<int32_t> vsrc;    // per nonzero: index into the plan's value space, -1 = unit
                                // weight (value refresh, N3); empty = no refresh entries
  std::vector<int32_t> out_row;
  bool ptr_rows = false;        // rows addressed by per-row output pointers
  std::vector<int64_t> src_bounds;   // non-empty: source s owns columns
                                     // [src_bounds[s], src_bounds[s+1]) -> per-unit masks
  int64_t hot_rows = -1;        // >= 0: number of source rows (hot/cold L2 marks)
  std::vector<int32_t> mid;     // two-phase op: per row, the number of leading
                                // (local-part) nonzeros; empty = one phase
  int64_t nnz() const { return (int64_t)col.size(); }
};

// Device image of a SpMM op (arrays live in the plan's arena)
// Device image of a gather (pack) or gather-sum (scatter) op
struct DevPack {
  int64_t n = 0;
  const int32_t *src = nullptr, *dst = nullptr;
};
struct DevSpmm {
  SpmmArgs a;            // pointers to device arrays; X/Y filled at run time
  int64_t nnz = 0;
  const int32_t *vsrc = nullptr;   // refresh map (nnz entries) or nullptr
  DevPack hot;                     // compact hot buffer: rows of X0 copied each step
  float *hot_buf = nullptr;        // ... into this buffer, read as X1 (columns >= hot_base)
  int64_t hot_base = 0;
};
struct DevScatter {
  int64_t nt = 0;
  const int32_t *tgt = nullptr;
  const int64_t *ptr = nullptr;
  const int32_t *src = nullptr;
  int64_t nsrc = 0;
};

// Destination of a produced row in the hierarchical routing: the segment of
// the sending rank inside buffer `buf` (0 = R1, 1 = R2) of rank `rank`.
struct Dest {
  int32_t rank, buf;
  int64_t pos;
};

// Hierarchical (two-stage) routing of one rank (hier.cpp).
struct Route {
  bool active = false;
  int64_t r1_rows = 0, r2_rows = 0;
  std::vector<int64_t> r1_off, r2_off;                 // segment offset per source (rows)
  std::vector<std::vector<int64_t>> h_send[2], h_recv[2];
  // Stage I producers (read B_local)
  std::vector<int32_t> s1_pack_src;
  std::vector<Dest> s1_pack_dst;
  HostCsr s1_part;
  std::vector<Dest> s1_part_dst;
  // Stage II producers (read own R1)
  std::vector<int32_t> s2_fwd_src;
  std::vector<Dest> s2_fwd_dst;
  HostCsr s2_agg;
  std::vector<Dest> s2_agg_dst;
  // final remote SpMM over [R1 || R2]
  HostCsr fin;
  // device state
  void *arena = nullptr;           // R1 || R2 and flags (IPC-exported)
  float *rb = nullptr;
  int32_t *xflags = nullptr;       // ready1[P], ready2[P], consumed[P], err
  int64_t rb_off = 0, flags_off = 0;
  void *ops = nullptr;             // op arrays
  void *ptrs = nullptr;            // resolved destination pointers
  DevSpmm d_part, d_agg, d_fin;
  DevPack d_pack1, d_fwd;
  float *const *pack1_dstp = nullptr, *const *fwd_dstp = nullptr;
  int32_t *const *ready1_ptrs = nullptr, *const *ready2_ptrs = nullptr,
          *const *consumed_ptrs = nullptr;
  std::vector<void *> peer_base;   // opened IPC mappings
};

// Plan-time transport: collective all-to-allv of host byte segments.
using Alltoallv = std::function<void(const std::vector<std::vector<char>> &send,
                                     std::vector<std::vector<char>> &recv)>;

struct Plan {
  // identity
  int32_t rank = 0, P = 1, g = 1;
  uint32_t flags = 0;
  int64_t n = 0;
  int32_t N = 0;
  std::vector<int64_t> part;
  int64_t M = 0;            // local rows (= local B rows)
  int device = 0;
  bool loopback_view = false;

  // lists, global ids ascending, indexed by peer
  std::vector<std::vector<int64_t>> send_b, send_c, recv_b, recv_c;
  std::vector<int64_t> send_off, recv_off;   // rows, [P+1]
  int64_t send_rows = 0, recv_rows = 0;

  // hierarchical routing (group_size > 1)
  Route route;

  // host images of the ops
  HostCsr A_diag, A_out, A_col, A_rem;
  std::vector<int32_t> pack_src, pack_dst;
  std::vector<int32_t> sc_tgt, sc_src;
  std::vector<int64_t> sc_ptr{0};

  // stats
  shiro_info_t info{};
  int64_t loc_cols = 0, loc_rows = 0, loc_block = 0, loc_setup = 0;   // owned blocks

  // device state
  void *arena = nullptr;
  size_t arena_bytes = 0;
  float *send_buf = nullptr, *recv_buf = nullptr;
  float *recv_buf2 = nullptr;         // second receive buffer (double-buffered fused exchange)
  DevSpmm d_diag, d_out, d_col, d_rem;
  DevPack d_pack;
  DevScatter d_scatter;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_recvd = nullptr;
  ncclComm_t comm = nullptr;
  int64_t last_launches = 0;
  // stage profiling (shiro_profile)
  bool prof_on = false;
  cudaEvent_t prof[12] = {};
  int prof_used = 0;
  // fused NVLink exchange (CUDA IPC peer mappings, p2p_host.cpp)
  bool p2p = false;
  int32_t epoch = 0;
  // local flags: ready[P], consumed[P], err, ep_sig, ep_wait, done_ctr
  int32_t *xflags = nullptr;
  int64_t recv_buf_off = 0, flags_off = 0, recv_buf2_off = -1;
  // double buffering: step parity selects the receive buffer peers write
  // (and the producer's destination table); no CONSUMED round trip
  bool dbuf = false;
  int step_parity = 0;
  float *const *prod_out_ptr[2] = {nullptr, nullptr};
  std::vector<void *> peer_base;      // opened IPC mappings
  void *p2p_arena = nullptr;
  int32_t *const *ready_ptrs = nullptr, *const *consumed_ptrs = nullptr;
  // fused producer launch: pack rows (unit weight) + row-based partials, both
  // stored into peers' receive buffers (K4+K3); hierarchical Stage I also
  // carries the local rows into C (K1)
  DevSpmm d_prod;
  void *prod_ops = nullptr;
  // two-phase consumer of the fused exchange (default, "CX"): every local row
  // from [B_local || receive buffer]; per work unit its local parts (K1)
  // first, then -- after the READY of the sources it reads -- its remote
  // parts (K2 + K5), so K1 overlaps the producer and each peer's rows are
  // consumed as they land
  bool merged = false;
  DevSpmm d_cx;
  void *merged_ops = nullptr;
  cudaStream_t s_hi = nullptr;        // producer branch of a step (high priority)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int32_t *err_host = nullptr;        // pinned copy of the error flag
  int64_t wait_timeout_ns = 20000000000LL;
  // CUDA graph of one step (P = 1, fused exchange, hierarchical), keyed by
  // (B, C, stream, profiling); replayed while the key matches
  struct GraphSlot {
    int parity = -1;
    cudaGraphExec_t exec = nullptr;
    const float *B = nullptr;
    float *C = nullptr;
    cudaStream_t s = nullptr;
    bool prof = false;
    int64_t launches = 0;
  } graphs[4];                        // keyed by (step parity, B, C, stream): both
                                      // parities x both host-batch staging slots
  int graph_next = 0;                 // round-robin replacement
  // device staging of B and C for shiro_spmm_host (stage) and the
  // double-buffered shiro_spmm_host_batch (stage2: two slots of B and C)
  float *stage = nullptr, *stage2 = nullptr;
  cudaStream_t h2d_s = nullptr, d2h_s = nullptr;   // copy engines of the batch pipeline
  cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
  // value refresh (N3): value space V = [local values || row-based values
  // received from each peer, peers ascending]; every device op's nonzeros
  // map into it (vsrc)
  int64_t nnz_local = 0, nnz_recv_vals = 0;
  std::vector<std::vector<int64_t>> ship_idx;   // per q: local nonzeros shipped to q (message order)
  std::vector<int64_t> recv_vals;               // per peer: row-based values received (count)
  std::vector<int64_t> tperm;                   // transposed plans: local entry -> received index
  std::vector<DevSpmm *> refresh_ops;           // device ops carrying values
  float *vspace = nullptr;                      // device value space (first refresh)
  Alltoallv refresh_xchg;                       // transport for the refresh exchange
  double refresh_seconds = 0.0;

  ~Plan();
};

struct PlanInput {
  int32_t rank, P, g;
  uint32_t flags;
  int64_t n;
  const int64_t *part;
  const int64_t *row_ptr;   // this rank's rows
  const int32_t *col;
  const float *val;
  int32_t N;
  const int64_t *w_row = nullptr;   // weighted covers (N2): [M_p] cost of this rank's C rows
  const int64_t *w_col = nullptr;   //   [n] cost of every B row (global ids)
};

// planner phases (plan.cpp)
void validate_input(const PlanInput &in);
// phase 1: covers of the owned blocks -> outgoing messages per peer
struct Phase1 {
  std::vector<std::vector<char>> out;             // message to each peer
  std::vector<int8_t> tag;                        // per local nonzero: 0 local, 1 row, 2 col
  std::vector<std::vector<int64_t>> recv_b, recv_c;   // what each q sends us
  std::vector<int64_t> n_rows, n_cols, nnz_row;       // per q: |Rows|, |Cols| of A^(p,q)
  std::vector<std::vector<int64_t>> ship_idx;         // per q: row-based nonzeros, message order
};
Phase1 plan_phase1(const PlanInput &in);
void plan_phase2(const PlanInput &in, Phase1 &p1, const std::vector<std::vector<char>> &in_msgs,
                 Plan &plan);
// global statistics (needs one more all-to-allv)
void plan_stats(const PlanInput &in, Plan &plan, const Alltoallv &xchg);
// device upload
void plan_upload(Plan &plan, cudaStream_t s);

// hierarchical routing (hier.cpp, runtime.cpp, p2p_host.cpp)
std::vector<std::vector<char>> hier_meta_messages(const Plan &pl);
void hier_build(const PlanInput &in, const Phase1 &p1, Plan &pl,
                const std::vector<std::vector<char>> &meta);
void hier_upload(Plan &pl);
// resolve destinations: seg(d, buf) = address of THIS rank's segment in
// buffer buf of rank d; flag(d, i) = address of flag i of rank d
void hier_resolve(Plan &pl, const std::function<char *(int, int)> &seg,
                  const std::function<int32_t *(int, int)> &flag);
void hier_p2p_setup(Plan &pl, const Alltoallv &xchg);
void hier_release(Plan &pl);
void exec_hier(Plan &pl, const float *B, float *C, cudaStream_t s);
int64_t hier_stage(Plan &pl, int stage, const float *B, float *C, cudaStream_t s);

// executor (runtime.cpp)
void exec_flat(Plan &plan, const float *B, float *C, cudaStream_t s);
// fused NVLink exchange (p2p_host.cpp): IPC setup (collective) and executor
void p2p_setup(Plan &plan, const Alltoallv &xchg);
// build + upload the fused producer op; pack_addr / part_addr are the
// destination addresses of the packed B rows and of the A_out rows
void upload_prod(Plan &plan, const std::vector<int32_t> &pack_src,
                 const std::vector<uint64_t> &pack_addr, const std::vector<uint64_t> &part_addr,
                 bool with_local, const std::vector<uint64_t> *pack_addr2 = nullptr,
                 const std::vector<uint64_t> *part_addr2 = nullptr);
// value refresh of a plan's device ops from the new value space V (host)
void refresh_device(Plan &plan, const std::vector<float> &V, cudaStream_t s);
void plan_drop_host(Plan &plan);
// build + upload the two-phase consumer (CX) of the fused exchange
void upload_merged(Plan &plan);
bool merged_enabled(const Plan &plan);
void p2p_release(Plan &plan);
void exec_p2p(Plan &plan, const float *B, float *C, cudaStream_t s);
bool dbuf_enabled();   // SHIRO_DBUF (default on): double-buffered fused exchange
void exec_plan(Plan &plan, const float *B, float *C, cudaStream_t s);

}  // namespace shiro

namespace shiro {
// distributed transpose for SHIRO_F_TRANSPOSE (plan.cpp)
std::vector<std::vector<char>> transpose_messages(const PlanInput &in);
void transpose_assemble(const PlanInput &in, const std::vector<std::vector<char>> &msgs,
                        std::vector<int64_t> &rp, std::vector<int32_t> &col,
                        std::vector<float> &val, std::vector<int64_t> *perm = nullptr);
// value refresh exchange (plan.cpp): new values of this rank's nonzeros ->
// the plan's value space (transposed plans first redistribute the values)
std::vector<float> refresh_value_space(Plan &plan, const PlanInput &in, const float *val,
                                       const Alltoallv &xchg);
// its two halves (loopback runs the exchange in process): the row-based values
// this rank ships to each peer, and V from the local values + received ones
std::vector<std::vector<char>> refresh_ship(const Plan &plan, const float *lv);
std::vector<float> refresh_assemble(const Plan &plan, const float *lv,
                                    const std::vector<std::vector<char>> &rcv);
}  // namespace shiro
