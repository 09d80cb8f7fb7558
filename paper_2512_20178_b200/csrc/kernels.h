// kernels.h -- internal launch interface of the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace shiro {

// One CSR SpMM launch (K1/K2/K3 of DESIGN.md):
//   Y[out_row[t]] (+)= sum_{k in [rp[t], rp[t+1])} val[k] * X(col[k])
// with X(c) = X0[c] for c < n0 and X1[c - n0] otherwise (unified source row
// space, e.g. [B_local || receive buffer]).  out_row == nullptr means
// out_row[t] = t.  Rows with more than L nonzeros are split into chunk tasks
// (power-law hub rows); the chunk partials are reduced in a fixed order by the
// last-arriving chunk, so the result is deterministic.  All other rows are
// packed into row groups of at most ~L nonzeros (plan time); one lane group
// streams a whole group, so the gathers of consecutive short rows are in
// flight together.
// A row group: consecutive short rows [r0, r1) whose nonzeros are [k0, k1).
// Two-phase ops (the fused-exchange consumer) store the group's phase-A
// nonzeros (every row's local part, row order) in [k0, kmid) and its phase-B
// nonzeros (every row's remote part, row order) in [kmid, k1); kmid = k1
// otherwise.
struct RowGroup {
  int64_t k0, k1, kmid;
  int32_t r0, r1;
};

// Bit 31 of a column id in `cv` marks a "hot" source row (one of the most
// referenced rows of the op, chosen at plan time): with the hot/cold L2
// policy its gathers are L2 evict_last and the other gathers evict_first.
constexpr int32_t kHotBit = (int32_t)0x80000000u;

struct SpmmArgs {
  int64_t nrows = 0;
  const int64_t *rp = nullptr;          // [nrows+1]
  const int2 *cv = nullptr;             // [nnz] interleaved (column [| kHotBit], value bits)
  const uint8_t *roff = nullptr;        // [nnz] row offset inside its row group
  const int32_t *out_row = nullptr;
  float *const *out_ptr = nullptr;      // per-row output address (fused exchange)
  const float *X0 = nullptr;
  int64_t n0 = 0;
  const float *X1 = nullptr;
  float *Y = nullptr;
  int32_t N = 0;
  int32_t L = 0x7fffffff;               // long-row threshold = chunk size
  int32_t n_groups = 0;
  const RowGroup *groups = nullptr;     // [n_groups]
  int32_t n_tasks = 0;                  // chunk tasks (long rows)
  const int32_t *task_long = nullptr;   // [n_tasks] long-row index of each task
  const int32_t *long_row = nullptr;    // [n_long] CSR row t of each long row
  const int32_t *long_first = nullptr;  // [n_long+1] first task of each long row
  int32_t *long_counter = nullptr;      // [n_long] zero-initialised arrival counters
  float *scratch = nullptr;             // [n_tasks * N] chunk partials
  int32_t hot = 0;                      // 1: cv carries kHotBit marks (hot/cold L2 policy);
                                        // 2: X1 is the op's compact hot buffer
  // Two-phase op (fused-exchange consumer CX): each row's nonzeros are its
  // local part (columns < n0, source X0 = B_local) then its remote part
  // (columns >= n0, X1 = receive buffer); long_mid[l] = first remote nonzero
  // of long row l.  A unit computes its local parts, then waits for the
  // sources of its remote parts (when `ready` is set), then adds them.
  const int64_t *long_mid = nullptr;
  // Per-source wait (fused exchange consumer): unit u reads
  // receive-buffer rows of the sources in unit_src[u] (bit s = source rank
  // s); before it, its warp spins until ready[s] >= *wait_epoch + 1 for
  // those sources only (ld.acquire.sys), so rows of a peer are consumed as
  // soon as that peer's READY lands.  Source rows are then read with
  // L2-coherent loads (the buffer is written by peers during the launch).
  // A timeout (per warp, %globaltimer) or an error raised by any other warp
  // sets / sees *wait_err and skips the unit instead of hanging the GPU.
  // *wait_epoch is only read (target = *wait_epoch + 1); the step-end barrier
  // (READY from every peer) and the epoch advance are the following k_wait
  // launch.  ready == nullptr: off.  With ready the
  // launch must be a two-phase overwrite with two sources [X0 = B_local ||
  // X1 = receive buffer]; only X1 rows use coherent loads.
  const int32_t *ready = nullptr;       // [P] local READY flags (one per source)
  const uint64_t *unit_src = nullptr;   // [n_tasks + n_groups] source masks
  int32_t *wait_epoch = nullptr;
  int32_t *wait_err = nullptr;
  // two-phase consumer: launch stage (1 = concurrent first launch that defers
  // units whose sources are not READY yet, 2 = their continuation), the
  // deferred-unit list [n_tasks + n_groups], its length and a work counter
  // (all zero-initialised; re-armed by a memset after stage 2)
  int32_t cx_stage = 0;
  int32_t *defer_list = nullptr;
  int32_t *defer_n = nullptr;
  int32_t *work_ctr = nullptr;
  int64_t wait_timeout_ns = 0;
};

// accumulate: false -> Y = A*X (overwrite, empty rows get zeros); true -> Y += A*X
// returns the number of kernel launches issued (0 if nothing to do)
int launch_spmm(const SpmmArgs &a, bool accumulate, cudaStream_t s);

// K4: Y[dst[i]] = X[src[i]] for i < n (gather B rows into the send buffer)
int launch_pack(int64_t n, const int32_t *src, const int32_t *dst, const float *X, float *Y,
                int32_t N, cudaStream_t s);

// K4 into peer memory: dstp[i] is the (peer-mapped) address of packed row i
int launch_pack_ptr(int64_t n, const int32_t *src, float *const *dstp, const float *X, int32_t N,
                    cudaStream_t s);

// Fused-exchange synchronisation over NVLink (p2p.cu), value = *epoch + add
// read on the device.  signal: for each i, st.release.sys *flags[i] = value
// (flags[i] may be a peer address); bump: then *epoch = value.  wait: spin
// until every local flags[i] >= value (ld.acquire.sys); after timeout_ns (or
// as soon as *err is set by another waiter) sets *err = 1 and gives up
// instead of hanging the GPU.
int launch_signal(int32_t *const *flags, int n, int32_t *epoch, int add, bool bump,
                  cudaStream_t s);
int launch_wait(const int32_t *flags, int n, int32_t *epoch, int add, int32_t *err,
                int64_t timeout_ns, cudaStream_t s, bool bump = false);   // bump: *epoch = value after the wait

// K5: C[tgt[u]] += sum_{k in [ptr[u], ptr[u+1])} R[src[k]] (gather-sum of
// received partial C rows, fixed order: C first, then sources ascending)
int launch_scatter_add(int64_t nt, const int32_t *tgt, const int64_t *ptr, const int32_t *src,
                       const float *R, float *C, int32_t N, cudaStream_t s);

// N3 value refresh: cv[k].y = bits(V[vsrc[k]]) for every k < nnz with
// vsrc[k] >= 0 (a fixed pattern's device op takes new values in place).
int launch_refresh(int64_t nnz, const int32_t *vsrc, const float *V, int2 *cv, cudaStream_t s);

// SM count of the current device (cached)
int num_sms();

// vector shape of width N for the pack / scatter kernels: LPR lanes per row,
// VPL float4 per lane; false -> generic (scalar) path
bool vec_shape(int N, int *lpr, int *vpl);
// SpMM lane shape: LPR lanes per output row, W floats per lane load (1, 2, 4),
// VPL loads per lane; N = 32 / 64 use one 32-lane group per warp
bool spmm_vec_shape(int N, int *lpr, int *w, int *vpl);

}  // namespace shiro
