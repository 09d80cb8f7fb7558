/*
 * shiro.h -- C ABI of the B200-native SHIRO distributed SpMM hot path.
 *
 * Computes C = A * B (section II-A) with A an n x n sparse
 * matrix in CSR form and B, C dense n x N fp32 matrices, all 1D
 * row-partitioned over P processes (section II-B): process p
 * owns rows part[p] .. part[p+1]-1 of A, B and C; the columns of A use the
 * same boundaries.
 *
 *  shiro_plan   -- the offline phase (workflow steps 1-2):
 *                  per off-diagonal block A^(p,q) a minimum vertex cover of the
 *                  bipartite row/column graph (L315-375) decides, per nonzero,
 *                  whether q sends B rows (column-based) or computes and sends
 *                  partial C rows (row-based); the row-based part of A^(p,q) is
 *                  shipped to q once (L300).  Reused by every shiro_spmm
 *                  (L300, L375).
 *  shiro_spmm   -- one SpMM (workflow steps 3-5, L301-303): pack B rows and
 *                  compute partial C rows into the send buffer, all-to-allv
 *                  exchange over NVLink (NCCL), local SpMM overlapped with the
 *                  exchange, remote SpMM on the received B rows, scatter-add of
 *                  the received partial C rows.  With group_size > 1 the
 *                  hierarchical two-stage schedule of Algorithm 1 (L542-574).
 *
 * Conventions: block A^(p,q) = rows owned by p x columns owned by q; p
 * receives, q sends (R5).  All list ids are GLOBAL row ids.
 *
 * Errors: every call returns SHIRO_OK (0) or a positive shiro_status; the
 * message of the last failure on the calling thread is shiro_last_error().
 * shiro_plan agrees on the validation status across ranks before any payload
 * exchange, so a bad input on one rank fails every rank (no hang).
 *
 * Threads: a plan may be used by one thread at a time; one shiro_spmm in
 * flight per plan (internal buffers are reused).
 */
#ifndef SHIRO_H
#define SHIRO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct shiro_plan_s *shiro_plan_t;

enum shiro_status {
  SHIRO_OK = 0,
  SHIRO_E_ARG = 1,      /* bad n, N, P, group size, rank or NULL pointer        */
  SHIRO_E_CSR = 2,      /* row_ptr not monotone, column out of range, unsorted
                           or duplicate columns within a row      */
  SHIRO_E_PART = 3,     /* invalid partition vector            */
  SHIRO_E_CUDA = 4,     /* CUDA runtime error                                   */
  SHIRO_E_NCCL = 5,     /* NCCL error (also asynchronous errors, next call)     */
  SHIRO_E_OOM = 6,      /* device or host allocation failed                     */
  SHIRO_E_INTERNAL = 7, /* infeasible cover or broken invariant  */
  SHIRO_E_PEER = 8,     /* another rank reported an error during shiro_plan     */
  SHIRO_E_TRANSPORT = 9 /* the caller's host transport callback failed          */
};

/* flags (bitwise or) */
#define SHIRO_F_COVER_ROWMAX 0u       /* canonical cut = s-reachable set (R1)    */
#define SHIRO_F_COVER_COLMAX (1u << 0) /* canonical cut = t-side (R1)           */
#define SHIRO_F_MODE_JOINT 0u          /* joint row/column   */
#define SHIRO_F_MODE_COL (1u << 1)     /* column-based only (Eq. 2)    */
#define SHIRO_F_MODE_ROW (1u << 2)     /* row-based only (Eq. 3)       */
#define SHIRO_F_SPLIT_RECV (1u << 3)   /* remote SpMM (K2) and scatter-add (K5) as
                                          two launches; default: one fused pass  */
#define SHIRO_F_HOST_ONLY (1u << 4)    /* plan lists/stats only, no device state */
#define SHIRO_F_NO_OVERLAP (1u << 5)   /* local SpMM after the exchange (ablation)*/
#define SHIRO_F_MODE_BLOCK (1u << 7)   /* sparsity-oblivious: whole B row block
                                          per non-empty A^(p,q) (Eq. 1) */
#define SHIRO_F_COVER_BALANCE (1u << 9) /* joint mode: a block whose all-rows
                                           cover is within max(1, mu/1000) rows
                                           of the minimum mu is covered by all
                                           its rows (column owner computes it),
                                           balancing dense-ish blocks across
                                           ranks (R18)               */
#define SHIRO_F_TRANSPOSE (1u << 8)    /* plan and run A^T (GNN backward, SURVEY
                                          8(f) N3): the caller still passes its
                                          rows of A; one distributed transpose at
                                          plan time                              */
#define SHIRO_F_XCHG_NCCL (1u << 6)    /* exchange with NCCL grouped send/recv
                                          instead of the default fused exchange
                                          (K4/K3 store straight into the peers'
                                          receive buffers over NVLink, CUDA IPC) */

/* list kinds for shiro_plan_list */
#define SHIRO_LIST_SEND_B 0 /* B rows this rank sends to `peer` (global ids)     */
#define SHIRO_LIST_SEND_C 1 /* C rows this rank computes partials of for `peer`  */
#define SHIRO_LIST_RECV_B 2 /* B rows this rank receives from `peer`             */
#define SHIRO_LIST_RECV_C 3 /* C rows of this rank `peer` sends partials of      */
/* hierarchical schedule (group_size > 1), per stage s in {1,2}: rows this rank
 * sends to `peer` in that stage, B-row ids first then C-row ids, each section
 * ascending and, for C rows, grouped by final destination ascending.        */
#define SHIRO_LIST_H1_SEND 4
#define SHIRO_LIST_H2_SEND 5
#define SHIRO_LIST_H1_RECV 6
#define SHIRO_LIST_H2_RECV 7

/*
 * Host transport for the plan-time exchange (optional).  A collective
 * all-to-allv of bytes: segment for peer d is send + sum(send_bytes[0..d-1]),
 * send_bytes[d] long; likewise for recv (recv_bytes is known to the caller
 * from a previous call with 8-byte segments).  Must return 0 on success.
 */
typedef int (*shiro_alltoallv_fn)(void *ctx, const void *send, const int64_t *send_bytes,
                                  void *recv, const int64_t *recv_bytes);

typedef struct {
  int32_t rank;       /* this rank, 0 <= rank < nranks                          */
  int32_t nranks;     /* P, 1..64                                               */
  int32_t group_size; /* 1 = flat; g > 1 = hierarchical groups of g ranks
                         (contiguous, must divide nranks)                        */
  uint32_t flags;     /* SHIRO_F_*                                              */
  const void *nccl_id; /* 128-byte ncclUniqueId from shiro_get_unique_id on rank
                         0, identical on all ranks; may be NULL if
                         nranks == 1, or if host_xchg != NULL and either
                         SHIRO_F_HOST_ONLY is set or the fused NVLink
                         exchange is used (no NCCL communicator is created;
                         shiro_plan fails with SHIRO_E_ARG on every rank if
                         the peer mappings cannot be set up)              */
  shiro_alltoallv_fn host_xchg; /* optional plan-time transport (e.g. gloo);
                                   NULL = use NCCL                              */
  void *host_xchg_ctx;
} shiro_dist_t;

typedef struct {
  int32_t rank, nranks, group_size, N;
  int64_t n, m_local, nnz_local;
  /* nonzeros of this rank's rows by role, and row-based nnz received */
  int64_t nnz_diag, nnz_colbased, nnz_rowbased_shipped, nnz_rowbased_computed;
  /* per-iteration rows this rank sends / receives (flat plan) */
  int64_t send_b_rows, send_c_rows, recv_b_rows, recv_c_rows;
  /* global totals over all ranks (identical on every rank), in rows */
  int64_t g_joint_rows;     /* sum of mu over blocks (Eq. 10)                    */
  int64_t g_col_rows;       /* sum |Cols| (Eq. 2)                                */
  int64_t g_row_rows;       /* sum |Rows| (Eq. 3)                                */
  int64_t g_block_rows;     /* sum over non-empty blocks of K_q (Eq. 1)          */
  int64_t g_oblivious_rows; /* (P-1) * n, all-gather of B (R6)         */
  int64_t g_setup_bytes;    /* row-based nnz * 8, one-time (R14)                 */
  int64_t g_flat_inter_rows;/* flat rows crossing group boundaries               */
  int64_t g_hier_inter_rows, g_hier_intra_rows; /* hierarchical schedule (g > 1) */
  int64_t g_max_send_rows, g_max_recv_rows;     /* per-rank maxima (flat)         */
  int64_t dev_bytes;        /* device memory owned by this plan                  */
  double plan_seconds;      /* wall time of shiro_plan on this rank              */
  /* per device op of one shiro_spmm (index SHIRO_OP_*): nonzeros (or gathered
   * rows), output rows and distinct source rows read -- the algorithmic
   * traffic of each kernel launch */
  int64_t op_nnz[5], op_rows[5], op_src_rows[5];
  double refresh_seconds;   /* wall time of the last value refresh (0 if none)   */
} shiro_info_t;
#define SHIRO_OP_LOCAL 0   /* K1: A_diag * B_local             */
#define SHIRO_OP_PARTIAL 1 /* K3: A_out * B_local -> send_buf   */
#define SHIRO_OP_REMOTE 2  /* K2 (or fused K2+K5) over recv_buf */
#define SHIRO_OP_SCATTER 3 /* K5: partial rows -> C             */
#define SHIRO_OP_PACK 4    /* K4: B rows -> send_buf            */

/* Fill a 128-byte buffer with a fresh ncclUniqueId (call on rank 0 only). */
int shiro_get_unique_id(void *id128);

/*
 * Build a plan.  Collective over all ranks (every rank must call it).
 *   n        global rows (= global cols), n >= 0
 *   part     host int64[P+1], 0 = part[0] <= ... <= part[P] = n
 *   row_ptr  host int64[M_p+1] for this rank's rows part[p]..part[p+1]-1,
 *            row_ptr[0] = 0, non-decreasing
 *   col_idx  host int32[nnz_p], GLOBAL column ids, strictly increasing per row
 *   val      host float[nnz_p]
 *   N        dense width, 1 <= N <= 4096
 *   stream   cudaStream_t used for the uploads (ignored with HOST_ONLY)
 * Host arrays are read during the call only (copied).  The plan binds to the
 * CUDA device current at the call.  On failure *out = NULL.
 */
int shiro_plan(const shiro_dist_t *d, int64_t n, const int64_t *part, const int64_t *row_ptr,
               const int32_t *col_idx, const float *val, int32_t N, void *stream,
               shiro_plan_t *out);

/*
 * Weighted covers (Eqs. 4-8, and the weighted network of
 * L372-375): as shiro_plan, but block covers minimise
 *     sum_{selected C rows i} w_row[i] + sum_{selected B rows j} w_col[j]
 * instead of the row count (exact minimum s-t cut by Dinic's algorithm; the
 * canonical s-reachable read-off of DESIGN.md R1 applies unchanged).
 *   w_row  host int64[M_p]: cost of communicating a partial C row of each of
 *          this rank's rows (local row index), every used entry > 0
 *   w_col  host int64[n]:   cost of communicating B row j (global id), > 0;
 *          entries of columns this rank's rows do not reference are unused
 * With SHIRO_F_TRANSPOSE the weights refer to the planned matrix A^T.
 * Weights only affect joint-mode covers (ignored by SHIRO_F_MODE_*).
 * Errors: as shiro_plan; SHIRO_E_ARG if a weight pointer is NULL or a used
 * weight is <= 0 (detected while planning the block on that rank).
 */
int shiro_plan_weighted(const shiro_dist_t *d, int64_t n, const int64_t *part,
                        const int64_t *row_ptr, const int32_t *col_idx, const float *val, int32_t N,
                        const int64_t *w_row, const int64_t *w_col, void *stream,
                        shiro_plan_t *out);

/*
 * Value refresh for a fixed sparsity pattern (the plan "can be
 * reused across multiple SpMM operations with the same sparsity pattern";
 * SURVEY 8(f) N3).  Collective.  `val` holds the new values of this rank's
 * nonzeros, in the order of the col_idx array given to shiro_plan (same
 * row_ptr / col_idx pattern).  The cover, lists and device layouts are kept;
 * each rank re-ships only the values of its row-based nonzeros (4 B each, one
 * all-to-allv over the plan's transport) and rewrites the values of its
 * device operations in place.  Returns after the device copy is updated
 * (synchronous on `stream`); the next shiro_spmm uses the new values.
 * row_ptr / col_idx: only read for SHIRO_F_TRANSPOSE plans (the values are
 * redistributed like the plan-time transpose), may be NULL otherwise.
 * A plan built with a host transport (host_xchg) keeps using it here: the
 * callback and its context must stay valid for the plan's lifetime.
 * Errors: SHIRO_E_ARG (loopback or HOST_ONLY plan, NULL val), SHIRO_E_NCCL /
 * SHIRO_E_TRANSPORT (exchange), SHIRO_E_CUDA.
 */
int shiro_plan_update_values(shiro_plan_t plan, const int64_t *row_ptr, const int32_t *col_idx,
                             const float *val, void *stream);

/*
 * One distributed SpMM: C_p = A^(p,:) * B.  Collective, stream-ordered,
 * asynchronous.  B_p: device fp32 [M_p x N] row-major, read-only until the
 * stream passes this call.  C_p: device fp32 [M_p x N], fully overwritten.
 * Both 16-byte aligned.  A peer that fails to signal within the timeout
 * (SHIRO_P2P_TIMEOUT_MS, default 20 s) is reported by the NEXT call on this
 * plan (SHIRO_E_PEER), since this call returns before the device runs; the
 * host-buffer calls below synchronise and report it themselves.
 */
int shiro_spmm(shiro_plan_t plan, const float *B_p, float *C_p, void *stream);

/* Same as shiro_spmm with HOST buffers: copies B_p host->device, runs the
 * SpMM and copies C_p device->host; returns after C_p is on the host.
 * Pinned host memory gives full PCIe bandwidth. */
int shiro_spmm_host(shiro_plan_t plan, const float *B_host, float *C_host, void *stream);

/* A batch of nb independent SpMMs with the same plan (e.g. feature blocks or
 * GNN layers), HOST buffers: item i reads B_host[i] ([M_p x N] fp32) and
 * writes C_host[i] ([M_p x N] fp32).  Collective: every rank passes the same
 * nb.  Uploads, SpMMs and downloads are pipelined over the batch with two
 * device slots of B and C owned by the plan (4 x M_p x N x 4 bytes): the
 * upload of item i+1 and the download of item i-1 overlap the SpMM of item i
 * (full-duplex PCIe), so an item costs max(H2D, SpMM, D2H) in steady state.  `stream` orders the SpMMs;
 * returns after every C_host[i] is written.  B_host/C_host are arrays of nb
 * host pointers (pinned memory for full bandwidth); nb = 0 is a no-op.
 * Errors: SHIRO_E_ARG (NULL arrays with nb > 0, negative nb, loopback or
 * HOST_ONLY plan), SHIRO_E_CUDA. */
int shiro_spmm_host_batch(shiro_plan_t plan, int64_t nb, const float *const *B_host,
                          float *const *C_host, void *stream);

/* Release the plan (local, not collective).  NULL is a no-op. */
int shiro_free(shiro_plan_t plan);

/* Statistics of the plan (see shiro_info_t). */
int shiro_plan_info(shiro_plan_t plan, shiro_info_t *out);

/* Copy one index list (global ids) into buf[0..cap); *len = its full length.
 * buf may be NULL with cap = 0 to query the length. */
int shiro_plan_list(shiro_plan_t plan, int32_t peer, int32_t kind, int64_t *buf, int64_t cap,
                    int64_t *len);

/* Thread-local message of the last failure ("" if none). */
const char *shiro_last_error(void);

/*
 * Loopback: all P virtual ranks in ONE process on ONE device; the exchange is
 * a set of device-to-device copies.  Same planner, lists and kernels as the
 * distributed path (development / single-GPU tests).  row_ptr/col_idx/val
 * hold the FULL matrix (n rows).  shiro_spmm_loopback takes B and C as full
 * device matrices [n x N]; virtual rank r reads/writes rows part[r]..
 */
int shiro_plan_loopback(int32_t nranks, int32_t group_size, uint32_t flags, int64_t n,
                        const int64_t *part, const int64_t *row_ptr, const int32_t *col_idx,
                        const float *val, int32_t N, void *stream, shiro_plan_t *out);
int shiro_spmm_loopback(shiro_plan_t plan, const float *B, float *C, void *stream);
/* Loopback variants of shiro_plan_weighted (w_row: int64[n], all rows) and
 * shiro_plan_update_values (val: the full matrix's new values, same order as
 * the col_idx given to shiro_plan_loopback). */
int shiro_plan_loopback_weighted(int32_t nranks, int32_t group_size, uint32_t flags, int64_t n,
                                 const int64_t *part, const int64_t *row_ptr,
                                 const int32_t *col_idx, const float *val, int32_t N,
                                 const int64_t *w_row, const int64_t *w_col, void *stream,
                                 shiro_plan_t *out);
int shiro_plan_update_values_loopback(shiro_plan_t plan, const float *val, void *stream);
/* Borrowed view of virtual rank r of a loopback plan (do not free). */
int shiro_plan_rank(shiro_plan_t plan, int32_t r, shiro_plan_t *out);

/* Stage timing (CUDA events recorded on the stream each stage runs on).
 * After shiro_profile(plan, 1), every shiro_spmm records events around each
 * stage; shiro_stage_times waits for the last call and writes the durations
 * in milliseconds, indexed by SHIRO_STAGE_* (0 for stages that did not run).
 * Distributed plans only. */
#define SHIRO_STAGE_PACK 0     /* E1: K4 pack of B rows (NCCL exchange)        */
#define SHIRO_STAGE_PARTIAL 1  /* E2: K3 row-based partial SpMM; fused exchange:
                                  the producer launch (K4 + K3 -> peers)       */
#define SHIRO_STAGE_EXCHANGE 2 /* E3: NCCL all-to-allv (communication stream);
                                  fused exchange: the READY signal             */
#define SHIRO_STAGE_LOCAL 3    /* E4: K1 local SpMM (fused exchange: measured
                                  from the step's start, concurrent with the
                                  producer)                                    */
#define SHIRO_STAGE_REMOTE 4   /* E5: K2 (or fused K2+K5) remote SpMM, incl. its
                                  per-source waits                             */
#define SHIRO_STAGE_SCATTER 5  /* E6: K5 scatter-add                           */
#define SHIRO_STAGE_TOTAL 6    /* first event to last event                    */
#define SHIRO_NUM_STAGES 7
int shiro_profile(shiro_plan_t plan, int32_t enable);
int shiro_stage_times(shiro_plan_t plan, double *ms /* [SHIRO_NUM_STAGES] */);

/* Measurement probe (not on the hot path): out[c] = sum of the rows
 * X[idx[k]] over chunks c of `chunk` consecutive indices (out: ceil(n/chunk)
 * x N).  Device pointers; N in {32, 64, 128}.  Timing it on an SpMM's own
 * column-index stream gives that SpMM's gather-aware roofline. */
int shiro_probe_gather(const float *X, int32_t N, const int32_t *idx, int64_t n_idx, float *out,
                       int32_t chunk, void *stream);

/* TMA variant of the probe (measurement only): the same sums with the rows
 * staged into shared memory by cp.async.bulk.tensor tile::gather4 (4 rows per
 * instruction) through a `stages`-deep ring per warp (stages in {2, 4, 8}).
 * X: device [x_rows x N] fp32, N = 128 only; chunk a multiple of 4.
 * Errors: SHIRO_E_ARG (shape), SHIRO_E_CUDA (no tensor-map entry point,
 * launch failure). */
int shiro_probe_gather_tma(const float *X, int64_t x_rows, int32_t N, const int32_t *idx,
                           int64_t n_idx, float *out, int32_t chunk, int32_t stages, void *stream);

/* Warp-specialized TMA variant (measurement only): `ctas` CTAs of 9 warps
 * (1 producer lane issuing tile::gather4 into a `stages`-deep ring of 2 KB
 * stages, 8 consumer warps), each CTA a contiguous range of the index
 * stream.  out: device float[ctas * 8 * 128], one float4 sum per consumer
 * lane (the total over `out` equals the sum of all gathered rows).  N = 128,
 * n_idx a positive multiple of 4, stages in {8, 16, 24}.
 * Errors: SHIRO_E_ARG (shape), SHIRO_E_CUDA. */
int shiro_probe_gather_tma_ws(const float *X, int64_t x_rows, int32_t N, const int32_t *idx,
                              int64_t n_idx, float *out, int32_t stages, int32_t ctas,
                              void *stream);

/* Roofline denominators (measurement only, SURVEY 8(d) microbenchmarks):
 * shiro_probe_fma: `blocks` x 256 threads, each 8 independent FMA chains x 4
 *   FMAs x `iters` (2 flops each); out: device float[blocks * 256].
 *   FLOP = blocks * 256 * iters * 64.
 * shiro_probe_copy: y[0..n) = x[0..n) with float4 loads/stores (n % 4 == 0,
 *   16-byte aligned device buffers); bytes moved = 8 * n.
 * Errors: SHIRO_E_ARG, SHIRO_E_CUDA (launch). */
int shiro_probe_fma(float *out, int32_t blocks, int32_t iters, void *stream);
int shiro_probe_copy(const float *x, float *y, int64_t n_floats, void *stream);

/* Number of kernel launches the last shiro_spmm* issued on this plan (all
 * virtual ranks for loopback), NCCL kernels excluded. */
int64_t shiro_last_launches(shiro_plan_t plan);

#ifdef __cplusplus
}
#endif
#endif /* SHIRO_H */
