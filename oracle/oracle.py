"""Plain CPU oracle for SHIRO's joint row/column plan and its execution.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Nothing in the product
package imports this module; the product must fail loudly without its CUDA
library instead of falling back here.

Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
R<n> = reading n in DESIGN.md ("Readings of the paper").

Conventions (R5): block A^(p,q) = rows owned by p x columns owned by
q, p != q.  p owns the rows and *receives*; q owns B rows Cols(A^(p,q)) and
*sends*.  Lists are keyed (sender, receiver) = (q, p).

Parity status: every function here is pinned by tests/test_oracle_*.py
against paper-fixed facts (worked examples, closed forms, brute force,
invariants).  There is no "parity unpinned" function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC_PATH = os.path.join(_HERE, "oracle_core.c")
_lib = None

ROW, COL, LOCAL = 1, 2, 0


def build_oracle_lib(force: bool = False) -> str:
    """Compile oracle_core.c with gcc (plain C, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC_PATH)):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC",
                               _SRC_PATH, "-o", _LIB_PATH])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build_oracle_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.oracle_spmm_f64.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, P,
                                        ctypes.c_int64, P, P]
        lib.oracle_spmm_f64.restype = None
        lib.oracle_dinic_cover.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                           P, P, P, P, ctypes.c_int32, P, P, P]
        lib.oracle_dinic_cover.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


# --------------------------------------------------------------------------
# Partition
# --------------------------------------------------------------------------
def uniform_partition(n: int, P: int) -> np.ndarray:
    """Contiguous 1D row partition, sizes ceil/floor(n/P), larger blocks first
    (S:101).  Columns use the same boundaries (R8)."""
    if P < 1:
        raise ValueError("P must be >= 1")
    base, extra = divmod(n, P)
    sizes = [base + (1 if p < extra else 0) for p in range(P)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def owner_of(part: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """Process owning global row/col id (block p owns [part[p], part[p+1]))."""
    return (np.searchsorted(part, ids, side="right") - 1).astype(np.int64)


# --------------------------------------------------------------------------
# Dense product by its plain definition
# --------------------------------------------------------------------------
def spmm_ref(row_ptr, col, val, B, rows=None) -> np.ndarray:
    """C[r,:] = sum_k a_rk * B[k,:], fp64 accumulation in ascending column
    order within each row.  ``rows`` optionally selects CSR rows."""
    lib = _load()
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    N = B.shape[1]
    if rows is None:
        nr = row_ptr.shape[0] - 1
        rsel = None
    else:
        rsel = np.ascontiguousarray(rows, dtype=np.int64)
        nr = rsel.shape[0]
    C = np.empty((nr, N), dtype=np.float64)
    if nr:
        lib.oracle_spmm_f64(nr, N, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(B), N,
                            _ptr(rsel), _ptr(C))
    return C


# --------------------------------------------------------------------------
# Minimum weighted vertex cover of one block
# --------------------------------------------------------------------------
def min_cover_local(nr: int, nc: int, er, ec, w_row=None, w_col=None, rule="rowmax"):
    """Cover of the bipartite graph G=(R u C, E) with local vertex ids.

    Solved as the paper's s-t min cut by Dinic in
    oracle_core.c.  rule 'rowmax' reads the cover off the s-reachable set of
    the residual graph; 'colmax' off the t-side (R1).
    Returns (sel_row bool[nr], sel_col bool[nc], flow)."""
    lib = _load()
    er = np.ascontiguousarray(er, dtype=np.int32)
    ec = np.ascontiguousarray(ec, dtype=np.int32)
    w_row = np.ones(nr, np.int64) if w_row is None else np.ascontiguousarray(w_row, np.int64)
    w_col = np.ones(nc, np.int64) if w_col is None else np.ascontiguousarray(w_col, np.int64)
    if (w_row <= 0).any() or (w_col <= 0).any():
        raise ValueError("weights must be positive (S:170)")
    sr = np.zeros(max(nr, 1), np.uint8)
    sc = np.zeros(max(nc, 1), np.uint8)
    flow = ctypes.c_int64(0)
    rc = lib.oracle_dinic_cover(nr, nc, er.shape[0], _ptr(er), _ptr(ec), _ptr(w_row),
                                _ptr(w_col), 0 if rule == "rowmax" else 1,
                                _ptr(sr), _ptr(sc), ctypes.byref(flow))
    if rc != 0:
        raise RuntimeError(f"oracle_dinic_cover failed rc={rc} (S:197 infeasible cover)")
    return sr[:nr].astype(bool), sc[:nc].astype(bool), int(flow.value)


def min_cover(gi, gj, rule="rowmax", w_row=None, w_col=None):
    """Cover of a block given by its edges in global ids.
    Rows = Rows(A^(p,q)), Cols = Cols(A^(p,q)) (Table I).
    Uniform weights unless w_row / w_col (indexed by GLOBAL row / column
    id) give the per-vertex costs w^row_i, w^col_j of Eqs. 4-6.
    Returns (selected rows ascending, selected cols ascending, flow)."""
    rows = np.unique(gi)
    cols = np.unique(gj)
    li = np.searchsorted(rows, gi)
    lj = np.searchsorted(cols, gj)
    wr = None if w_row is None else np.asarray(w_row, np.int64)[rows]
    wc = None if w_col is None else np.asarray(w_col, np.int64)[cols]
    sr, sc, f = min_cover_local(rows.size, cols.size, li, lj, w_row=wr, w_col=wc, rule=rule)
    return rows[sr], cols[sc], f


def brute_force_cover(nr: int, nc: int, edges, w_row=None, w_col=None):
    """Exhaustive minimum weighted vertex cover for tiny blocks.
    Returns (min weight, list of all minimum covers as (rows frozenset,
    cols frozenset))."""
    w = np.array(([1] * nr if w_row is None else list(w_row)) +
                 ([1] * nc if w_col is None else list(w_col)), np.int64)
    nv = nr + nc
    if nv > 22:
        raise ValueError("instance too large for brute force (S:211)")
    masks = np.arange(1 << nv, dtype=np.int64)           # bit v set = vertex v chosen
    bits = (masks[:, None] >> np.arange(nv)) & 1           # [2^nv, nv]
    ok = np.ones(masks.size, bool)
    for i, j in edges:                                      # Eq. 7: x_j + y_i >= a_ij
        ok &= (bits[:, i] | bits[:, nr + j]).astype(bool)
    weight = bits @ w                                       # Eq. 6 objective
    best = int(weight[ok].min())
    covers = []
    for mk in masks[ok & (weight == best)]:
        covers.append((frozenset(i for i in range(nr) if (mk >> i) & 1),
                       frozenset(j for j in range(nc) if (mk >> (nr + j)) & 1)))
    return best, covers


def max_matching_kuhn(nr: int, nc: int, edges) -> int:
    """Maximum bipartite matching by Kuhn's augmenting paths (textbook), an
    algorithm independent of the flow code; König: |max matching| = mu."""
    adj = [[] for _ in range(nr)]
    for i, j in edges:
        adj[i].append(j)
    match_col = [-1] * nc

    def try_row(i, seen):
        for j in adj[i]:
            if j in seen:
                continue
            seen.add(j)
            if match_col[j] < 0 or try_row(match_col[j], seen):
                match_col[j] = i
                return True
        return False

    return sum(1 for i in range(nr) if try_row(i, set()))


# --------------------------------------------------------------------------
# Flat plan (P:299-303 workflow steps 1-2)
# --------------------------------------------------------------------------
@dataclass
class FlatPlan:
    n: int
    part: np.ndarray
    mode: str
    rule: str
    # (sender q, receiver p) -> global ids ascending
    send_b: dict = field(default_factory=dict)   # B rows q sends p (selected cols)
    send_c: dict = field(default_factory=dict)   # C rows q computes for p (selected rows)
    n_cols: dict = field(default_factory=dict)   # |Cols(A^(p,q))| keyed (q, p)
    n_rows: dict = field(default_factory=dict)   # |Rows(A^(p,q))| keyed (q, p)
    nnz_row: dict = field(default_factory=dict)  # row-based nnz of A^(p,q) keyed (q, p)
    tag: np.ndarray = None                       # per stored nonzero: LOCAL/ROW/COL

    @property
    def P(self):
        return self.part.size - 1

    def mu(self, q, p):
        return self.send_b.get((q, p), np.empty(0)).size + self.send_c.get((q, p), np.empty(0)).size


def _row_ids(row_ptr):
    return np.repeat(np.arange(row_ptr.size - 1, dtype=np.int64), np.diff(row_ptr))


def balance_slack(mu):
    """Row slack of the balanced cover rule: max(1, floor(mu / 1000)) (R18)."""
    return max(1, int(mu) // 1000)


def plan_flat(n, part, row_ptr, col, mode="joint", rule="rowmax", balance=False, w_row=None,
              w_col=None) -> FlatPlan:
    """Per ordered pair (p, q), p != q, decide per nonzero ROW vs COL.

    joint: canonical min cover of A^(p,q) (R1); nonzero (i,j) is
      ROW if row i is selected else COL; under 'colmax' COL if col j is
      selected else ROW (R2: doubly covered nonzeros follow the rule side).
    col:   every off-diagonal nonzero COL (Eq. 2).
    row:   every off-diagonal nonzero ROW (Eq. 3).
    block: sparsity-oblivious, q sends its whole B row block to every p with
           a non-empty A^(p,q) (Eq. 1); all nonzeros COL.
    balance (joint only, R18, not from the paper): when the block's
      all-rows cover is within balance_slack(mu) rows of the minimum mu, every
      nonzero of the block is ROW (the column owner q computes the block), so
      dense-ish symmetric blocks are computed by alternating sides instead of
      all on one rank; bytes rise by at most the slack per block.
    w_row, w_col (joint only): per-vertex costs indexed by global row / column
      id (Eqs. 4-6); the block cover is then the minimum-weight
      cover of the weighted network of P:372-375, read off the same way (R1).
    Lists: send_b[(q,p)] = selected cols, send_c[(q,p)] = selected rows,
    global ids ascending."""
    part = np.asarray(part, np.int64)
    row_ptr = np.asarray(row_ptr, np.int64)
    col = np.asarray(col, np.int64)
    gi = _row_ids(row_ptr)
    po = owner_of(part, gi)
    qo = owner_of(part, col)
    plan = FlatPlan(n=n, part=part, mode=mode, rule=rule)
    tag = np.full(col.size, LOCAL, np.int8)
    P = part.size - 1
    pair_key = po * P + qo
    order = np.argsort(pair_key, kind="stable")
    keys_sorted = pair_key[order]
    bounds = np.searchsorted(keys_sorted, np.arange(P * P + 1))
    for p in range(P):
        for q in range(P):
            if p == q:
                continue
            k = p * P + q
            idx = order[bounds[k]:bounds[k + 1]]
            if idx.size == 0:
                continue                      # empty block: no message
            bi, bj = gi[idx], col[idx]
            rows_u, cols_u = np.unique(bi), np.unique(bj)
            plan.n_rows[(q, p)] = rows_u.size
            plan.n_cols[(q, p)] = cols_u.size
            if mode == "joint":
                sel_r, sel_c, mu = min_cover(bi, bj, rule=rule, w_row=w_row, w_col=w_col)
                if rule == "rowmax":
                    is_row = np.isin(bi, sel_r)
                else:
                    is_row = ~np.isin(bj, sel_c)
                if w_row is None:
                    assert sel_r.size + sel_c.size == mu
                else:
                    mu = sel_r.size + sel_c.size        # rows moved, not the cut weight
                if balance and rows_u.size <= mu + balance_slack(mu):
                    is_row = np.ones(idx.size, bool)
            elif mode == "col":
                is_row = np.zeros(idx.size, bool)
            elif mode == "row":
                is_row = np.ones(idx.size, bool)
            elif mode == "block":
                is_row = np.zeros(idx.size, bool)
            else:
                raise ValueError(mode)
            tag[idx] = np.where(is_row, ROW, COL)
            plan.send_c[(q, p)] = np.unique(bi[is_row]).astype(np.int64)
            plan.send_b[(q, p)] = np.unique(bj[~is_row]).astype(np.int64)
            if mode == "block":
                plan.send_b[(q, p)] = np.arange(part[q], part[q + 1], dtype=np.int64)
            plan.nnz_row[(q, p)] = int(is_row.sum())
            if plan.send_c[(q, p)].size == 0:
                del plan.send_c[(q, p)]
            if plan.send_b[(q, p)].size == 0:
                del plan.send_b[(q, p)]
    plan.tag = tag
    return plan


def plan_flat_digests(n, part, row_ptr, col):
    """The joint row-max lists of plan_flat (same steps: P:315-375 cover per
    block, R1 read-off, R2 assignment), streamed one receiving rank p at a
    time for matrices too large to plan at once (c5): returns
    {(q, p): (sha256 of send_b as int64 bytes, sha256 of send_c, |send_b|,
    |send_c|)} for every non-empty block.  Memory ~ the rows of one rank."""
    import hashlib
    part = np.asarray(part, np.int64)
    P = part.size - 1
    out = {}
    for p in range(P):
        lo, hi = int(part[p]), int(part[p + 1])
        k0, k1 = int(row_ptr[lo]), int(row_ptr[hi])
        gi = np.repeat(np.arange(lo, hi, dtype=np.int64), np.diff(row_ptr[lo:hi + 1]))
        gj = np.asarray(col[k0:k1], np.int64)
        qo = owner_of(part, gj)
        order = np.argsort(qo, kind="stable")
        bounds = np.searchsorted(qo[order], np.arange(P + 1))
        for q in range(P):
            if q == p or bounds[q + 1] == bounds[q]:
                continue
            idx = order[bounds[q]:bounds[q + 1]]
            bi, bj = gi[idx], gj[idx]
            sel_r, sel_c, mu = min_cover(bi, bj)
            is_row = np.isin(bi, sel_r)
            send_c = np.unique(bi[is_row]).astype(np.int64)
            send_b = np.unique(bj[~is_row]).astype(np.int64)
            assert send_b.size + send_c.size == mu
            out[(q, p)] = (hashlib.sha256(send_b.tobytes()).hexdigest(),
                           hashlib.sha256(send_c.tobytes()).hexdigest(), send_b.size, send_c.size)
        del gi, gj, qo, order
    return out


def volumes(plan: FlatPlan, N: int, sz: int = 4) -> dict:
    """Volume accounting in rows and bytes (rows * N * sz):
    joint = sum mu (Eq. 10), col = sum |Cols| (Eq. 2),
    row = sum |Rows| (Eq. 3), block = sum over non-empty blocks of K_q
    (Eq. 1), oblivious all-gather = (P-1)*n (north star, R6),
    Red_col / Red_row over summed volumes (Eq. 11).
    setup = row-based nnz * 8 bytes, reported separately (R14)."""
    P, part = plan.P, plan.part
    K = np.diff(part)
    joint = sum(plan.mu(q, p) for (q, p) in plan.n_cols)
    colv = sum(plan.n_cols.values())
    rowv = sum(plan.n_rows.values())
    block = sum(int(K[q]) for (q, p) in plan.n_cols)
    obliv = (P - 1) * plan.n
    pair = np.zeros((P, P), np.int64)
    for (q, p) in plan.n_cols:
        pair[q, p] = plan.mu(q, p)
    rb = lambda r: int(r) * N * sz
    return dict(joint_rows=joint, col_rows=colv, row_rows=rowv, block_rows=block,
                oblivious_rows=obliv, joint_bytes=rb(joint), col_bytes=rb(colv),
                row_bytes=rb(rowv), block_bytes=rb(block), oblivious_bytes=rb(obliv),
                red_col=(1 - joint / colv) if colv else 0.0,
                red_row=(1 - joint / rowv) if rowv else 0.0,
                setup_bytes=8 * sum(plan.nnz_row.values()), pair_rows=pair)


# --------------------------------------------------------------------------
# Hierarchical plan (Alg. 1)
# --------------------------------------------------------------------------
@dataclass
class Msg:
    stage: int          # 1 or 2
    src: int
    dst: int
    kind: str           # 'B' (B rows), 'C' (partials of src), 'CA' (aggregated partials)
    ids: np.ndarray     # global B-row ids ('B') or global C-row ids ('C','CA')
    tier: str           # 'inter' or 'intra'
    final: int = -1     # for 'C' routed to a representative: the destination p
    owner: int = -1     # for 'B' forwarded in stage 2: the owning process q


def rep_col(q: int, G: int, g: int) -> int:
    """Destination-group representative receiving q's deduplicated B rows:
    the member of G with rank = q (mod g) (R12)."""
    return G * g + (q % g)


def rep_row(G: int, p: int, g: int) -> int:
    """Source-group representative aggregating partials for p: the member of
    G with rank = p (mod g) (R12)."""
    return G * g + (p % g)


def plan_hier(plan: FlatPlan, g: int):
    """Stage I = column inter-group fetch || row intra-group aggregation;
    Stage II = row inter-group transmission || column intra-group
    distribution (Alg. 1 and P:582, R13).  Same-group traffic goes directly in
    stage I.  Messages with src == dst are elided."""
    P = plan.P
    if g < 1 or P % g:
        raise ValueError("group size must divide P")
    grp = lambda r: r // g
    ngrp = P // g
    msgs = []
    # Stage I: column inter-group, source aggregation (P:517 step 1-2)
    for q in range(P):
        for G in range(ngrp):
            if G == grp(q):
                continue
            parts = [plan.send_b[(q, p)] for p in range(G * g, G * g + g) if (q, p) in plan.send_b]
            if parts:
                U = np.unique(np.concatenate(parts))
                msgs.append(Msg(1, q, rep_col(q, G, g), "B", U, "inter"))
    # Stage I: row intra-group, partials to the source-group representative (P:519 stage 1)
    for m in range(P):
        for p in range(P):
            if grp(p) == grp(m) or (m, p) not in plan.send_c:
                continue
            r = rep_row(grp(m), p, g)
            if r != m:
                msgs.append(Msg(1, m, r, "C", plan.send_c[(m, p)], "intra", final=p))
    # Stage I: same-group direct traffic (R12)
    for q in range(P):
        for p in range(P):
            if p == q or grp(p) != grp(q):
                continue
            if (q, p) in plan.send_b:
                msgs.append(Msg(1, q, p, "B", plan.send_b[(q, p)], "intra", owner=q))
            if (q, p) in plan.send_c:
                msgs.append(Msg(1, q, p, "C", plan.send_c[(q, p)], "intra", final=p))
    # Stage II: row inter-group transmission of aggregated partials (P:519 stage 2)
    for p in range(P):
        for G in range(ngrp):
            if G == grp(p):
                continue
            parts = [plan.send_c[(m, p)] for m in range(G * g, G * g + g) if (m, p) in plan.send_c]
            if parts:
                V = np.unique(np.concatenate(parts))
                msgs.append(Msg(2, rep_row(G, p, g), p, "CA", V, "inter", final=p))
    # Stage II: column intra-group distribution (P:517 step 3)
    for q in range(P):
        for G in range(ngrp):
            if G == grp(q):
                continue
            r = rep_col(q, G, g)
            for p in range(G * g, G * g + g):
                if p != r and (q, p) in plan.send_b:
                    msgs.append(Msg(2, r, p, "B", plan.send_b[(q, p)], "intra", owner=q))
    return msgs


def tier_traffic(msgs, N: int, sz: int = 4) -> dict:
    """Rows and bytes per tier."""
    inter = sum(m.ids.size for m in msgs if m.tier == "inter")
    intra = sum(m.ids.size for m in msgs if m.tier == "intra")
    return dict(inter_rows=inter, intra_rows=intra, inter_bytes=inter * N * sz,
                intra_bytes=intra * N * sz)


def flat_inter_rows(plan: FlatPlan, g: int) -> int:
    """Inter-group rows of the flat joint plan under grouping g."""
    return sum(plan.mu(q, p) for (q, p) in plan.n_cols if q // g != p // g)


# --------------------------------------------------------------------------
# Execution simulator -- message passing over P virtual ranks
# --------------------------------------------------------------------------
def exec_flat(plan: FlatPlan, row_ptr, col, val, B):
    """Five-stage workflow: q computes partials for its ROW
    nonzeros of A^(p,q) and packs the selected B rows; messages are
    exchanged; p adds local, COL-based remote and received partials, in the
    fixed order local, COL remote by ascending peer, partials by ascending
    peer.  Raises on a missing B row (coverage error)."""
    part = plan.part
    P = plan.P
    row_ptr = np.asarray(row_ptr, np.int64)
    col = np.asarray(col, np.int64)
    B = np.asarray(B)
    C = np.zeros((plan.n, B.shape[1]), np.float64)
    tag = plan.tag
    for p in range(P):
        lo, hi = part[p], part[p + 1]
        for i in range(lo, hi):
            for k in range(row_ptr[i], row_ptr[i + 1]):
                if tag[k] == LOCAL:
                    C[i] += float(val[k]) * B[col[k]].astype(np.float64)
        for q in range(P):
            ids = plan.send_b.get((q, p))
            recv = {int(j): B[j].astype(np.float64) for j in ids} if ids is not None else {}
            for i in range(lo, hi):
                for k in range(row_ptr[i], row_ptr[i + 1]):
                    if tag[k] == COL and part[q] <= col[k] < part[q + 1]:
                        if int(col[k]) not in recv:
                            raise RuntimeError(f"coverage error at ({i},{col[k]})")
                        C[i] += float(val[k]) * recv[int(col[k])]
        for q in range(P):
            ids = plan.send_c.get((q, p))
            if ids is None:
                continue
            # q computes the partials of the ROW nonzeros it received
            for t, i in enumerate(ids):
                acc = np.zeros(B.shape[1], np.float64)
                for k in range(row_ptr[i], row_ptr[i + 1]):
                    if tag[k] == ROW and part[q] <= col[k] < part[q + 1]:
                        acc += float(val[k]) * B[col[k]].astype(np.float64)
                C[i] += acc
    # coverage: every ROW nonzero's row must be in the matching send_c list
    rows_of = _row_ids(row_ptr)
    po, qo = owner_of(part, rows_of), owner_of(part, col)
    for k in np.nonzero(tag == ROW)[0]:
        ids = plan.send_c.get((int(qo[k]), int(po[k])))
        if ids is None or rows_of[k] not in ids:
            raise RuntimeError(f"coverage error at ({rows_of[k]},{col[k]})")
    return C


def exec_hier(plan: FlatPlan, msgs, g, row_ptr, col, val, B):
    """Execute the hierarchical schedule: B rows reach p either directly
    (same group), in the stage-I union (p is the representative) or forwarded
    in stage II; partials reach p directly (same group) or pre-aggregated by
    the source group's representative in member order.
    Returns C (fp64)."""
    part, P = plan.part, plan.P
    row_ptr = np.asarray(row_ptr, np.int64)
    col = np.asarray(col, np.int64)
    B = np.asarray(B)
    N = B.shape[1]
    tag = plan.tag

    def own_partials(q, p):
        ids = plan.send_c[(q, p)]
        out = np.zeros((ids.size, N), np.float64)
        for t, i in enumerate(ids):
            for k in range(row_ptr[i], row_ptr[i + 1]):
                if tag[k] == ROW and part[q] <= col[k] < part[q + 1]:
                    out[t] += float(val[k]) * B[col[k]].astype(np.float64)
        return out

    # mailbox[(dst)] -> list of (msg, payload)
    box = {r: [] for r in range(P)}
    for m in msgs:
        if m.stage != 1:
            continue
        if m.kind == "B":
            box[m.dst].append((m, B[m.ids].astype(np.float64)))
        else:
            box[m.dst].append((m, own_partials(m.src, m.final)))
    # stage II payloads are built from what stage I delivered
    for m in msgs:
        if m.stage != 2:
            continue
        r = m.src
        if m.kind == "CA":
            p = m.final
            G = r // g
            agg = np.zeros((m.ids.size, N), np.float64)
            pos = {int(x): t for t, x in enumerate(m.ids)}
            for mem in range(G * g, G * g + g):         # member order ascending
                if (mem, p) not in plan.send_c:
                    continue
                if mem == r:
                    rows, data = plan.send_c[(mem, p)], own_partials(mem, p)
                else:
                    got = [(mm, d) for (mm, d) in box[r]
                           if mm.stage == 1 and mm.kind == "C" and mm.src == mem and mm.final == p]
                    assert len(got) == 1
                    rows, data = got[0][0].ids, got[0][1]
                for t, x in enumerate(rows):
                    agg[pos[int(x)]] += data[t]
            box[p].append((m, agg))
        else:
            q = m.owner
            got = [(mm, d) for (mm, d) in box[r] if mm.stage == 1 and mm.kind == "B" and mm.src == q]
            assert len(got) == 1
            U, data = got[0][0].ids, got[0][1]
            box[m.dst].append((m, data[np.searchsorted(U, m.ids)]))
    C = np.zeros((plan.n, N), np.float64)
    for p in range(P):
        lo, hi = part[p], part[p + 1]
        brow = {}
        for (m, d) in box[p]:
            if m.kind == "B":
                for t, j in enumerate(m.ids):
                    brow[int(j)] = d[t]
        for i in range(lo, hi):
            for k in range(row_ptr[i], row_ptr[i + 1]):
                if tag[k] == LOCAL:
                    C[i] += float(val[k]) * B[col[k]].astype(np.float64)
                elif tag[k] == COL:
                    if int(col[k]) not in brow:
                        raise RuntimeError(f"coverage error at ({i},{col[k]})")
                    C[i] += float(val[k]) * brow[int(col[k])]
        for (m, d) in sorted(box[p], key=lambda md: (md[0].stage, md[0].src)):
            if m.kind in ("C", "CA") and m.final == p and m.dst == p:
                for t, i in enumerate(m.ids):
                    C[int(i)] += d[t]
    return C


__all__ = [
    "ROW", "COL", "LOCAL", "build_oracle_lib", "uniform_partition", "owner_of",
    "spmm_ref", "min_cover_local", "min_cover", "brute_force_cover",
    "max_matching_kuhn", "FlatPlan", "balance_slack", "plan_flat", "volumes", "Msg", "rep_col",
    "rep_row", "plan_hier", "tier_traffic", "flat_inter_rows", "exec_flat", "plan_flat_digests",
    "exec_hier",
]
