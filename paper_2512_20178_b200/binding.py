"""Thin ctypes binding of libshiro.so (include/shiro.h).

Argument marshalling only: every step of the hot path runs inside the C/CUDA
library.  There is no fallback: if libshiro.so is missing or fails to load,
``load()`` raises.  PyTorch is used only for device memory and streams (the
caller passes torch tensors; their data pointers cross the ABI).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libshiro.so")

SHIRO_OK = 0
STATUS = {0: "SHIRO_OK", 1: "SHIRO_E_ARG", 2: "SHIRO_E_CSR", 3: "SHIRO_E_PART", 4: "SHIRO_E_CUDA",
          5: "SHIRO_E_NCCL", 6: "SHIRO_E_OOM", 7: "SHIRO_E_INTERNAL", 8: "SHIRO_E_PEER",
          9: "SHIRO_E_TRANSPORT"}

F_COVER_ROWMAX = 0
F_COVER_COLMAX = 1 << 0
F_MODE_JOINT = 0
F_MODE_COL = 1 << 1
F_MODE_ROW = 1 << 2
F_SPLIT_RECV = 1 << 3
F_COVER_BALANCE = 1 << 9
F_HOST_ONLY = 1 << 4
F_NO_OVERLAP = 1 << 5
F_XCHG_NCCL = 1 << 6
F_MODE_BLOCK = 1 << 7
F_TRANSPOSE = 1 << 8

STAGES = ("pack", "partial", "exchange", "local", "remote", "scatter", "total")

LIST_SEND_B, LIST_SEND_C, LIST_RECV_B, LIST_RECV_C = 0, 1, 2, 3
LIST_H1_SEND, LIST_H2_SEND, LIST_H1_RECV, LIST_H2_RECV = 4, 5, 6, 7

ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p,
                                ctypes.POINTER(ctypes.c_int64))


class ShiroError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class DistT(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("group_size", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("nccl_id", ctypes.c_void_p), ("host_xchg", ALLTOALLV_FN),
                ("host_xchg_ctx", ctypes.c_void_p)]


_INFO_FIELDS = ["rank", "nranks", "group_size", "N"]
_INFO_FIELDS64 = ["n", "m_local", "nnz_local", "nnz_diag", "nnz_colbased",
                  "nnz_rowbased_shipped", "nnz_rowbased_computed", "send_b_rows", "send_c_rows",
                  "recv_b_rows", "recv_c_rows", "g_joint_rows", "g_col_rows", "g_row_rows",
                  "g_block_rows", "g_oblivious_rows", "g_setup_bytes", "g_flat_inter_rows",
                  "g_hier_inter_rows", "g_hier_intra_rows", "g_max_send_rows", "g_max_recv_rows",
                  "dev_bytes"]


class InfoT(ctypes.Structure):
    _fields_ = ([(f, ctypes.c_int32) for f in _INFO_FIELDS] +
                [(f, ctypes.c_int64) for f in _INFO_FIELDS64] +
                [("plan_seconds", ctypes.c_double)] +
                [(f, ctypes.c_int64 * 5) for f in ("op_nnz", "op_rows", "op_src_rows")] +
                [("refresh_seconds", ctypes.c_double)])

OPS = ("local", "partial", "remote", "scatter", "pack")


_lib = None


def load():
    """Load libshiro.so (fails loudly; there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() or "
                          "python -m paper_2512_20178_b200.build")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    sig = {
        "shiro_get_unique_id": [P],
        "shiro_plan": [ctypes.POINTER(DistT), I64, P, P, P, P, I32, P, ctypes.POINTER(P)],
        "shiro_plan_weighted": [ctypes.POINTER(DistT), I64, P, P, P, P, I32, P, P, P,
                                ctypes.POINTER(P)],
        "shiro_plan_update_values": [P, P, P, P, P],
        "shiro_plan_loopback_weighted": [I32, I32, U32, I64, P, P, P, P, I32, P, P, P,
                                         ctypes.POINTER(P)],
        "shiro_plan_update_values_loopback": [P, P, P],
        "shiro_spmm": [P, P, P, P],
        "shiro_spmm_host": [P, P, P, P],
        "shiro_spmm_host_batch": [P, I64, P, P, P],
        "shiro_free": [P],
        "shiro_plan_info": [P, ctypes.POINTER(InfoT)],
        "shiro_plan_list": [P, I32, I32, P, I64, ctypes.POINTER(I64)],
        "shiro_plan_loopback": [I32, I32, U32, I64, P, P, P, P, I32, P, ctypes.POINTER(P)],
        "shiro_spmm_loopback": [P, P, P, P],
        "shiro_plan_rank": [P, I32, ctypes.POINTER(P)],
        "shiro_profile": [P, I32],
        "shiro_stage_times": [P, P],
        "shiro_probe_gather": [P, I32, P, I64, P, I32, P],
        "shiro_probe_gather_tma": [P, I64, I32, P, I64, P, I32, I32, P],
        "shiro_probe_fma": [P, I32, I32, P],
        "shiro_probe_gather_tma_ws": [P, I64, I32, P, I64, P, I32, I32, P],
        "shiro_probe_copy": [P, P, I64, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.shiro_last_error.argtypes = []
    lib.shiro_last_error.restype = ctypes.c_char_p
    lib.shiro_last_launches.argtypes = [P]
    lib.shiro_last_launches.restype = ctypes.c_int64
    _lib = lib
    return lib


def _check(rc):
    if rc != SHIRO_OK:
        raise ShiroError(rc, load().shiro_last_error().decode())


def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _stream_ptr(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def probe_gather(X, idx, out, chunk=256, stream=None):
    """shiro_probe_gather on torch CUDA tensors (X fp32 [*, N], idx int32)."""
    _check(load().shiro_probe_gather(ctypes.c_void_p(X.data_ptr()), X.shape[1],
                                     ctypes.c_void_p(idx.data_ptr()), idx.numel(),
                                     ctypes.c_void_p(out.data_ptr()), chunk, _stream_ptr(stream)))


def probe_gather_tma(X, idx, out, chunk=256, stages=4, stream=None):
    """shiro_probe_gather_tma (TMA gather4 staging) on torch CUDA tensors."""
    _check(load().shiro_probe_gather_tma(ctypes.c_void_p(X.data_ptr()), X.shape[0], X.shape[1],
                                         ctypes.c_void_p(idx.data_ptr()), idx.numel(),
                                         ctypes.c_void_p(out.data_ptr()), chunk, stages,
                                         _stream_ptr(stream)))


def probe_gather_tma_ws(X, idx, out, stages=24, ctas=None, stream=None):
    """shiro_probe_gather_tma_ws (warp-specialized TMA gather4 ring)."""
    if ctas is None:
        import torch
        ctas = 4 * torch.cuda.get_device_properties(X.device).multi_processor_count
    _check(load().shiro_probe_gather_tma_ws(ctypes.c_void_p(X.data_ptr()), X.shape[0], X.shape[1],
                                            ctypes.c_void_p(idx.data_ptr()), idx.numel(),
                                            ctypes.c_void_p(out.data_ptr()), stages, ctas,
                                            _stream_ptr(stream)))


def probe_fma(out, blocks, iters, stream=None):
    """shiro_probe_fma (FP32 FMA peak probe); out: CUDA float tensor >= blocks*256."""
    _check(load().shiro_probe_fma(ctypes.c_void_p(out.data_ptr()), blocks, iters,
                                  _stream_ptr(stream)))


def probe_copy(x, y, stream=None):
    """shiro_probe_copy (HBM copy probe) between two CUDA float tensors."""
    _check(load().shiro_probe_copy(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                   x.numel(), _stream_ptr(stream)))


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().shiro_get_unique_id(buf))
    return buf.raw


def _host_arrays(row_ptr, col, val):
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float32)
    return row_ptr, col, val


class Plan:
    """A SHIRO plan handle (distributed rank, loopback, or borrowed rank view)."""

    def __init__(self, handle, owner=True, keep=None):
        self._h = ctypes.c_void_p(handle)
        self._owner = owner
        self._keep = keep          # keeps ctypes callbacks alive

    # ---------------------------------------------------------------- build
    @classmethod
    def distributed(cls, rank, nranks, n, part, row_ptr, col, val, N, group_size=1, flags=0,
                    nccl_id=None, host_xchg=None, stream=None, w_row=None, w_col=None):
        """shiro_plan (or shiro_plan_weighted with w_row [M_p] / w_col [n]
        int64 costs): this rank's CSR rows (global column ids).  ``host_xchg``:
        optional Python all-to-allv (list of bytes per peer -> list of bytes)
        used for the plan-time exchange (e.g. over gloo) and later value
        refreshes."""
        lib = load()
        part = np.ascontiguousarray(part, dtype=np.int64)
        row_ptr, col, val = _host_arrays(row_ptr, col, val)
        keep = []
        d = DistT(rank, nranks, group_size, flags, None, ALLTOALLV_FN(), None)
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            keep.append(idbuf)
            d.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
        if host_xchg is not None:
            cb = _make_alltoallv(host_xchg, nranks, rank)
            keep.append(cb)
            d.host_xchg = cb
        out = ctypes.c_void_p()
        s = ctypes.c_void_p(0) if flags & F_HOST_ONLY else _stream_ptr(stream)
        if w_row is None and w_col is None:
            _check(lib.shiro_plan(ctypes.byref(d), n, _np_ptr(part), _np_ptr(row_ptr),
                                  _np_ptr(col), _np_ptr(val), N, s, ctypes.byref(out)))
        else:
            wr = np.ascontiguousarray(w_row, dtype=np.int64)
            wc = np.ascontiguousarray(w_col, dtype=np.int64)
            _check(lib.shiro_plan_weighted(ctypes.byref(d), n, _np_ptr(part), _np_ptr(row_ptr),
                                           _np_ptr(col), _np_ptr(val), N, _np_ptr(wr),
                                           _np_ptr(wc), s, ctypes.byref(out)))
        return cls(out.value, True, keep)

    @classmethod
    def loopback(cls, nranks, n, part, row_ptr, col, val, N, group_size=1, flags=0,
                 stream=None, w_row=None, w_col=None):
        """shiro_plan_loopback (shiro_plan_loopback_weighted with w_row [n] /
        w_col [n] int64 costs): all virtual ranks on one device (full CSR)."""
        lib = load()
        part = np.ascontiguousarray(part, dtype=np.int64)
        row_ptr, col, val = _host_arrays(row_ptr, col, val)
        out = ctypes.c_void_p()
        s = ctypes.c_void_p(0) if flags & F_HOST_ONLY else _stream_ptr(stream)
        if w_row is None and w_col is None:
            _check(lib.shiro_plan_loopback(nranks, group_size, flags, n, _np_ptr(part),
                                           _np_ptr(row_ptr), _np_ptr(col), _np_ptr(val), N, s,
                                           ctypes.byref(out)))
        else:
            wr = np.ascontiguousarray(w_row, dtype=np.int64)
            wc = np.ascontiguousarray(w_col, dtype=np.int64)
            _check(lib.shiro_plan_loopback_weighted(nranks, group_size, flags, n, _np_ptr(part),
                                                    _np_ptr(row_ptr), _np_ptr(col),
                                                    _np_ptr(val), N, _np_ptr(wr), _np_ptr(wc), s,
                                                    ctypes.byref(out)))
        pl = cls(out.value, True)
        pl._loopback = True
        return pl

    def update_values(self, val, row_ptr=None, col=None, stream=None):
        """shiro_plan_update_values (distributed; row_ptr/col needed only for
        SHIRO_F_TRANSPOSE plans) or shiro_plan_update_values_loopback."""
        val = np.ascontiguousarray(val, dtype=np.float32)
        lib = load()
        if self._is_loopback():
            _check(lib.shiro_plan_update_values_loopback(self._h, _np_ptr(val),
                                                         _stream_ptr(stream)))
            return
        rp = None if row_ptr is None else np.ascontiguousarray(row_ptr, dtype=np.int64)
        cl = None if col is None else np.ascontiguousarray(col, dtype=np.int32)
        _check(lib.shiro_plan_update_values(self._h, _np_ptr(rp), _np_ptr(cl), _np_ptr(val),
                                            _stream_ptr(stream)))

    def _is_loopback(self):
        return getattr(self, "_loopback", False)

    # ---------------------------------------------------------------- run
    def spmm(self, B, C, stream=None):
        """shiro_spmm(B_p, C_p) on torch CUDA tensors (fp32, contiguous)."""
        _check(load().shiro_spmm(self._h, ctypes.c_void_p(B.data_ptr()),
                                 ctypes.c_void_p(C.data_ptr()), _stream_ptr(stream)))

    def spmm_host(self, B, C, stream=None):
        """shiro_spmm_host on host buffers (numpy or pinned torch CPU tensors)."""
        bp = B.ctypes.data if isinstance(B, np.ndarray) else B.data_ptr()
        cp = C.ctypes.data if isinstance(C, np.ndarray) else C.data_ptr()
        _check(load().shiro_spmm_host(self._h, ctypes.c_void_p(bp), ctypes.c_void_p(cp),
                                      _stream_ptr(stream)))

    def spmm_host_batch(self, Bs, Cs, stream=None):
        """shiro_spmm_host_batch: item i reads host buffer Bs[i], writes Cs[i]
        (uploads, SpMMs and downloads pipelined over the batch)."""
        if len(Bs) != len(Cs):
            raise ValueError("Bs and Cs differ in length")
        ptr = lambda x: x.ctypes.data if isinstance(x, np.ndarray) else x.data_ptr()
        nb = len(Bs)
        bp = (ctypes.c_void_p * max(nb, 1))(*[ptr(b) for b in Bs])
        cp = (ctypes.c_void_p * max(nb, 1))(*[ptr(c) for c in Cs])
        _check(load().shiro_spmm_host_batch(self._h, nb, ctypes.cast(bp, ctypes.c_void_p),
                                            ctypes.cast(cp, ctypes.c_void_p), _stream_ptr(stream)))

    def spmm_loopback(self, B, C, stream=None):
        _check(load().shiro_spmm_loopback(self._h, ctypes.c_void_p(B.data_ptr()),
                                          ctypes.c_void_p(C.data_ptr()), _stream_ptr(stream)))

    def profile(self, enable=True):
        _check(load().shiro_profile(self._h, 1 if enable else 0))

    def stage_times(self) -> dict:
        """Stage durations (ms) of the last profiled shiro_spmm."""
        buf = (ctypes.c_double * len(STAGES))()
        _check(load().shiro_stage_times(self._h, buf))
        return dict(zip(STAGES, list(buf)))

    def last_launches(self):
        return int(load().shiro_last_launches(self._h))

    # ---------------------------------------------------------------- query
    def rank_view(self, r):
        out = ctypes.c_void_p()
        _check(load().shiro_plan_rank(self._h, r, ctypes.byref(out)))
        return Plan(out.value, owner=False, keep=self)

    def info(self) -> dict:
        inf = InfoT()
        _check(load().shiro_plan_info(self._h, ctypes.byref(inf)))
        d = {}
        for f, _ in InfoT._fields_:
            v = getattr(inf, f)
            d[f] = dict(zip(OPS, list(v))) if f.startswith("op_") else v
        return d

    def list(self, peer, kind) -> np.ndarray:
        lib = load()
        n = ctypes.c_int64()
        _check(lib.shiro_plan_list(self._h, peer, kind, None, 0, ctypes.byref(n)))
        buf = np.empty(n.value, np.int64)
        _check(lib.shiro_plan_list(self._h, peer, kind, _np_ptr(buf), n.value, ctypes.byref(n)))
        return buf

    def free(self):
        if self._owner and self._h:
            _check(load().shiro_free(self._h))
        self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            if self._owner and self._h:
                load().shiro_free(self._h)
        except Exception:
            pass


def _make_alltoallv(py_fn, P, rank):
    """Wrap ``py_fn(list_of_bytes) -> list_of_bytes`` as a shiro_alltoallv_fn."""

    def cb(ctx, send, send_bytes, recv, recv_bytes):
        try:
            ss = [send_bytes[p] for p in range(P)]
            rs = [recv_bytes[p] for p in range(P)]
            segs, o = [], 0
            for p in range(P):
                segs.append(ctypes.string_at(send + o, ss[p]) if ss[p] else b"")
                o += ss[p]
            got = py_fn(segs)
            o = 0
            for p in range(P):
                if rs[p]:
                    if len(got[p]) != rs[p]:
                        return 1
                    ctypes.memmove(recv + o, got[p], rs[p])
                o += rs[p]
            return 0
        except Exception:      # noqa: BLE001 - reported as SHIRO_E_TRANSPORT
            import traceback
            traceback.print_exc()
            return 1

    return ALLTOALLV_FN(cb)


def torch_dist_alltoallv(group=None):
    """A host all-to-allv over torch.distributed (gloo or any backend with
    CPU send/recv): list of bytes per peer -> list of bytes per peer."""
    import torch
    import torch.distributed as dist

    def fn(segs):
        P, me = dist.get_world_size(group), dist.get_rank(group)
        sizes = torch.tensor([len(s) for s in segs], dtype=torch.int64)
        all_sizes = [torch.zeros(P, dtype=torch.int64) for _ in range(P)]
        dist.all_gather(all_sizes, sizes, group=group)
        reqs, bufs = [], [None] * P
        for p in range(P):
            if p == me:
                bufs[p] = segs[p]
                continue
            n_in = int(all_sizes[p][me])
            if len(segs[p]):
                t = torch.frombuffer(bytearray(segs[p]), dtype=torch.uint8)
                reqs.append(dist.isend(t, p, group=group))
            if n_in:
                bufs[p] = torch.empty(n_in, dtype=torch.uint8)
                reqs.append(dist.irecv(bufs[p], p, group=group))
            else:
                bufs[p] = b""
        for r in reqs:
            r.wait()
        return [b if isinstance(b, (bytes, bytearray)) else bytes(b.numpy().tobytes())
                for b in bufs]

    return fn


def uniform_partition(n: int, P: int) -> np.ndarray:
    """Default 1D row partition: contiguous blocks of
    ceil/floor(n/P) rows, larger blocks first; columns use the same
    boundaries."""
    base, extra = divmod(int(n), int(P))
    sizes = np.full(P, base, np.int64)
    sizes[:extra] += 1
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def local_rows(row_ptr, col, val, part, rank):
    """This rank's CSR rows (row_ptr rebased to 0; global column ids)."""
    lo, hi = int(part[rank]), int(part[rank + 1])
    s, e = int(row_ptr[lo]), int(row_ptr[hi])
    return (np.asarray(row_ptr[lo:hi + 1], np.int64) - s, np.asarray(col[s:e]),
            np.asarray(val[s:e]))
