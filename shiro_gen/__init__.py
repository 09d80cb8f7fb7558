"""Seeded synthetic inputs for SHIRO's distributed SpMM (shared by both sides).

This module is the ONLY code both the oracle (``oracle/``) and the product
(``paper_2512_20178_b200/``) tests use.  It holds none of the method's
arithmetic: it draws random sparsity patterns and values from a counter-based
hash (``gen_core.c``) and assembles CSR arrays.

Recipe:
  * RNG  h(seed, stream, i) = SplitMix64 finaliser chain, pure function.
  * R-MAT: sample k picks, at each of ceil(log2 n) levels, a quadrant with
    probabilities (a, b, c, d); ids >= n are rejected.  Uniform: row and col
    uniform in [0, n).
  * Count: keep the first ``nnz`` distinct entries in sample order (for
    symmetric configs the first nnz/2 distinct unordered pairs i != j, then
    mirror).  Independent of chunking and thread count.
  * Scramble: one seeded permutation applied to row and column ids (Graph500
    style), spreading hubs over the partitions.
  * Values: A uniform (0,1], B uniform [0,1) (non-negative, R11);
    integer mode A in {1..4}, B in {0..7} (all partial sums < 2^24, so fp32
    results are exact in any summation order).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libshirogen.so")
_SRC = os.path.join(_HERE, "gen_core.c")
_lib = None


def build_gen_lib(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", _LIB])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_gen_lib()
        lib = ctypes.CDLL(_LIB)
        P, I64, U64, I32, D = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                               ctypes.c_int32, ctypes.c_double)
        lib.gen_hash.argtypes = [U64, U64, U64]
        lib.gen_hash.restype = U64
        lib.gen_rmat_samples.argtypes = [U64, I64, I64, I32, D, D, D, I64, P, P]
        lib.gen_uniform_samples.argtypes = [U64, I64, I64, I64, P, P]
        lib.gen_perm_keys.argtypes = [U64, I64, P]
        lib.gen_fill_values.argtypes = [U64, P, P, I64, I64, I32, P]
        lib.gen_fill_B.argtypes = [U64, I64, I64, I64, I32, P]
        for f in ("gen_rmat_samples", "gen_uniform_samples", "gen_perm_keys",
                  "gen_fill_values", "gen_fill_B"):
            getattr(lib, f).restype = None
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    nnz: int
    kind: str            # 'uniform' | 'rmat'
    abc: tuple           # R-MAT (a, b, c); d = 1 - a - b - c
    symmetric: bool
    N: int
    seed: int
    P_list: tuple
    desc: str


# BASELINE.json configs; shapes per SURVEY.md section 8(d).
CONFIGS = {
    "c1": Config("c1", 4096, 40960, "uniform", (0.25, 0.25, 0.25), False, 32, 1, (1, 2),
                 "uniform random CSR 4096x4096, nnz~40k, N=32"),
    "c2": Config("c2", 169343, 1166243, "rmat", (0.57, 0.19, 0.19), False, 128, 2, (1, 2, 4, 8),
                 "ogbn-arxiv-shaped power-law (directed R-MAT), 169k rows, 1.17M nnz, N=128"),
    "c3": Config("c3", 232965, 114615892, "rmat", (0.45, 0.22, 0.22), True, 128, 3, (1, 2, 4, 8),
                 "Reddit-shaped dense-ish (symmetric R-MAT), 233k rows, 114.6M nnz, N=128"),
    "c4": Config("c4", 2449029, 61859140, "rmat", (0.57, 0.19, 0.19), True, 128, 4, (1, 2, 4, 8),
                 "ogbn-products-shaped (symmetric R-MAT), 2.45M rows, 61.9M nnz, N=128"),
    "c5": Config("c5", 1 << 26, 1 << 30, "rmat", (0.57, 0.19, 0.19), False, 64, 5, (2, 4, 8),
                 "Graph500 R-MAT scale 26, edge factor 16, N=64"),
}


def _samples(kind, seed, k0, m, n, abc, levels):
    lib = _load()
    r = np.empty(m, np.int64)
    c = np.empty(m, np.int64)
    if kind == "uniform":
        lib.gen_uniform_samples(seed, k0, m, n, _p(r), _p(c))
    else:
        a, b, cc = abc
        lib.gen_rmat_samples(seed, k0, m, levels, a, b, cc, n, _p(r), _p(c))
    return r, c


def gen_pattern(n, nnz, kind="rmat", abc=(0.57, 0.19, 0.19), symmetric=False, seed=1,
                scramble=True):
    """Distinct (row, col) entries, first-nnz-in-sample-order rule.
    Returns (rows int64, cols int64) sorted by (row, col)."""
    levels = max(1, math.ceil(math.log2(max(n, 2))))
    target = nnz // 2 if symmetric else nnz
    if symmetric and nnz % 2:
        raise ValueError("symmetric configs need even nnz")
    m = max(1024, int(target * 1.3) + 1024)
    keys_all, k_all = [], []
    drawn = 0
    while True:
        chunk = m - drawn
        r, c = _samples(kind, seed, drawn, chunk, n, abc, levels)
        k = np.arange(drawn, drawn + chunk, dtype=np.int64)
        ok = r >= 0
        if symmetric:
            ok &= r != c
            lo, hi = np.minimum(r, c), np.maximum(r, c)
            key = lo * n + hi
        else:
            key = r * n + c
        keys_all.append(key[ok])
        k_all.append(k[ok])
        drawn = m
        keys = np.concatenate(keys_all)
        ks = np.concatenate(k_all)
        uk, first = np.unique(keys, return_index=True)   # first occurrence = smallest k
        if uk.size >= target:
            break
        m = int(m * 1.5)
        keys_all, k_all = [keys], [ks]
    sel_k = ks[first]
    if uk.size > target:
        kth = np.partition(sel_k, target - 1)[target - 1]
        keep = sel_k <= kth
        uk = uk[keep]
    rows, cols = uk // n, uk % n
    if symmetric:
        rows, cols = np.concatenate([rows, cols]), np.concatenate([cols, rows])
    if scramble:
        lib = _load()
        pk = np.empty(n, np.uint64)
        lib.gen_perm_keys(seed, n, _p(pk))
        perm = np.argsort(pk, kind="stable").astype(np.int64)   # old id -> new id
        rows, cols = perm[rows], perm[cols]
    order = np.lexsort((cols, rows))
    return rows[order], cols[order]


def to_csr(n, rows, cols, seed, value_mode=0):
    """CSR (row_ptr int64[n+1], col int32[nnz], val float32[nnz])."""
    lib = _load()
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    col = cols.astype(np.int32)
    val = np.empty(cols.size, np.float32)
    rows64 = np.ascontiguousarray(rows, np.int64)
    if cols.size:
        lib.gen_fill_values(seed, _p(rows64), _p(col), cols.size, n, value_mode, _p(val))
    return row_ptr, col, val


def gen_B(seed, row_lo, nrows, N, mode=0):
    """Dense B rows [row_lo, row_lo+nrows), float32 row-major.
    mode 0 uniform [0,1); 1 integers {0..7}; 2 integers {0,1}."""
    lib = _load()
    out = np.empty((nrows, N), np.float32)
    if nrows and N:
        lib.gen_fill_B(seed, row_lo, nrows, N, mode, _p(out))
    return out


_CACHE = {}


def gen_matrix(cfg, value_mode=0, cache_dir=None):
    """Full CSR of a named config (or Config).  Cached in memory and, when
    ``cache_dir`` (or $SHIRO_GEN_CACHE) is set, on disk as .npz."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    key = (cfg, value_mode)
    if key in _CACHE:
        return _CACHE[key]
    cache_dir = cache_dir or os.environ.get("SHIRO_GEN_CACHE")
    path = None
    if cache_dir:
        os.makedirs(cache_dir, exist_ok=True)
        path = os.path.join(cache_dir, f"{cfg.name}_n{cfg.n}_z{cfg.nnz}_s{cfg.seed}_v{value_mode}.npz")
        if os.path.exists(path):
            d = np.load(path)
            out = (d["row_ptr"], d["col"], d["val"])
            _CACHE[key] = out
            return out
    rows, cols = gen_pattern(cfg.n, cfg.nnz, cfg.kind, cfg.abc, cfg.symmetric, cfg.seed)
    out = to_csr(cfg.n, rows, cols, cfg.seed, value_mode)
    del rows, cols
    if path:
        np.savez(path, row_ptr=out[0], col=out[1], val=out[2])
    _CACHE[key] = out
    return out


def degree_stats(row_ptr, col, n):
    deg = np.diff(row_ptr)
    cdeg = np.bincount(col, minlength=n)
    return dict(max_row_deg=int(deg.max(initial=0)), mean_row_deg=float(deg.mean()) if n else 0.0,
                max_col_deg=int(cdeg.max(initial=0)), empty_row_frac=float((deg == 0).mean()) if n else 0.0)


__all__ = ["Config", "CONFIGS", "gen_pattern", "to_csr", "gen_B", "gen_matrix",
           "degree_stats", "build_gen_lib"]
