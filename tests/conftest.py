import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    """Parse a tests/golden/*.txt fixture: header keys, entries, expectations."""
    meta, entries, expect = {}, [], {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "entry":
                entries.append((int(tok[2]), int(tok[3])))
            elif tok[0] == "expect":
                expect[tok[1]] = int(tok[2]) if tok[2].lstrip("-").isdigit() else float(tok[2])
            else:
                meta[tok[0]] = int(tok[1])
    return meta, entries, expect


def csr_from_entries(n, entries, values=None):
    """CSR with columns sorted within rows (entries given as (row, col))."""
    entries = sorted(set(entries))
    rows = np.array([e[0] for e in entries], np.int64)
    cols = np.array([e[1] for e in entries], np.int64)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    val = np.ones(len(entries), np.float32) if values is None else np.asarray(values, np.float32)
    return row_ptr, cols.astype(np.int32), val


def random_csr(rng, n, density, symmetric=False, integer=True):
    """Small random CSR for invariant tests (numpy RNG; test-local)."""
    m = rng.random((n, n)) < density
    if symmetric:
        m = np.triu(m, 1)
        m = m | m.T
    rows, cols = np.nonzero(m)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    if integer:
        val = rng.integers(1, 5, rows.size).astype(np.float32)
    else:
        val = rng.random(rows.size).astype(np.float32) + np.float32(1e-3)
    return row_ptr, cols.astype(np.int32), val
