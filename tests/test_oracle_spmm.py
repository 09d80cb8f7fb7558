"""Pins for oracle.spmm_ref (C = A*B by definition).

The oracle's hand-written C loop is checked against things it does not share:
the identity and zero matrices (closed forms), a dense fp64 matmul on
small matrices (numpy's BLAS, a different routine) and exact integer
arithmetic."""
import numpy as np

import oracle
from conftest import random_csr


def test_identity_gives_B():
    n, N = 37, 5
    row_ptr = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    val = np.ones(n, np.float32)
    B = np.random.default_rng(0).random((n, N)).astype(np.float32)
    C = oracle.spmm_ref(row_ptr, col, val, B)
    assert np.array_equal(C, B.astype(np.float64))


def test_zero_matrix_gives_zero():
    n, N = 20, 7
    C = oracle.spmm_ref(np.zeros(n + 1, np.int64), np.zeros(0, np.int32),
                        np.zeros(0, np.float32), np.ones((n, N), np.float32))
    assert C.shape == (n, N) and not C.any()


def test_matches_dense_matmul():
    rng = np.random.default_rng(1)
    for n in (1, 8, 33, 64):
        for N in (1, 4, 13):
            row_ptr, col, val = random_csr(rng, n, 0.3, integer=False)
            B = rng.random((n, N)).astype(np.float32)
            dense = np.zeros((n, n))
            for i in range(n):
                for k in range(row_ptr[i], row_ptr[i + 1]):
                    dense[i, col[k]] = val[k]
            ref = dense @ B.astype(np.float64)
            C = oracle.spmm_ref(row_ptr, col, val, B)
            assert np.allclose(C, ref, rtol=1e-12, atol=0)


def test_integer_exact_and_row_selection():
    rng = np.random.default_rng(2)
    n, N = 300, 9
    row_ptr, col, val = random_csr(rng, n, 0.05, integer=True)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    C = oracle.spmm_ref(row_ptr, col, val, B)
    dense = np.zeros((n, n), np.int64)
    for i in range(n):
        for k in range(row_ptr[i], row_ptr[i + 1]):
            dense[i, col[k]] = int(val[k])
    assert np.array_equal(C, (dense @ B.astype(np.int64)).astype(np.float64))
    rows = np.array([5, 0, 299, 17], np.int64)
    assert np.array_equal(oracle.spmm_ref(row_ptr, col, val, B, rows=rows), C[rows])
