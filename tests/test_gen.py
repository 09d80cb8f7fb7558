"""Generator determinism and shape (shiro_gen holds no method arithmetic)."""
import numpy as np

import shiro_gen


def test_pattern_deterministic_exact_nnz_and_sorted():
    a = shiro_gen.gen_pattern(5000, 30000, "rmat", (0.57, 0.19, 0.19), False, seed=11)
    b = shiro_gen.gen_pattern(5000, 30000, "rmat", (0.57, 0.19, 0.19), False, seed=11)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[0].size == 30000
    key = a[0] * 5000 + a[1]
    assert np.all(np.diff(key) > 0)                      # distinct, row-major sorted
    c = shiro_gen.gen_pattern(5000, 30000, "rmat", (0.57, 0.19, 0.19), False, seed=12)
    assert not np.array_equal(a[1], c[1])


def test_symmetric_pattern():
    r, c = shiro_gen.gen_pattern(3000, 20000, "rmat", (0.45, 0.22, 0.22), True, seed=3)
    assert r.size == 20000 and not np.any(r == c)
    s = set(zip(r.tolist(), c.tolist()))
    assert all((j, i) in s for i, j in s)


def test_values_and_B():
    rp, col, val = shiro_gen.gen_matrix("c1")
    assert rp[-1] == 40960 and np.all(val > 0) and np.all(val <= 1)
    _, _, vi = shiro_gen.gen_matrix("c1", value_mode=1)
    assert set(np.unique(vi).tolist()) <= {1.0, 2.0, 3.0, 4.0}
    B = shiro_gen.gen_B(1, 0, 100, 32)
    assert B.dtype == np.float32 and np.all((B >= 0) & (B < 1))
    assert np.array_equal(shiro_gen.gen_B(1, 40, 10, 32), B[40:50])    # shardable by rows
    Bi = shiro_gen.gen_B(1, 0, 100, 32, mode=1)
    assert set(np.unique(Bi).tolist()) <= set(float(x) for x in range(8))
