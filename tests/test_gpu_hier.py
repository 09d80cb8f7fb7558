"""GPU parity of the hierarchical schedule (section VI, Alg. 1) on
one device: all virtual ranks in the loopback ABI, Stage I / Stage II
producers storing through per-row destination pointers into the other
ranks' R1 / R2 buffers (the same kernels the multi-GPU path runs over NVLink).
Integer data: exact; float data: DESIGN.md R11 tolerance."""
import numpy as np
import pytest

import oracle
import shiro_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_20178_b200 as sh  # noqa: E402
from conftest import csr_from_entries, load_golden, random_csr  # noqa: E402


def run(n, part, row_ptr, col, val, B, g, flags=0):
    P = part.size - 1
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, B.shape[1], group_size=g, flags=flags)
    Bd = torch.from_numpy(B).cuda()
    Cd = torch.full((n, B.shape[1]), float("nan"), device="cuda")
    pl.spmm_loopback(Bd, Cd)
    torch.cuda.synchronize()
    return Cd.cpu().numpy(), pl


@pytest.mark.parametrize("P,g", [(4, 2), (8, 2), (8, 4), (6, 3), (8, 8)])
@pytest.mark.parametrize("N", [32, 128, 5])
def test_hier_random_integer_exact(P, g, N):
    rng = np.random.default_rng(P * 31 + g * 7 + N)
    n = 1500
    row_ptr, col, val = random_csr(rng, n, 0.01, symmetric=(P + g) % 2 == 0)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    part = oracle.uniform_partition(n, P)
    C, _ = run(n, part, row_ptr, col, val, B, g)
    assert np.array_equal(C.astype(np.float64), oracle.spmm_ref(row_ptr, col, val, B))


@pytest.mark.parametrize("name", ["hier_col.txt", "hier_row.txt"])
def test_hier_paper_fixtures(name):
    meta, entries, _ = load_golden(name)
    n, P, g = meta["n"], meta["P"], meta["g"]
    rng = np.random.default_rng(1)
    row_ptr, col, _ = csr_from_entries(n, entries)
    val = rng.integers(1, 5, col.size).astype(np.float32)
    B = rng.integers(0, 8, (n, 16)).astype(np.float32)
    C, _ = run(n, oracle.uniform_partition(n, P), row_ptr, col, val, B, g)
    assert np.array_equal(C.astype(np.float64), oracle.spmm_ref(row_ptr, col, val, B))


@pytest.mark.parametrize("g", [2, 4])
def test_hier_c2_float_and_repeat(g):
    c = shiro_gen.CONFIGS["c2"]
    row_ptr, col, val = shiro_gen.gen_matrix("c2")
    B = shiro_gen.gen_B(c.seed, 0, c.n, c.N)
    part = oracle.uniform_partition(c.n, 8)
    P = 8
    pl = sh.Plan.loopback(P, c.n, part, row_ptr, col, val, c.N, group_size=g)
    Bd = torch.from_numpy(B).cuda()
    C1 = torch.empty((c.n, c.N), device="cuda")
    C2 = torch.empty_like(C1)
    pl.spmm_loopback(Bd, C1)
    pl.spmm_loopback(Bd, C2)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    ref = oracle.spmm_ref(row_ptr, col, val, B)
    d = np.abs(C1.cpu().numpy().astype(np.float64) - ref)
    assert not (d > np.maximum(1e-4 * np.abs(ref), 1e-6)).any()


def test_graph_replay_matches_direct_launch():
    """shiro_spmm on a non-default stream is captured into a CUDA graph and
    replayed; results equal a direct (SHIRO_GRAPH-independent) check."""
    c = shiro_gen.CONFIGS["c2"]
    row_ptr, col, val = shiro_gen.gen_matrix("c2", value_mode=1)
    B = shiro_gen.gen_B(c.seed, 0, c.n, c.N, mode=1)
    pl = sh.Plan.distributed(0, 1, c.n, np.array([0, c.n]), row_ptr, col, val, c.N)
    st = torch.cuda.Stream()
    Bd = torch.from_numpy(B).cuda()
    ref = oracle.spmm_ref(row_ptr, col, val, B)
    for _ in range(3):
        Cd = torch.full((c.n, c.N), float("nan"), device="cuda")
        st.wait_stream(torch.cuda.current_stream())   # C's fill first
        pl.spmm(Bd, Cd, st)
        st.synchronize()
        assert np.array_equal(Cd.cpu().numpy().astype(np.float64), ref)
    assert pl.last_launches() == 1


@pytest.mark.parametrize("P", [1, 2, 4])
def test_transposed_product_integer_exact(P):
    """SHIRO_F_TRANSPOSE computes C = A^T B (GNN backward)."""
    from test_transpose import csr_transpose
    rng = np.random.default_rng(31 + P)
    n, N = 1200, 64
    row_ptr, col, val = random_csr(rng, n, 0.01)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    part = oracle.uniform_partition(n, P)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, N, flags=sh.F_TRANSPOSE)
    Bd = torch.from_numpy(B).cuda()
    Cd = torch.full((n, N), float("nan"), device="cuda")
    pl.spmm_loopback(Bd, Cd)
    torch.cuda.synchronize()
    trp, tcol, tval = csr_transpose(n, row_ptr, col, val)
    assert np.array_equal(Cd.cpu().numpy().astype(np.float64), oracle.spmm_ref(trp, tcol, tval, B))
