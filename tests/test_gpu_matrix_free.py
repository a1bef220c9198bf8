"""a3 matrix-free (MSK_FLAG_MATRIX_FREE): A_l is
never stored; every CG SpMV evaluates Phi over the level's cell list.

The hits of a row are visited in ascending spatial index -- the CSR column
order -- and each entry is evaluated exactly as the assembly stores it, so
the matrix-free solve must reproduce the assembled solve BIT FOR BIT (alpha,
iteration counts, kappa estimates, s_L), for one GPU and for the partitioned
path (single-process emulation).  The oracle bar then carries over.
"""
import numpy as np
import pytest

import oracle
from workloads import config, grid_hierarchy, halton_hierarchy, uniform_points

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def msk():
    import paper_2503_04914_b200 as m
    m.load()
    return m


HIERS = {
    "C1": lambda: config("C1", m_eval=0),
    "grid5": lambda: grid_hierarchy(5),
    "halton3d": lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5),
    "halton2d_k0": lambda: halton_hierarchy("h2k0", 2, [97, 1001, 4097], 4.0, k=0),
    "halton3d_k2": lambda: halton_hierarchy("h3k2", 3, [77, 1299, 5003], 2.0, k=2),
}


def _run(msk, ctx, H, flags, f, x):
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=flags)
    h.assemble()
    a, info = h.solve(f, tol=1e-12)
    s, einfo = h.evaluate(x)
    out = (a, s, info, h.info())
    h.close()
    return out


@pytest.mark.parametrize("name", list(HIERS))
def test_matrix_free_equals_assembled_bitwise(msk, name):
    H = HIERS[name]()
    f = H.f()
    x = uniform_points(3000, H.d, seed=11)
    ctx = msk.Context(0)
    a1, s1, i1, h1 = _run(msk, ctx, H, 0, f, x)
    a2, s2, i2, h2 = _run(msk, ctx, H, msk.MSK_FLAG_MATRIX_FREE, f, x)
    for l in range(H.L):
        assert np.array_equal(a2[l], a1[l]), (name, l, np.abs(a2[l] - a1[l]).max())
        assert i2.cg_iters[l] == i1.cg_iters[l]
        assert i2.kappa_est[l] == i1.kappa_est[l]
        assert h2.nnz_A[l] == h1.nnz_A[l]
    assert np.array_equal(s2, s1)
    assert i2.nnz_cg == i1.nnz_cg
    ctx.close()


@pytest.mark.parametrize("world", [2, 3])
def test_matrix_free_partitioned_bitwise(msk, world):
    H = config("C3P4", m_eval=0)
    f = H.f()
    x = uniform_points(3000, H.d, seed=12)
    c1 = msk.Context(0)
    a1, s1, i1, _ = _run(msk, c1, H, 0, f, x)
    cw = msk.Context(0, rank=-1, world=world)
    a2, s2, i2, _ = _run(msk, cw, H, msk.MSK_FLAG_MATRIX_FREE | msk.MSK_FLAG_DIST_ALL, f, x)
    for l in range(H.L):
        assert np.array_equal(a2[l], a1[l]), (world, l)
        assert i2.cg_iters[l] == i1.cg_iters[l]
    assert np.array_equal(s2, s1)
    c1.close()
    cw.close()


def test_matrix_free_oracle_and_blocks(msk):
    """C3 4-level prefix against the oracle (1e-9 per level); A_l applied and
    exported without a stored matrix."""
    H = config("C3P4", m_eval=0)
    f = H.f()
    ctx = msk.Context(0)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=msk.MSK_FLAG_MATRIX_FREE)
    h.assemble()
    a, _ = h.solve(f, tol=1e-12)
    ao, _, _ = oracle.sequential(H.points, H.delta, f, tol=1e-12, direct_max_n=0)
    for l in range(H.L):
        assert np.linalg.norm(a[l] - ao[l]) <= 1e-9 * np.linalg.norm(ao[l])
    rng = np.random.default_rng(3)
    for l in (1, 2):
        v = rng.standard_normal(H.n[l])
        y, _ = h.apply_block(l, l, v)
        ref = oracle.apply(H.points[l], H.points[l], H.delta[l], v, k=H.k)
        orp, ocol = oracle.pattern(H.points[l], H.points[l], H.delta[l], "grid")
        # rounding scale of a kernel sum: delta^-d sum_{row} |v_j|
        bound = H.delta[l] ** -H.d * np.add.reduceat(np.abs(v)[ocol], orp[:-1])
        assert np.all(np.abs(y - ref) <= 1e-14 * bound)
        rp, col, _ = h.export_block(l, l)
        assert np.array_equal(rp, orp) and np.array_equal(col, ocol)
    ctx.close()


def test_matrix_free_guards(msk):
    H = config("C1", m_eval=0)
    ctx = msk.Context(0)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=msk.MSK_FLAG_MATRIX_FREE)
    with pytest.raises(msk.MskError) as ei:
        h.assemble(T=3.0)
    assert ei.value.status == 1
    h.assemble()
    with pytest.raises(msk.MskError) as ei:
        h.cg_level(1, H.f()[1])
    assert ei.value.status == 6
    ctx.close()


@pytest.mark.parametrize("name", ["C1", "halton3d", "grid5"])
def test_matrix_free_literal_schedule_bitwise(msk, name):
    """The LITERAL schedule (Algorithm 2 as printed, the paper's own matrix-free
    mode) on a matrix-free hierarchy: every inner and final solve
    runs the phase kernels with k_mf_spmv; bit-identical to the assembled
    literal solve, and to the pruned solve on the finest level."""
    H = HIERS[name]()
    f = H.f()
    ctx = msk.Context(0)
    res = []
    for flags in (0, msk.MSK_FLAG_MATRIX_FREE):
        h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=flags)
        h.assemble()
        a, info = h.solve(f, tol=1e-12, schedule="literal")
        ap, _ = h.solve(f, tol=1e-12, schedule="pruned")
        res.append((a, list(info.cg_iters)[:H.L], list(info.inner_iters)[:H.L], ap))
        h.close()
    (a0, i0, n0, p0), (a1, i1, n1, p1) = res
    assert i1 == i0 and n1 == n0
    for l in range(H.L):
        assert np.array_equal(a1[l], a0[l]), (name, l)
    assert np.array_equal(a1[-1], p1[-1])
    ctx.close()
