"""Multi-RHS solve (msk_solve_multi / msk_evaluate_multi).

Columns are solved in groups of 4 (tail 2 or 4, zero-padded) sharing every
CSR piece and every kernel evaluation; per column the arithmetic is that of
msk_solve, so each column must equal its single-RHS solve BIT FOR BIT (alpha,
iteration counts, s_L).  The oracle bar carries over from the single solve.
"""
import numpy as np
import pytest

import oracle
from workloads import config, franke, grid_hierarchy, halton_hierarchy, uniform_points

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def msk():
    import paper_2503_04914_b200 as m
    m.load()
    return m


@pytest.fixture(scope="module")
def ctx(msk):
    c = msk.Context(0)
    yield c
    c.close()


HIERS = {
    "C1": lambda: config("C1", m_eval=0),
    "grid5": lambda: grid_hierarchy(5),
    "halton3d": lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5),
    "halton3d_k2": lambda: halton_hierarchy("h3k2", 3, [77, 1299, 5003], 2.0, k=2),
}


def _rhs(H, nrhs, seed=0):
    """Column 0: the target function; others: smooth random fields; one zero column."""
    rng = np.random.default_rng(seed)
    cols = []
    for r in range(nrhs):
        if r == 0:
            cols.append([franke(P) for P in H.points])
        elif r == 2:
            cols.append([np.zeros(len(P)) for P in H.points])
        else:
            w = rng.standard_normal(H.d)
            cols.append([np.sin(P @ w * (1 + r)) + 0.1 * r for P in H.points])
    return [np.stack([cols[r][l] for r in range(nrhs)], axis=1) for l in range(H.L)]


@pytest.mark.parametrize("name", list(HIERS))
@pytest.mark.parametrize("nrhs,r4", [(1, False), (3, False), (4, False), (3, True), (6, True)])
def test_multi_equals_single_bitwise(msk, ctx, name, nrhs, r4, monkeypatch):
    if r4:
        monkeypatch.setenv("MSK_MULTI_R4", "1")  # 4-wide column groups
    H = HIERS[name]()
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    F = _rhs(H, nrhs)
    am, it, _ = h.solve_multi(F, tol=1e-12)
    x = uniform_points(2000, H.d, seed=5)
    sm = h.evaluate_multi(x)
    for r in range(nrhs):
        a1, info = h.solve([np.ascontiguousarray(F[l][:, r]) for l in range(H.L)], tol=1e-12)
        s1, _ = h.evaluate(x)
        for l in range(H.L):
            assert np.array_equal(am[l][:, r], a1[l]), (name, nrhs, r, l, np.abs(am[l][:, r] - a1[l]).max())
            assert it[l, r] == info.cg_iters[l]
        assert np.array_equal(sm[:, r], s1), (name, nrhs, r)
    h.close()


def test_multi_oracle_and_torch(msk, ctx):
    """C3 4-level prefix, 5 right-hand sides from device buffers: every column
    within the 1e-9 per-level bar of the oracle's sequential solve."""
    import torch
    H = config("C3P4", m_eval=0)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    F = _rhs(H, 5, seed=2)
    am, it, t = h.solve_multi([torch.from_numpy(x).cuda() for x in F])
    assert t > 0 and it[:, 2].sum() == 0  # the zero column needs no iterations
    for r in (0, 1, 4):
        ao, _, _ = oracle.sequential(H.points, H.delta, [F[l][:, r].copy() for l in range(H.L)],
                                     tol=1e-12, direct_max_n=0)
        for l in range(H.L):
            a = am[l][:, r].cpu().numpy()
            assert np.linalg.norm(a - ao[l]) <= 1e-9 * np.linalg.norm(ao[l]), (r, l)
        assert not am[0][:, 2].abs().max().item()
    h.close()


def test_multi_guards(msk, ctx):
    H = config("C1", m_eval=0)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    with pytest.raises(msk.MskError) as ei:
        h.evaluate_multi(uniform_points(10, 2))
    assert ei.value.status == 6
    h.assemble(T=2.0)
    with pytest.raises(msk.MskError) as ei:
        h.solve_multi(_rhs(H, 2))
    assert ei.value.status == 1
    h.close()
