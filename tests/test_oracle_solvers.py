"""Pins of the oracle's linear solvers and of the level matrices' properties.

CG (Theorem cg, Algorithm 1, reading C-9) against its
special cases and against a direct solve; SPD-ness of A_l; the
level-independent conditioning of Lemma condA on the paper grids.
"""
import numpy as np
import pytest

import oracle
from oracle import dense
from workloads import grid_hierarchy, halton


def test_cg_identity_one_iteration():
    """delta below the separation => A = delta^-d I: CG converges in 1 step."""
    P = halton(300, 2)
    delta = 1e-4
    rp, col, val = oracle.block(P, P, delta)
    assert rp[-1] == 300
    b = np.cos(np.arange(300.0))
    x, it, st = oracle.cg(rp, col, val, b, 1e-12)
    assert st == 0 and it == 1
    np.testing.assert_allclose(x, b * delta ** 2, rtol=1e-15)


def test_cg_zero_rhs():
    P = halton(200, 3)
    rp, col, val = oracle.block(P, P, 0.3)
    x, it, st = oracle.cg(rp, col, val, np.zeros(200), 1e-12)
    assert it == 0 and st == 0 and not x.any()


def test_cg_no_convergence_flag():
    P = halton(500, 2)
    rp, col, val = oracle.block(P, P, 0.2)
    b = np.ones(500)
    x, it, st = oracle.cg(rp, col, val, b, 1e-14, max_iter=3)
    assert st == 1 and it == 3


@pytest.mark.parametrize("d,n,delta", [(2, 600, 0.15), (3, 700, 0.3)])
def test_cg_matches_direct_and_lapack(d, n, delta):
    P = halton(n, d)
    rp, col, val = oracle.block(P, P, delta)
    b = np.sin(3 * np.arange(n, dtype=float))
    x_cg, it, st = oracle.cg(rp, col, val, b, 1e-13)
    x_ch = oracle.cholesky_solve(rp, col, val, b)
    A = dense.kernel_matrix(P, P, delta)
    x_np = np.linalg.solve(A, b)
    assert st == 0 and it > 1
    np.testing.assert_allclose(x_ch, x_np, rtol=1e-10, atol=1e-10 * np.abs(x_np).max())
    assert np.linalg.norm(x_cg - x_np) <= 1e-10 * np.linalg.norm(x_np)
    # stopping rule: recurrence residual <= tol ||b|| (true residual close)
    assert np.linalg.norm(A @ x_cg - b) <= 1e-12 * np.linalg.norm(b)


def test_levels_spd_and_condA():
    """A_l SPD and kappa_2(A_l) bounded independently of l
    (Lemma condA, eq:condA P:389) on the paper's grids l = 1..6."""
    H = grid_hierarchy(6)
    kap = []
    for P, dl in zip(H.points, H.delta):
        A = dense.kernel_matrix(P, P, dl)
        ev = np.linalg.eigvalsh(A)
        assert ev.min() > 0
        kap.append(ev.max() / ev.min())
    assert max(kap[2:]) / min(kap[2:]) < 1.5      # level-independent
    assert max(kap) < 50


def test_cholesky_rejects_indefinite():
    rp = np.array([0, 2, 4], dtype=np.int64)
    col = np.array([0, 1, 0, 1], dtype=np.int32)
    val = np.array([1.0, 2.0, 2.0, 1.0])
    with pytest.raises(np.linalg.LinAlgError):
        oracle.cholesky_solve(rp, col, val, np.ones(2))


@pytest.mark.parametrize("threads", [1, 4])
def test_native_openmp_build_is_bitwise_identical(threads):
    """The CPU baseline's build of the same oracle source (-O3 -march=native
    -ffp-contract=off -fopenmp, rows split over threads, reductions serial) gives
    the plain build's results bit for bit: patterns, sequential alpha (CG), and
    the evaluation."""
    from workloads import config
    H = config("C3P4", m_eval=2000)
    H.points, H.delta = H.points[:3], H.delta[:3]
    f = H.f()
    oracle.use_plain()
    a0, it0, c0 = oracle.sequential(H.points, H.delta, f, tol=1e-12, direct_max_n=0)
    s0 = oracle.evaluate(H.points, H.delta, a0, H.eval_points)
    rp0, col0 = oracle.pattern(H.points[2], H.points[1], H.delta[1])
    try:
        assert oracle.use_native(threads) == threads
        a1, it1, c1 = oracle.sequential(H.points, H.delta, f, tol=1e-12, direct_max_n=0)
        s1 = oracle.evaluate(H.points, H.delta, a1, H.eval_points)
        rp1, col1 = oracle.pattern(H.points[2], H.points[1], H.delta[1])
    finally:
        oracle.use_plain()
    assert it0 == it1 and np.array_equal(c0, c1)
    for l in range(3):
        assert np.array_equal(a0[l], a1[l])
    assert np.array_equal(s0, s1)
    assert np.array_equal(rp0, rp1) and np.array_equal(col0, col1)
