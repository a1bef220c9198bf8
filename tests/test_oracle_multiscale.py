"""Pins of the oracle's multiscale solve (O4), monolithic Jacobi (O6),
evaluation (O5) and the dense structure of §3 (O8).

* sequential eq:mas (C) == dense LU of T_L (eq:bigt, numpy)
* T_L = T'_L D_L                                   eq:matrix_decomposition
* (id - T'_L)^L = 0, Neumann series == inverse
* Theorem reformulation path sums == inverse (L <= 4)
* Theorem jacobi: exact after L sweeps, any start vector
* f in W_1 => alpha = (c, 0, ..., 0)     (e_1 = 0 after level 1)
* f_L = f on every X_l of a nested hierarchy   (interpolation)
"""
import numpy as np
import pytest

import oracle
from oracle import dense
from workloads import config, franke, grid_hierarchy, halton_hierarchy, uniform_points


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _small_halton(d):
    return halton_hierarchy("t", d, [60, 240, 960] if d == 2 else [50, 400, 1200],
                            4.0 if d == 2 else 1.5)


@pytest.mark.parametrize("H", [grid_hierarchy(3), grid_hierarchy(4), _small_halton(2),
                               _small_halton(3)], ids=["grid3", "grid4", "halton2d", "halton3d"])
def test_sequential_equals_dense_lu(H):
    f = H.f()
    a_lu = dense.solve_dense(H.points, H.delta, f)
    a_ch, _, _ = oracle.sequential(H.points, H.delta, f, direct_max_n=10 ** 6)
    a_cg, it, _ = oracle.sequential(H.points, H.delta, f, tol=1e-13, direct_max_n=0)
    for l in range(H.L):
        assert _rel(a_ch[l], a_lu[l]) < 1e-10
        assert _rel(a_cg[l], a_lu[l]) < 1e-9
        assert it[l] > 0


def test_C1_sequential_equals_dense_lu():
    H = config("C1")
    f = H.f()
    a_lu = dense.solve_dense(H.points, H.delta, f)
    a, _, _ = oracle.sequential(H.points, H.delta, f, tol=1e-13, direct_max_n=0)
    for l in range(H.L):
        assert _rel(a[l], a_lu[l]) < 1e-9


def test_factorisation_nilpotency_neumann():
    H = grid_hierarchy(4)
    T = dense.T_matrix(H.points, H.delta)
    D = dense.D_matrix(H.points, H.delta)
    Xi = dense.Xi_blocks(H.points, H.delta)
    Tp = dense.Tprime_matrix(H.points, H.delta, Xi=Xi)
    np.testing.assert_allclose(Tp @ D, T, atol=1e-11 * np.abs(T).max())
    M = dense.M_matrix(H.points, H.delta, Xi=Xi)
    ML = np.linalg.matrix_power(M, H.L)
    assert np.abs(ML).max() < 1e-10 * np.abs(M).max() ** H.L
    # strictly block-lower => M^L is exactly zero in exact arithmetic; in FP
    # it is exactly zero too since the block structure is respected
    assert np.count_nonzero(ML) == 0
    inv = np.linalg.inv(Tp)
    assert np.abs(dense.neumann_inverse(M, H.L) - inv).max() < 1e-10 * np.abs(inv).max()


@pytest.mark.parametrize("L", [3, 4])
def test_path_sum_inverse(L):
    H = grid_hierarchy(L)
    Xi = dense.Xi_blocks(H.points, H.delta)
    inv = np.linalg.inv(dense.Tprime_matrix(H.points, H.delta, Xi=Xi))
    ps = dense.path_sum_inverse(H.points, H.delta, Xi=Xi)
    assert np.abs(ps - inv).max() < 1e-10 * np.abs(inv).max()


def test_jacobi_exact_after_L_any_start():
    H = grid_hierarchy(4)
    f = H.f()
    Xi = dense.Xi_blocks(H.points, H.delta)
    M = dense.M_matrix(H.points, H.delta, Xi=Xi)
    Tp = np.eye(M.shape[0]) - M
    exact = np.linalg.solve(Tp, np.concatenate(f))
    rng = np.random.default_rng(1)
    for beta0 in (None, [np.zeros_like(x) for x in f], [rng.standard_normal(x.shape) for x in f]):
        b = dense.jacobi(M, f, H.L, beta0)
        assert _rel(b, exact) < 1e-12
    # after L-1 sweeps from a generic start the residual is not zero
    b = dense.jacobi(M, f, H.L - 1, [rng.standard_normal(x.shape) for x in f])
    assert _rel(b, exact) > 1e-6


@pytest.mark.parametrize("H", [grid_hierarchy(4), _small_halton(3)], ids=["grid4", "halton3d"])
def test_literal_jacobi_equals_sequential(H):
    f = H.f()
    a_seq, _, _ = oracle.sequential(H.points, H.delta, f, tol=1e-12, direct_max_n=0)
    a_jac, beta = oracle.jacobi_literal(H.points, H.delta, f, tol=1e-12, direct_max_n=0)
    for l in range(H.L):
        assert _rel(a_jac[l], a_seq[l]) < 1e-10
    # start-vector independence (Theorem jacobi)
    rng = np.random.default_rng(3)
    a_j2, beta2 = oracle.jacobi_literal(H.points, H.delta, f, tol=1e-12, direct_max_n=0,
                                        beta0=[rng.standard_normal(x.shape) for x in f])
    for l in range(H.L):
        assert _rel(beta2[l], beta[l]) < 1e-10
    # beta equals T'^{-1} f with dense X (eq:exactjacobi)
    Tp = dense.Tprime_matrix(H.points, H.delta)
    ex = dense.split(np.linalg.solve(Tp, np.concatenate(f)), H.points)
    for l in range(H.L):
        assert _rel(beta[l], ex[l]) < 1e-10


def test_f_in_W1_gives_coarse_only():
    """f = sum_n c_n Phi_{delta_1}(. - x_n^{(1)}) lies in W_1, so s_1 = f,
    e_1 = 0 and alpha^{(l)} = 0 for l >= 2."""
    H = grid_hierarchy(3)
    rng = np.random.default_rng(0)
    c = rng.standard_normal(H.n[0])
    f = [dense.kernel_matrix(P, H.points[0], H.delta[0]) @ c for P in H.points]
    a, _, _ = oracle.sequential(H.points, H.delta, f, direct_max_n=10 ** 6)
    assert _rel(a[0], c) < 1e-12
    for l in range(1, H.L):
        assert np.abs(a[l]).max() < 1e-12 * np.abs(c).max()


@pytest.mark.parametrize("H", [grid_hierarchy(4), _small_halton(2), _small_halton(3)],
                         ids=["grid4", "halton2d", "halton3d"])
def test_interpolation_on_all_levels(H):
    f = H.f()
    a, _, _ = oracle.sequential(H.points, H.delta, f, tol=1e-13, direct_max_n=0)
    for l in range(H.L):     # nested sets => f_L = f on every X_l
        s = oracle.evaluate(H.points, H.delta, a, H.points[l])
        assert np.abs(s - f[l]).max() < 1e-9 * np.abs(f[l]).max()


def test_evaluate_closed_forms():
    H = _small_halton(2)
    x = uniform_points(500, 2, seed=11)
    zero = [np.zeros(n) for n in H.n]
    assert not oracle.evaluate(H.points, H.delta, zero, x).any()
    unit = [np.zeros(n) for n in H.n]
    unit[1][17] = 1.0
    s = oracle.evaluate(H.points, H.delta, unit, x)
    c = H.points[1][17]
    ref = np.array([oracle.kernel(2, 1, H.delta[1], xi, c) for xi in x])
    np.testing.assert_array_equal(s, ref)
    far = np.linalg.norm(x - c, axis=1) >= H.delta[1]
    assert far.any() and not s[far].any()


def test_linearity():
    H = _small_halton(3)
    f = H.f()
    g = [np.cos(7 * P[:, 0]) * P[:, 1] for P in H.points]
    fg = [2.0 * a - 3.0 * b for a, b in zip(f, g)]
    af, _, _ = oracle.sequential(H.points, H.delta, f, direct_max_n=10 ** 6)
    ag, _, _ = oracle.sequential(H.points, H.delta, g, direct_max_n=10 ** 6)
    afg, _, _ = oracle.sequential(H.points, H.delta, fg, direct_max_n=10 ** 6)
    for l in range(H.L):
        assert _rel(afg[l], 2 * af[l] - 3 * ag[l]) < 1e-10


def test_mas_row_residual():
    H = _small_halton(2)
    f = H.f()
    a, _, _ = oracle.sequential(H.points, H.delta, f, direct_max_n=10 ** 6)
    for l in range(H.L):
        for j in (0, H.n[l] // 2, H.n[l] - 1):
            r, scale = oracle.mas_row_residual(H.points, H.delta, a, l, j, f[l][j])
            assert abs(r) < 1e-10 * scale
    a[1][5] += 1e-3
    r, scale = oracle.mas_row_residual(H.points, H.delta, a, 1, 5, f[1][5])
    assert abs(r) > 1e-6
