"""Pins of oracle O2/O3 (neighbour patterns, block values, separation).

Ground truth is the definition (brute force over all pairs, strict r^2 <
delta^2, reading C-4); the bucket-grid oracle must equal it bit-exactly.
"""
import numpy as np
import pytest

import oracle
from workloads import grid_level, halton, uniform_points


def _same_pattern(a, b):
    return np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("d", [2, 3])
def test_grid_equals_bruteforce_square(d):
    for n, delta in ((200, 0.2), (700, 0.11), (1500, 0.05)):
        P = halton(n, d)
        assert _same_pattern(oracle.pattern(P, P, delta, "grid"),
                             oracle.pattern(P, P, delta, "brute"))


@pytest.mark.parametrize("d", [2, 3])
def test_grid_equals_bruteforce_rectangular(d):
    X = uniform_points(900, d, seed=7)
    Y = halton(300, d)
    for delta in (0.05, 0.17, 0.4):
        assert _same_pattern(oracle.pattern(X, Y, delta, "grid"),
                             oracle.pattern(X, Y, delta, "brute"))


def test_strict_boundary_hand_count():
    """5x5 grid, spacing 1/4, delta = 1/2: neighbours need a^2+b^2 < 4
    (offsets with |a|,|b| <= 1; (2,0) lies exactly on the boundary and is
    excluded).  Per axis the in-range offset counts are 2,3,3,3,2 => 13,
    so nnz = 13^2 = 169 (hand count)."""
    P = grid_level(2, 2)
    for method in ("grid", "brute"):
        rp, col = oracle.pattern(P, P, 0.5, method)
        assert rp[-1] == 169
        assert max(np.diff(rp)) == 9


def test_values_diag_symmetry_rowcost():
    """diag(A_l) = delta^-d (Phi_delta(0) = delta^-d phi(0)); A_l
    symmetric; row count <= (1 + delta/q)^d (eq:rowcost P:650)."""
    P = halton(800, 2)
    delta = 0.12
    rp, col, val = oracle.block(P, P, delta)
    n = P.shape[0]
    A = np.zeros((n, n))
    for i in range(n):
        A[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    np.testing.assert_array_equal(np.diag(A), np.full(n, delta ** -2))
    np.testing.assert_array_equal(A, A.T)
    q = oracle.separation(P)
    assert np.diff(rp).max() <= (1.0 + delta / q) ** 2


def test_table1_separation(golden):
    """q_l of the paper grids (Table 1), by the oracle's brute-force
    separation distance q_X = 1/2 min ||x_j - x_k||."""
    for lvl in ("1", "2", "3", "4"):
        P = grid_level(int(lvl), 2)
        assert P.shape[0] == golden["table1"]["N"][lvl]
        q = oracle.separation(P)
        printed = golden["table1"]["q"][lvl]
        # printed to 3 significant digits (round half up: 0.03125 -> 0.0313)
        assert abs(q - printed) <= 0.51 * 10 ** (np.floor(np.log10(printed)) - 2)
        assert q == 2.0 ** -(int(lvl) + 1)            # closed form, exact


def test_spmv_matches_dense():
    P = halton(400, 3)
    rp, col, val = oracle.block(P, P, 0.3)
    v = np.sin(np.arange(400.0))
    A = np.zeros((400, 400))
    for i in range(400):
        A[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    np.testing.assert_allclose(oracle.spmv(rp, col, val, v), A @ v, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(oracle.apply(P, P, 0.3, v), A @ v, rtol=1e-13, atol=1e-13)
