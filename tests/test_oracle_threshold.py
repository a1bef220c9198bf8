"""Pins of the dense thresholded oracle (O7): M~(T), eq:perturbed_split.

* T -> infinity keeps every entry: alpha~ == exact alpha
* Lagrange property chi_i(x_j) = delta_ij (eq:cardinal P:352-355): rows of
  X_{kl} at nodes coinciding with level-l nodes are unit vectors
* the (corrected, reading C-22) Lemma pert1 inequality
  ||beta - beta~|| <= ||f|| ||M - M~|| sum_{k=1}^{L-1} k max(||M||,||M~||)^{k-1}
* Theorem decayerror property: the error shrinks as T grows (overall)
"""
import numpy as np
import pytest

import oracle
from oracle import dense
from workloads import grid_hierarchy, halton_hierarchy


def test_infinite_T_equals_exact():
    H = grid_hierarchy(4)
    f = H.f()
    Xi = dense.Xi_blocks(H.points, H.delta)
    a_ex = dense.solve_dense(H.points, H.delta, f)
    a_t, _ = dense.thresholded_solve(H.points, H.delta, H.q, f, 1e9, Xi=Xi)
    for l in range(H.L):
        assert np.linalg.norm(a_t[l] - a_ex[l]) <= 1e-10 * max(np.linalg.norm(a_ex[l]), 1e-300) + 1e-14


def test_lagrange_property_nested_grid():
    H = grid_hierarchy(4)
    Xi = dense.Xi_blocks(H.points, H.delta)
    for (a, b), blk in Xi.items():
        # grid level b node x_i coincides with level a node j
        Pa, Pb = H.points[a], H.points[b]
        for i in range(0, Pb.shape[0], 3):
            j = int(np.argmin(np.sum((Pa - Pb[i]) ** 2, axis=1)))
            assert np.all(Pa[j] == Pb[i])
            e = np.zeros(Pb.shape[0])
            e[i] = 1.0
            assert np.abs(blk[j] - e).max() < 1e-10


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("L", [3, 4])
@pytest.mark.parametrize("T", [1.0, 2.5, 4.0])
def test_c_oracle_equals_dense_thresholded(L, T):
    """The C oracle's forward substitution with M~(T) (O7) equals the dense
    numpy form (Jacobi on the dense masked M, itself pinned by Figures 2-3),
    and its entry count equals the geometric mask size."""
    H = grid_hierarchy(L)
    f = H.f()
    Xi = dense.Xi_blocks(H.points, H.delta)
    a_d, b_d = dense.thresholded_solve(H.points, H.delta, H.q, f, T, Xi=Xi)
    a_c, b_c, nnz = oracle.thresholded(H.points, H.delta, H.q, T, f)
    mask = dense.truncation_mask(H.points, H.q, T)
    assert nnz == sum(int(m.sum()) for m in mask.values())
    for l in range(H.L):
        assert _rel(b_c[l], b_d[l]) < 1e-11
        assert _rel(a_c[l], a_d[l]) < 1e-10


def test_c_oracle_thresholded_large_T_is_exact():
    H = halton_hierarchy("t", 3, [40, 320, 1200], 1.5)
    f = H.f()
    a_t, _, _ = oracle.thresholded(H.points, H.delta, H.q, 1e6, f)
    a_s, _, _ = oracle.sequential(H.points, H.delta, f, direct_max_n=10 ** 6)
    for l in range(H.L):
        assert _rel(a_t[l], a_s[l]) < 1e-10


def test_pert1_bound_and_decay():
    H = grid_hierarchy(4)
    f = H.f()
    fv = np.concatenate(f)
    Xi = dense.Xi_blocks(H.points, H.delta)
    M = dense.M_matrix(H.points, H.delta, Xi=Xi)
    beta_ex = dense.jacobi(M, f, H.L)
    errs = []
    for T in range(1, 7):
        Mt = dense.Mtilde_matrix(H.points, H.delta, H.q, T, Xi=Xi)
        bt = dense.jacobi(Mt, f, H.L)
        err = np.linalg.norm(beta_ex - bt)
        nM, nMt = np.linalg.norm(M, 2), np.linalg.norm(Mt, 2)
        bound = np.linalg.norm(fv) * np.linalg.norm(M - Mt, 2) * sum(
            k * max(nM, nMt) ** (k - 1) for k in range(1, H.L))
        assert err <= bound
        errs.append(err)
    assert errs[-1] < 0.2 * errs[0]
