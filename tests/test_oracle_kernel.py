"""Pins of oracle O1 (Wendland phi_{d,k}, scaled kernel) against closed forms.

PAPER.md:1275 phi_(3,1)(r) = (1-r)_+^4 (4r+1); PAPER.md:66-67 eq:kernelscaling;
reading C-3 for the phi_{d,k} family.  The C oracle and the numpy dense
oracle are both checked.
"""
import numpy as np
import pytest

import oracle
from oracle import dense
from workloads import halton, uniform_points


def test_phi31_printed_examples(golden):
    for r, v in golden["kernel_examples"]["phi31"]:
        assert oracle.phi(3, 1, r) == pytest.approx(v, abs=1e-15)
        assert oracle.phi(2, 1, r) == pytest.approx(v, abs=1e-15)   # phi_{2,1} == phi_{3,1}
        assert float(dense.phi(3, 1, r)) == pytest.approx(v, abs=1e-15)


def test_scaled_examples(golden):
    for delta, r, v in golden["kernel_examples"]["scaled_d2"]:
        x = np.array([0.3, 0.7])
        y = x + np.array([r, 0.0])
        assert oracle.kernel(2, 1, delta, x, y) == pytest.approx(v, rel=1e-15)
        km = dense.kernel_matrix(x[None], y[None], delta, 1)[0, 0]
        assert km == pytest.approx(v, rel=1e-15)


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("k", [0, 1, 2])
def test_phi_family_structure(d, k):
    """Structure that fixes phi_{d,k} uniquely (Wendland): a polynomial on
    [0,1] of degree floor(d/2)+3k+1, value 1 at 0, a zero of order
    floor(d/2)+2k+1 at r=1, and vanishing odd derivatives 1,3,..,2k-1 at 0
    (C^{2k} as a radial function).  A wrong exponent, coefficient or
    normalisation fails one of these."""
    l = d // 2 + k + 1
    deg = l + 2 * k
    r = np.linspace(0.0, 0.999, 400)
    vals = np.array([oracle.phi(d, k, t) for t in r])
    coef = np.polynomial.polynomial.polyfit(r, vals, deg)
    poly = np.polynomial.polynomial.Polynomial(coef)
    assert np.max(np.abs(poly(r) - vals)) < 1e-12
    assert poly(0.0) == pytest.approx(1.0, abs=1e-12)
    # zero of order exactly l+k at r = 1: phi(1-e)/e^(l+k) tends to a finite
    # nonzero limit (ratio at e and e/10 agree to O(e))
    g = [oracle.phi(d, k, 1.0 - e) / e ** (l + k) for e in (1e-3, 1e-4)]
    assert abs(g[0]) > 1e-3 and abs(g[0] / g[1] - 1.0) < 0.05
    for m in range(1, 2 * k, 2):                # odd derivatives vanish at 0
        assert abs(poly.deriv(m)(0.0)) < 1e-6
    assert oracle.phi(d, k, 1.0) == 0.0 and oracle.phi(d, k, 1.5) == 0.0
    np.testing.assert_allclose(dense.phi(d, k, r), vals, rtol=1e-14, atol=1e-16)


def test_phi32_hand_value():
    # (1/2)^6 (35/4 + 9 + 3)/3 = 20.75/192
    assert oracle.phi(3, 2, 0.5) == pytest.approx(20.75 / 192.0, rel=1e-15)
    assert oracle.phi(3, 0, 0.5) == pytest.approx(0.25, rel=1e-15)


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("k", [0, 1, 2])
def test_positive_definite(d, k):
    """Wendland functions are strictly positive definite on R^d (P:57-75,
    P:279 'A_l are SPD'): Gram matrices of distinct points are SPD."""
    for seed in range(5):
        P = uniform_points(30, d, seed=seed)
        G = dense.kernel_matrix(P, P, 0.7, k)
        assert np.allclose(G, G.T)
        assert np.linalg.eigvalsh(G).min() > 0.0


def test_scaling_law_and_symmetry():
    P = halton(50, 3)
    for i in range(0, 50, 7):
        for j in range(0, 50, 5):
            for delta in (0.3, 0.9):
                v = oracle.kernel(3, 1, delta, P[i], P[j])
                assert v == oracle.kernel(3, 1, delta, P[j], P[i])
                u = oracle.kernel(3, 1, 1.0, P[i] / delta, P[j] / delta)
                assert v == pytest.approx(delta ** -3 * u, rel=1e-13, abs=1e-300)


def test_compact_support_strict():
    x = np.array([0.0, 0.0])
    y = np.array([0.5, 0.0])
    assert oracle.kernel(2, 1, 0.5, x, y) == 0.0          # r == delta
    assert oracle.kernel(2, 1, 0.5000001, x, y) > 0.0
