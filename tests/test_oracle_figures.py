"""The paper's printed worked examples: Figures 1-3.

Grids l = 1..L on [0,1]^2 (Table 1), mu = 0.5, nu = 4, phi_(3,1), the
column level's delta in B_{kl} (reading C-1), truncation radius T q_l with
the coarse column level's q and strict '<' (reading C-5), Figure 3 counting
|v| > 1e-8 (reading C-6).  Every printed digit must be reproduced: a wrong
block index, delta convention, sign of M, truncation radius or boundary
fails these.
"""
import numpy as np
import pytest

from oracle import dense
from workloads import grid_hierarchy


def _printed_eq(val, printed, digits):
    return abs(val - printed) <= 0.5 * 10.0 ** (-digits) + 1e-12


@pytest.mark.parametrize("L", [2, 3, 4, 5])
def test_figure1_norm(golden, L):
    H = grid_hierarchy(L)
    v = dense.fig1_norm(H.points, H.delta)
    assert _printed_eq(v, golden["figure1"]["numerical"][str(L)], 3)


@pytest.mark.slow
def test_figure1_norm_L6(golden):
    H = grid_hierarchy(6)
    assert _printed_eq(dense.fig1_norm(H.points, H.delta), golden["figure1"]["numerical"]["6"], 3)


def test_figure1_bound_curve_reading(golden):
    """Reading C-23: the printed bound curve is sqrt(L) 2^(L-1)."""
    for L, v in golden["figure1"]["bound"].items():
        assert _printed_eq(dense.fig1_bound(int(L)), v, 3)


@pytest.mark.parametrize("L", [3, 4, 5])
def test_figure2_and_3(golden, L):
    H = grid_hierarchy(L)
    Xi = dense.Xi_blocks(H.points, H.delta)
    for T in range(1, 7):
        r2 = dense.fig2_ratio(H.points, H.delta, H.q, T, Xi=Xi)
        r3 = dense.fig3_ratio(H.points, H.delta, H.q, T, Xi=Xi)
        assert _printed_eq(r2, golden["figure2"][str(L)][T - 1], 5), (L, T, r2)
        assert _printed_eq(r3, golden["figure3"][str(L)][T - 1], 5), (L, T, r3)


@pytest.mark.slow
def test_figure2_and_3_L6(golden):
    H = grid_hierarchy(6)
    Xi = dense.Xi_blocks(H.points, H.delta)
    for T in range(1, 7):
        assert _printed_eq(dense.fig2_ratio(H.points, H.delta, H.q, T, Xi=Xi),
                           golden["figure2"]["6"][T - 1], 5)
        assert _printed_eq(dense.fig3_ratio(H.points, H.delta, H.q, T, Xi=Xi),
                           golden["figure3"]["6"][T - 1], 5)


def test_figure3_needs_value_filter():
    """Reading C-6: counting the purely geometric pattern does NOT reproduce
    Figure 3 (L=3, T=1 gives ~0.0279 instead of 0.03714)."""
    H = grid_hierarchy(3)
    Xi = dense.Xi_blocks(H.points, H.delta)
    geo = dense.fig3_ratio(H.points, H.delta, H.q, 1, Xi=Xi, eps=-1.0)
    assert abs(geo - 0.03714) > 5e-3
