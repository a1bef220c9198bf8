"""Truncation diagnostics on the GPU (msk_m_norm).

||M_L||_2 of Figure 1 by power iteration with M and M^T
applied matrix-free (CG solves + kernel sums, incl. the transposed B^T
products).  Pinned to the paper's printed values (tests/golden/, every printed
digit, L = 2..7) and to the dense oracle (L <= 5, 1e-7 relative).
"""
import json
import os

import numpy as np
import pytest

from workloads import grid_hierarchy, halton_hierarchy

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


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


def _printed_eq(v, printed, digits=3):
    return abs(v - printed) <= 0.5 * 10 ** -digits + 1e-12


@pytest.mark.parametrize("L", [2, 3, 4, 5, 6, 7])
def test_figure1_norm_matches_paper(msk, ctx, L):
    H = grid_hierarchy(L)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    nrm, it = h.m_norm(max_iter=2000, rel_tol=1e-10)
    assert _printed_eq(nrm, GOLDEN["figure1"]["numerical"][str(L)]), (L, nrm, it)
    h.close()


@pytest.mark.parametrize("name", ["grid4", "halton2d", "halton3d"])
def test_m_norm_matches_dense_oracle(msk, ctx, name):
    from oracle import dense
    H = {"grid4": lambda: grid_hierarchy(4),
         "halton2d": lambda: halton_hierarchy("h2", 2, [60, 240, 960], 4.0),
         "halton3d": lambda: halton_hierarchy("h3", 3, [80, 640, 2000], 1.5)}[name]()
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    nrm, it = h.m_norm(max_iter=3000, rel_tol=1e-12)
    ref = dense.fig1_norm(H.points, H.delta, H.k)
    assert abs(nrm / ref - 1) < 1e-7, (name, nrm, ref, it)
    h.close()


def test_m_norm_single_level_is_zero(msk, ctx):
    H = grid_hierarchy(1)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    assert h.m_norm()[0] == 0.0
    h.close()


@pytest.mark.parametrize("L", [3, 4, 5, 6, 7])
def test_figure2_ratio_matches_paper(msk, ctx, L):
    """||M_L - M~_L(T)||_2 / ||M_L||_2, T = 1..6: every
    printed digit, with the stored thresholded factor (a6) and its transpose;
    L = 7 is beyond the dense oracle."""
    H = grid_hierarchy(L)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    m, _ = h.m_norm(max_iter=2000, rel_tol=1e-11)
    got = []
    for T in range(1, 7):
        h.assemble(T=float(T), lagrange_tol=1e-14)
        d, it = h.m_diff_norm(max_iter=3000, rel_tol=1e-11)
        got.append(d / m)
    want = GOLDEN["figure2"][str(L)]
    for T, (g, w) in enumerate(zip(got, want), start=1):
        assert _printed_eq(g, w, 5), (L, T, g, w)
    h.close()


@pytest.mark.parametrize("L", [3, 4, 5, 6])
def test_figure3_nnz_ratio_matches_paper(msk, ctx, L):
    """nnz(M~_L(T)) / nnz(M_L), T = 1..6, entries counted
    as |v| > 1e-8 (reading C-6) from the stored factor; T = 1e9 keeps every
    entry of X (the denominator)."""
    def count(h):
        return sum(int(np.count_nonzero(np.abs(h.export_factor(k, l)[2]) > 1e-8))
                   for k in range(1, L) for l in range(k))
    H = grid_hierarchy(L)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble(T=1e9, lagrange_tol=1e-14)
    den = count(h)
    want = GOLDEN["figure3"][str(L)]
    for T in range(1, 7):
        h.assemble(T=float(T), lagrange_tol=1e-14)
        assert _printed_eq(count(h) / den, want[T - 1], 5), (L, T)
    h.close()


@pytest.mark.parametrize("L", [5, 6])
def test_figures_2_3_from_one_build(msk, ctx, L):
    """Figures 2 and 3 from ONE factor build (T = 1e9, every entry of X) swept
    with msk_set_threshold(T), T = 1..6: every printed digit of PAPER.md:
    1365-1413 and 1439-1487, as with a build per T."""
    H = grid_hierarchy(L)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    m, _ = h.m_norm(max_iter=2000, rel_tol=1e-11)
    h.assemble(T=1e9, lagrange_tol=1e-14)

    def count():
        return sum(int(np.count_nonzero(np.abs(h.export_factor(k, l)[2]) > 1e-8))
                   for k in range(1, L) for l in range(k))
    den = count()
    for T in range(1, 7):
        h.set_threshold(float(T))
        d, _ = h.m_diff_norm(max_iter=3000, rel_tol=1e-11)
        assert _printed_eq(d / m, GOLDEN["figure2"][str(L)][T - 1], 5), (L, T, d / m)
        assert _printed_eq(count() / den, GOLDEN["figure3"][str(L)][T - 1], 5), (L, T)
    h.set_threshold(1e9)
    assert count() == den
    h.close()


def test_m_diff_norm_needs_a_factor(msk, ctx):
    H = grid_hierarchy(3)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    with pytest.raises(msk.MskError) as ei:
        h.m_diff_norm()
    assert ei.value.status == 6
    h.close()
