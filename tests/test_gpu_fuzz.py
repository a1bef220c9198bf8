"""Seeded random hierarchies (dimension, Wendland k, level count and sizes,
support multiplier nu, point family incl. non-nested uniform levels, a
translated and scaled domain) through the whole path against the oracle:
alpha per level within the 1e-9 bar, s_L within the kernel-sum rounding bound,
both schedules; patterns of every A_l bit-exact."""
import numpy as np
import pytest

import oracle
from workloads import Hierarchy, franke, halton

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


def _random_hierarchy(seed, small=False):
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.choice([2, 3]))
    k = int(rng.integers(0, 3))
    L = int(rng.integers(2, 4)) if small else int(rng.integers(1, 5))
    n0 = int(rng.integers(20, 60)) if small else int(rng.integers(20, 200))
    growth = (3 if d == 2 else 4) if small else (4 if d == 2 else 6)
    sizes = [int(n0 * growth ** l * rng.uniform(0.8, 1.2)) for l in range(L)]
    nu = float(rng.uniform(2.0, 4.5) if d == 2 else rng.uniform(1.3, 2.2))
    nested = bool(rng.integers(0, 2))
    shift = rng.uniform(-3, 3, size=d)
    scale = float(rng.uniform(0.5, 4.0))
    if nested:
        allp = halton(max(sizes), d)
        pts = [allp[:n] for n in sizes]
    else:  # independent uniform levels (C-17: nesting is not required)
        pts = [rng.random((n, d)) for n in sizes]
    pts = [np.ascontiguousarray(p * scale + shift) for p in pts]
    delta = [nu * scale * (np.sqrt(d) / 2) * n ** (-1.0 / d) for n in sizes]
    q = [0.5 * scale * n ** (-1.0 / d) for n in sizes]
    H = Hierarchy(f"fuzz{seed}", d, k, pts, delta, q, None)
    f = [franke((p - shift) / scale) for p in pts]
    x = np.ascontiguousarray(rng.random((500, d)) * scale + shift)
    return H, f, x


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_against_oracle(msk, ctx, seed):
    H, f, x = _random_hierarchy(seed)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble()
    for l in range(H.L):
        rp, col, _ = h.export_block(l, l)
        orp, ocol = oracle.pattern(H.points[l], H.points[l], H.delta[l], "grid")
        assert np.array_equal(rp, orp) and np.array_equal(col, ocol), (seed, l)
    ao, _, _ = oracle.sequential(H.points, H.delta, f, tol=1e-12, k=H.k, direct_max_n=0)
    so = oracle.evaluate(H.points, H.delta, ao, x, k=H.k)
    scale = oracle.evaluate(H.points, H.delta, [np.abs(a) for a in ao], x, k=H.k)
    for schedule in ("pruned", "literal"):
        a, info = h.solve(f, tol=1e-12, schedule=schedule)
        for l in range(H.L):
            assert np.linalg.norm(a[l] - ao[l]) <= 1e-9 * np.linalg.norm(ao[l]) + 1e-300, (seed, schedule, l)
        s, _ = h.evaluate(x)
        # same coefficients to 1e-9 => values to 1e-9 of the absolute kernel sum
        assert np.all(np.abs(s - so) <= 1e-9 * scale + 1e-300), (seed, schedule)
    h.close()


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_thresholded_against_oracle(msk, ctx, seed):
    """The thresholded path (a6/a7) on random small hierarchies (2-3 levels):
    the factor's nonzero count equals the oracle's geometric count and alpha is
    within the bar (exact Lagrange build)."""
    H, f, x = _random_hierarchy(100 + seed, small=True)
    T = float(np.random.default_rng(seed).choice([1.5, 2.0, 3.0, 5.0]))
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    h.assemble(T=T, lagrange_tol=1e-14)
    a, info = h.solve(f, tol=1e-12)
    ao, _, nnz = oracle.thresholded(H.points, H.delta, H.q, T, f, k=H.k)
    assert info.nnz_gather == nnz
    for l in range(H.L):
        assert np.linalg.norm(a[l] - ao[l]) <= 1e-9 * np.linalg.norm(ao[l]) + 1e-300, (seed, T, l)
    h.close()


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_partitioned_bitwise(msk, ctx, seed):
    """The partitioned solve (single-GPU emulation, every level with enough
    chunks partitioned) on random hierarchies: the persistent peer-memory CG
    (k_pcg) reproduces the single-GPU alpha, iteration counts and s_L bit for
    bit, for a random world size and both schedules; matrix-free hierarchies
    take the phase path and must match as well."""
    H, f, x = _random_hierarchy(200 + seed)
    rng = np.random.default_rng(seed)
    world = int(rng.integers(2, 6))
    flags = msk.MSK_FLAG_MATRIX_FREE if seed % 4 == 3 else 0
    schedule = "literal" if seed % 2 else "pruned"
    out = []
    for c, fl in ((ctx, flags), (msk.Context(0, rank=-1, world=world), flags | msk.MSK_FLAG_DIST_ALL)):
        h = msk.Hierarchy(c, H.points, H.delta, H.q, k=H.k, flags=fl)
        h.assemble()
        a, info = h.solve(f, tol=1e-12, schedule=schedule)
        s, _ = h.evaluate(x)
        out.append((a, list(info.cg_iters)[:H.L], s))
        h.close()
        if c is not ctx:
            c.close()
    (a1, i1, s1), (aw, iw, sw) = out
    assert iw == i1, (seed, world, iw, i1)
    for l in range(H.L):
        assert np.array_equal(aw[l], a1[l]), (seed, world, schedule, l)
    assert np.array_equal(sw, s1)
