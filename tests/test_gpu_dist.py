"""Partitioned (multi-GPU) path, run as the single-process emulation on one
GPU: `world` partitions per level with separate buffers; chunk partials and r
halos exchanged either inside one persistent launch over "peer" stores (k_pcg,
the path of a real multi-GPU job) or by host-driven phase kernels (DESIGN.md
§Multi-GPU).

Because every partial is formed per chunk exactly as in the single-GPU
kernel and summed over all chunks in the same order, the partitioned solve
must reproduce the single-GPU alpha and s_L BIT FOR BIT for any world size.
The oracle bar (1e-9 per level) then carries over.
"""
import numpy as np
import pytest

import oracle
from workloads import config, halton_hierarchy, uniform_points

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def msk():
    import paper_2503_04914_b200 as m
    m.load()
    return m


HIERS = {
    "C1": lambda: config("C1", m_eval=0),
    "halton3d": lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5),
    "C3P4": lambda: config("C3P4", m_eval=0),
}


def _solve(msk, ctx, H, flags, f, x):
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=flags)
    h.assemble()
    a, info = h.solve(f, tol=1e-12)
    s, einfo = h.evaluate(x)
    return a, s, info, einfo


@pytest.mark.parametrize("name", list(HIERS))
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("path", ["p2p", "phase"])
def test_partitioned_equals_single_gpu_bitwise(msk, name, world, path, monkeypatch):
    """path p2p: the whole CG of a partitioned level in one launch over peer
    memory (k_pcg: partials and r halos stored into the other partitions'
    buffers, device-side cross-partition barrier); path phase: host-driven phase
    kernels with the partials summed and the halos copied between launches."""
    monkeypatch.setenv("MSK_DIST_P2P", "1" if path == "p2p" else "0")
    H = HIERS[name]()
    f = H.f()
    x = uniform_points(5000, H.d, seed=4)
    c1 = msk.Context(0)
    a1, s1, i1, e1 = _solve(msk, c1, H, 0, f, x)
    cw = msk.Context(0, rank=-1, world=world)
    aw, sw, iw, ew = _solve(msk, cw, H, msk.MSK_FLAG_DIST_ALL, f, x)
    for l in range(H.L):
        assert np.array_equal(aw[l], a1[l]), (name, world, l, np.abs(aw[l] - a1[l]).max())
        assert iw.cg_iters[l] == i1.cg_iters[l]
        assert iw.kappa_est[l] == i1.kappa_est[l]
    assert np.array_equal(sw, s1)
    assert ew.nnz == e1.nnz
    c1.close()
    cw.close()


def test_partitioned_matches_oracle_and_default_threshold(msk):
    """C3 4-level prefix: with the default threshold no level is partitioned;
    with DIST_ALL every level with >= world chunks is.  Both match the oracle
    within the 1e-9 bar."""
    H = config("C3P4", m_eval=0)
    f = H.f()
    cw = msk.Context(0, rank=-1, world=4)
    for flags in (0, msk.MSK_FLAG_DIST_ALL):
        h = msk.Hierarchy(cw, H.points, H.delta, H.q, k=1, flags=flags)
        h.assemble()
        a, _ = h.solve(f)
        ao, _, _ = oracle.sequential(H.points, H.delta, f, tol=1e-12, direct_max_n=0)
        for l in range(H.L):
            assert np.linalg.norm(a[l] - ao[l]) <= 1e-9 * np.linalg.norm(ao[l])
    with pytest.raises(msk.MskError) as ei:
        h.cg_level(3, f[3])
    assert ei.value.status == 6
    cw.close()


@pytest.mark.parametrize("name,T,patch_R", [("C1", 2.0, 0.0), ("halton3d", 3.0, 0.0), ("C3P4", 2.0, 0.0),
                                             ("halton3d", 3.0, 9.0)])
@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_thresholded_equals_single_gpu_bitwise(msk, name, T, patch_R, world):
    """a6/a7 in a distributed context: the factor build is
    replicated, the thresholded Jacobi runs on each partition's rows of the
    partitioned levels and the CG of those levels is the partitioned CG; alpha,
    iterations and the stored factor equal the single-GPU thresholded solve bit
    for bit."""
    H = HIERS[name]()
    f = H.f()
    res = []
    for ctx, flags in ((msk.Context(0), 0), (msk.Context(0, rank=-1, world=world), msk.MSK_FLAG_DIST_ALL)):
        h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=flags)
        # patch_R > 0: local-patch Lagrange functions for the column levels above 1000 points
        h.assemble(T=T, lagrange_tol=1e-14, patch_R=patch_R, patch_min_n=1000)
        a, info = h.solve(f, tol=1e-12)
        fac = [h.export_factor(k, l) for k in range(1, H.L) for l in range(k)]
        # the T sweep works on the distributed factor as well
        h.set_threshold(1.0)
        a1, _ = h.solve(f, tol=1e-12)
        res.append((a, info, fac, a1, h.info().nnz_A))
        h.close()
        ctx.close()
    (a, i, fac, a1, nA), (aw, iw, facw, a1w, nAw) = res
    for l in range(H.L):
        assert np.array_equal(aw[l], a[l]), (name, world, l, np.abs(aw[l] - a[l]).max())
        assert np.array_equal(a1w[l], a1[l])
        assert iw.cg_iters[l] == i.cg_iters[l]
    assert list(nAw) == list(nA)
    for x, y in zip(fac, facw):
        assert all(np.array_equal(u, v) for u, v in zip(x[:3], y[:3]))


@pytest.mark.parametrize("name", ["halton3d", "C3P4"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("path", ["p2p", "phase"])
def test_partitioned_literal_schedule_bitwise(msk, name, world, path, monkeypatch):
    """The LITERAL schedule (Algorithm 2 as printed: L sweeps of
    inner solves on levels 1..L-1 + B products, then the block CG) with
    partitioned levels: every inner and final solve of a partitioned level is
    the partitioned CG; bit-identical to the single-GPU literal solve."""
    monkeypatch.setenv("MSK_DIST_P2P", "1" if path == "p2p" else "0")
    H = HIERS[name]()
    f = H.f()
    out = []
    for ctx, flags in ((msk.Context(0), 0), (msk.Context(0, rank=-1, world=world), msk.MSK_FLAG_DIST_ALL)):
        h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=flags)
        h.assemble()
        a, info = h.solve(f, tol=1e-12, schedule="literal")
        out.append((a, list(info.cg_iters)[:H.L], list(info.inner_iters)[:H.L], info.jacobi_sweeps))
        h.close()
        ctx.close()
    (a1, i1, n1, s1), (aw, iw, nw, sw) = out
    assert sw == s1 == H.L and iw == i1 and nw == n1
    for l in range(H.L):
        assert np.array_equal(aw[l], a1[l]), (name, world, l)
