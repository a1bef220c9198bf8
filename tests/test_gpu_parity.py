"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (north_star / DESIGN.md §Parity):
* cell lists, neighbour indices, sparsity patterns: bit-exact;
* kernel values / SpMV: 1e-14 relative (FP64 rounding order only);
* alpha per level and s_L: <= 1e-9 relative L2 at solver tolerance 1e-12
  (reading C-21: per level).
Sizes span several 256-row tiles with ragged tails; configs follow
SURVEY.md §8(d) (C1, C3 prefixes, paper grids).
"""
import numpy as np
import pytest

import oracle
from workloads import config, franke, grid_hierarchy, halton_hierarchy, uniform_points

pytestmark = pytest.mark.gpu

TOL = 1e-12
BAR = 1e-9


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


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - b) / (nb if nb > 0 else 1.0)


def _row_abs_bound(X, Y, delta, v, d):
    """delta^-d sum_{j: |x_i - y_j| < delta} |v_j| per row i: the scale of the
    rounding error of a kernel sum (Phi <= Phi(0) = delta^-d)."""
    rp, col = oracle.pattern(X, Y, delta)
    out = np.zeros(X.shape[0])
    cnt = np.diff(rp)
    if len(col):
        out[cnt > 0] = np.add.reduceat(np.abs(np.asarray(v))[col], rp[:-1][cnt > 0])
    return delta ** -d * out


def _hier(msk, ctx, H, assemble=True):
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    if assemble:
        h.assemble()
    return h


HIERS = {
    "C1": lambda: config("C1"),
    "grid5": lambda: grid_hierarchy(5),
    "halton3d": lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5),
    "halton2d_k0": lambda: halton_hierarchy("h2k0", 2, [97, 1001, 4097], 4.0, k=0),
    "halton3d_k2": lambda: halton_hierarchy("h3k2", 3, [77, 1299, 5003], 2.0, k=2),
}


# --------------------------------------------------------------- a1 cell list
def _assert_keys_exact(P, c):
    """Every sorted point's key equals the key map recomputed here from the
    exported grid: floor((x_a - lo_a) * inv_cell[a]) per axis with one rounded
    subtraction and one rounded multiplication (numpy evaluates each ufunc
    separately, so no FMA: reading C-4), clamped to the grid, row-major
    x-major (reading C-26); the last axis has thin cells (inv_cell[-1] = zf x
    inv_cell[0], zf a power of two).  Bit-exact, no tolerance."""
    Ps = P[c["perm"]]
    dims = np.asarray(c["dims"], dtype=np.int64)
    cc = np.floor((Ps - np.asarray(c["lo"])) * c["inv_cell"]).astype(np.int64)
    cc = np.clip(cc, 0, dims - 1)
    key = cc[:, 0]
    for a in range(1, P.shape[1]):
        key = key * dims[a] + cc[:, a]
    assert np.array_equal(key, c["keys"])
    # the key map is the grid the cell side describes; the last axis is refined by a power of two
    inv = np.asarray(c["inv_cell"])
    assert abs(inv[0] * c["cell"] - 1.0) < 1e-15 and np.all(inv[:-1] == inv[0])
    zf = inv[-1] / inv[0]
    assert zf in (1.0, 2.0, 4.0, 8.0)



@pytest.mark.parametrize("name", ["C1", "halton3d", "grid5"])
def test_cell_list_structure(msk, ctx, name):
    H = HIERS[name]()
    h = _hier(msk, ctx, H, assemble=False)
    for l in range(H.L):
        c = h.export_cells(l)
        perm, keys, cs = c["perm"], c["keys"], c["cell_start"]
        P = H.points[l]
        assert np.array_equal(np.sort(perm), np.arange(H.n[l]))          # permutation
        assert np.all(np.diff(keys) >= 0)                                # sorted by key
        same = keys[1:] == keys[:-1]
        assert np.all(perm[1:][same] > perm[:-1][same])                  # ties by caller index
        assert cs[0] == 0 and cs[-1] == H.n[l] and np.all(np.diff(cs) >= 0)
        _assert_keys_exact(P, c)
        assert c["cell"] >= H.delta[l]


# ------------------------------------------------------------ a2 patterns
@pytest.mark.parametrize("name", list(HIERS))
def test_pattern_bitexact_and_values(msk, ctx, name):
    H = HIERS[name]()
    h = _hier(msk, ctx, H)
    for rl in range(H.L):
        for cl in range(rl + 1):
            rp, col, val = h.export_block(rl, cl)
            orp, ocol = oracle.pattern(H.points[rl], H.points[cl], H.delta[cl], "brute")
            assert np.array_equal(rp, orp), (rl, cl)
            assert np.array_equal(col, ocol), (rl, cl)
            _, _, oval = oracle.block(H.points[rl], H.points[cl], H.delta[cl], k=H.k)
            # entries are Phi = delta^-d phi(r/delta); near r = delta the factor
            # (1 - r/delta) cancels, so the bar is relative to Phi(0) = delta^-d
            np.testing.assert_allclose(val, oval, rtol=0, atol=1e-14 * H.delta[cl] ** -H.d)
    info = h.info()
    for l in range(H.L):
        orp, _ = oracle.pattern(H.points[l], H.points[l], H.delta[l], "grid")
        assert info.nnz_A[l] == orp[-1]


def test_pattern_C3_prefix_level3(msk, ctx):
    """19,531-point 3-D level of C3 (77 tiles, ragged tail): bit-exact."""
    H = config("C3P4", m_eval=0)
    h = _hier(msk, ctx, H)
    rp, col, _ = h.export_block(2, 2)
    orp, ocol = oracle.pattern(H.points[2], H.points[2], H.delta[2], "brute")
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol)
    rp, col, _ = h.export_block(3, 1)
    orp, ocol = oracle.pattern(H.points[3], H.points[1], H.delta[1], "grid")
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol)


# -------------------------------------------------------------- a3 SpMV
@pytest.mark.parametrize("name", ["C1", "halton3d", "halton3d_k2"])
def test_spmv_assembled_and_matrix_free(msk, ctx, name):
    H = HIERS[name]()
    h = _hier(msk, ctx, H)
    rng = np.random.default_rng(5)
    for rl in range(H.L):
        for cl in range(rl + 1):
            v = rng.standard_normal(H.n[cl])
            y, _ = h.apply_block(rl, cl, v)
            ref = oracle.apply(H.points[rl], H.points[cl], H.delta[cl], v, k=H.k)
            # per-entry error <= c eps Phi(0) (cancellation in 1 - r/delta near
            # the support boundary), so the bar is 1e-14 delta^-d sum_row |v_j|
            scale = _row_abs_bound(H.points[rl], H.points[cl], H.delta[cl], v, H.d)
            bad = np.abs(y - ref) > 1e-14 * scale + 1e-300
            assert not bad.any(), (rl, cl, np.flatnonzero(bad)[:5], y[bad][:5], ref[bad][:5],
                                   scale[bad][:5])


# -------------------------------------------------------------- a4 CG
@pytest.mark.parametrize("name", ["C1", "halton3d"])
def test_cg_level(msk, ctx, name):
    H = HIERS[name]()
    h = _hier(msk, ctx, H)
    for l in range(H.L):
        b = franke(H.points[l])
        x, it, rr, _ = h.cg_level(l, b, tol=TOL)
        rp, col, val = oracle.block(H.points[l], H.points[l], H.delta[l], k=H.k)
        xo, ito, st = oracle.cg(rp, col, val, b, TOL)
        assert st == 0 and abs(it - ito) <= 2 and rr <= TOL
        assert _rel(x, xo) < BAR
        if len(H.points[l]) <= 5000:  # the oracle's dense Cholesky is O(n^3) in plain C (n = 9999: ~160 s)
            xd = oracle.cholesky_solve(rp, col, val, b)
            assert _rel(x, xd) < BAR and _rel(xo, xd) < BAR
        # the returned x satisfies the stopping rule on the true residual
        assert np.linalg.norm(oracle.spmv(rp, col, val, x) - b) <= 10 * TOL * np.linalg.norm(b)


def test_cg_zero_rhs_and_noconv(msk, ctx):
    H = HIERS["C1"]()
    h = _hier(msk, ctx, H)
    x, it, rr, _ = h.cg_level(2, np.zeros(H.n[2]))
    assert it == 0 and not np.any(x)
    with pytest.raises(msk.MskError) as ei:
        h.cg_level(2, franke(H.points[2]), tol=1e-14, max_iter=2)
    assert ei.value.status == 5 and "level 2" in str(ei.value)


@pytest.mark.parametrize("name,levels", [("C1", [0, 1, 2]), ("grid5", [0, 1, 2, 3, 4]),
                                         ("halton3d", [0, 1])])
@pytest.mark.parametrize("schedule", ["pruned", "literal"])
def test_kappa_estimate(msk, ctx, name, levels, schedule):
    """kappa(A_l) estimated from the CG coefficients (Lanczos
    tridiagonal) of the solve that produced alpha_l, against the dense
    spectrum lambda_max / lambda_min of A_l (oracle.dense).  Ritz values lie
    inside [lambda_min, lambda_max], so the estimate is a lower bound; with a
    smooth right-hand side the extreme eigenvectors are weakly excited, so it
    is within 10 %, not exact."""
    from oracle import dense
    H = HIERS[name]()
    h = _hier(msk, ctx, H)
    _, info = h.solve(H.f(), tol=TOL, schedule=schedule)
    for l in levels:
        ev = np.linalg.eigvalsh(dense.kernel_matrix(H.points[l], H.points[l], H.delta[l], k=H.k))
        kap = ev[-1] / ev[0]
        assert info.cg_iters[l] > 0
        assert 0.9 * kap <= info.kappa_est[l] <= kap * (1 + 1e-9), (l, info.kappa_est[l], kap)


# -------------------------------------------------------------- full solve
@pytest.mark.parametrize("name", list(HIERS))
@pytest.mark.parametrize("schedule", ["pruned", "literal"])
def test_solve_matches_oracle(msk, ctx, name, schedule):
    H = HIERS[name]()
    h = _hier(msk, ctx, H)
    f = H.f()
    alpha, info = h.solve(f, tol=TOL, schedule=schedule)
    a_or, _, _ = oracle.sequential(H.points, H.delta, f, tol=TOL, k=H.k, direct_max_n=0)
    a_ex, _, _ = oracle.sequential(H.points, H.delta, f, k=H.k, direct_max_n=3000)
    for l in range(H.L):
        assert _rel(alpha[l], a_or[l]) < BAR, (l, _rel(alpha[l], a_or[l]))
        assert _rel(alpha[l], a_ex[l]) < BAR
        assert info.rel_res[l] <= TOL
    assert info.nnz_cg > 0 and info.t_cg_ms > 0
    # evaluation: GPU s_L vs oracle eq:fapproximation with the same alpha
    x = uniform_points(3000, H.d, seed=9)
    s, einfo = h.evaluate(x)
    so = oracle.evaluate(H.points, H.delta, alpha, x, k=H.k)
    scale = sum(_row_abs_bound(x, P, dl, a, H.d) for P, dl, a in zip(H.points, H.delta, alpha))
    assert np.all(np.abs(s - so) <= 1e-14 * scale + 1e-300)
    s_or = oracle.evaluate(H.points, H.delta, a_or, x, k=H.k)
    assert _rel(s, s_or) < BAR
    # hit counts of the matrix-free kernels == exact pattern sizes (the FP32
    # prefilter never drops a pair inside the support)
    ev_nnz = sum(int(oracle.pattern(x, P, dl)[0][-1]) for P, dl in zip(H.points, H.delta))
    assert einfo.nnz == ev_nnz
    b_nnz = sum(int(oracle.pattern(H.points[k], H.points[l], H.delta[l])[0][-1])
                for k in range(H.L) for l in range(k))
    sweeps = H.L if schedule == "literal" else 1
    assert info.nnz_gather == sweeps * b_nnz


def test_pruned_equals_literal(msk, ctx):
    H = HIERS["halton3d"]()
    h = _hier(msk, ctx, H)
    f = H.f()
    a1, i1 = h.solve(f, tol=TOL, schedule="pruned")
    a2, i2 = h.solve(f, tol=TOL, schedule="literal")
    for l in range(H.L):
        assert _rel(a1[l], a2[l]) < BAR
    assert i2.jacobi_sweeps == H.L and sum(i2.inner_iters) > sum(i1.inner_iters)
    # the finest level sees bit-identical beta in both schedules and is solved
    # at the same tolerance by the same deterministic kernel
    assert np.array_equal(a1[-1], a2[-1])


def test_deterministic_repeat(msk, ctx):
    H = HIERS["C1"]()
    h = _hier(msk, ctx, H)
    f = H.f()
    a1, _ = h.solve(f)
    a2, _ = h.solve(f)
    h2 = _hier(msk, ctx, H)
    a3, _ = h2.solve(f)
    for l in range(H.L):
        assert np.array_equal(a1[l], a2[l]) and np.array_equal(a1[l], a3[l])


def test_interpolation_property_on_levels(msk, ctx):
    """f_L = f on every X_l of a nested hierarchy."""
    H = HIERS["halton3d"]()
    h = _hier(msk, ctx, H)
    f = H.f()
    h.solve(f, tol=1e-13)
    for l in range(H.L):
        s, _ = h.evaluate(H.points[l])
        assert np.abs(s - f[l]).max() < 1e-9 * np.abs(f[l]).max()


def test_torch_device_buffers_match_host(msk, ctx):
    import torch
    H = HIERS["C1"]()
    h = _hier(msk, ctx, H)
    f = H.f()
    a_host, _ = h.solve(f)
    fd = [torch.from_numpy(x).cuda() for x in f]
    a_dev, _ = h.solve(fd)
    for l in range(H.L):
        assert np.array_equal(a_dev[l].cpu().numpy(), a_host[l])
    x = torch.from_numpy(uniform_points(1000, 2, seed=1)).cuda()
    s_dev, _ = h.evaluate(x)
    s_host, _ = h.evaluate(x.cpu().numpy())
    assert np.array_equal(s_dev.cpu().numpy(), s_host)
    hd = msk.Hierarchy(ctx, [torch.from_numpy(p).cuda() for p in H.points], H.delta, H.q)
    hd.assemble()
    a3, _ = hd.solve(f)
    for l in range(H.L):
        assert np.array_equal(a3[l], a_host[l])


@pytest.mark.parametrize("chunk", ["257", "4096", "1048576"])
def test_pipelined_host_evaluate(msk, ctx, chunk, monkeypatch):
    """Host buffers: s_L is evaluated in chunks with the copies overlapped
    (copy streams); every value must equal the device-buffer path's, for
    chunkings with ragged tails (MSK_EVAL_CHUNK is a test hook)."""
    import torch
    H = HIERS["halton3d"]()
    h = _hier(msk, ctx, H)
    h.solve(H.f())
    xh = uniform_points(20_011, 3, seed=9)
    s_dev, e_dev = h.evaluate(torch.from_numpy(xh).cuda())
    monkeypatch.setenv("MSK_EVAL_CHUNK", chunk)
    s_host, e_host = h.evaluate(xh)
    assert np.array_equal(s_dev.cpu().numpy(), s_host)
    assert e_host.nnz == e_dev.nnz
    ref = oracle.evaluate(H.points, H.delta, [h_ for h_ in h.solve(H.f())[0]], xh[:500], k=H.k)
    assert _rel(s_host[:500], ref) < 1e-12


# -------------------------------------------------------------- edge cases
def test_edge_cases(msk, ctx):
    H = HIERS["C1"]()
    # single level == plain interpolation
    h1 = msk.Hierarchy(ctx, [H.points[0]], [H.delta[0]])
    with pytest.raises(msk.MskError) as ei:
        h1.solve([franke(H.points[0])])
    assert ei.value.status == 6                      # solve before assemble
    h1.assemble()
    with pytest.raises(msk.MskError) as ei:
        h1.evaluate(H.points[0])
    assert ei.value.status == 6                      # evaluate before solve
    a, _ = h1.solve([franke(H.points[0])])
    rp, col, val = oracle.block(H.points[0], H.points[0], H.delta[0])
    assert _rel(a[0], oracle.cholesky_solve(rp, col, val, franke(H.points[0]))) < BAR
    s, _ = h1.evaluate(np.zeros((0, 2)))
    assert s.shape == (0,)
    # zero right-hand side
    h = _hier(msk, ctx, H)
    a, info = h.solve([np.zeros(n) for n in H.n])
    assert all(not np.any(x) for x in a) and list(info.cg_iters)[:3] == [0, 0, 0]
    # one-point level and a level far from the others
    pts = [np.array([[0.5, 0.5]]), H.points[1]]
    h3 = msk.Hierarchy(ctx, pts, [0.3, H.delta[1]])
    h3.assemble()
    f = [franke(p) for p in pts]
    a, _ = h3.solve(f)
    ao, _, _ = oracle.sequential(pts, [0.3, H.delta[1]], f, direct_max_n=10 ** 6)
    for l in range(2):
        assert _rel(a[l], ao[l]) < BAR
    # invalid arguments
    dup = np.vstack([H.points[0], H.points[0][:1]])
    with pytest.raises(msk.MskError) as ei:
        msk.Hierarchy(ctx, [dup], [0.2])
    assert ei.value.status == 1
    with pytest.raises(msk.MskError):
        msk.Hierarchy(ctx, [H.points[0]], [-1.0])
    with pytest.raises(msk.MskError):
        msk.Hierarchy(ctx, [np.zeros((3, 4))], [0.1])
    with pytest.raises(msk.MskError) as ei:             # empty level
        msk.Hierarchy(ctx, [H.points[0], np.zeros((0, 2))], [0.2, 0.1])
    assert ei.value.status == 1
    with pytest.raises(msk.MskError):
        h.solve(H.f(), tol=1.5)


def test_c_example_runs(tmp_path):
    """The C-ABI from plain C (examples/msk_example.c): host buffers, the
    interpolation property s_L = f on X_L within 1e-10."""
    import json
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2503_04914_b200")
    exe = str(tmp_path / "msk_example")
    subprocess.check_call(["gcc", "-std=c99", "-O2", os.path.join(root, "examples", "msk_example.c"),
                           "-I", os.path.join(root, "include"), "-L", libdir, "-lmsk",
                           f"-Wl,-rpath,{libdir}", "-lm", "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    assert out["points"] == [9, 25, 81] and out["max_interpolation_error"] < 1e-10


def test_failed_reassemble_leaves_state_error(msk, ctx):
    """A failed msk_assemble after a successful one leaves the hierarchy
    unassembled: msk_solve must report MSK_ERR_STATE (never run on a half-built
    factor or freed CSR arrays) until the next successful msk_assemble."""
    H = HIERS["C1"]()
    h = _hier(msk, ctx, H)
    f = H.f()
    a0, _ = h.solve(f, tol=TOL)
    with pytest.raises(msk.MskError) as ei:   # Lagrange CG cannot reach 1e-300
        h.assemble(T=3.0, lagrange_tol=1e-300)
    assert ei.value.status == 5
    with pytest.raises(msk.MskError) as ei:
        h.solve(f, tol=TOL)
    assert ei.value.status == 6
    h.assemble()
    a1, _ = h.solve(f, tol=TOL)
    for l in range(H.L):
        assert np.array_equal(a0[l], a1[l])


@pytest.mark.parametrize("delta_scale", [1.0, 0.05])
def test_q_null_is_exact_half_min_distance(msk, ctx, delta_scale):
    """q = NULL: the library reports q_l = 1/2 min_{j != k} ||x_j - x_k||
     exactly -- the oracle's brute-force separation (pinned by
    Table 1 in test_oracle_pattern) -- also when delta_l is below the
    separation (no pair within the support: widening cell search)."""
    H = HIERS["C1"]()
    delta = [dl * delta_scale for dl in H.delta]
    h = msk.Hierarchy(ctx, H.points, delta, None, k=H.k)
    info = h.info()
    for l in range(H.L):
        q = oracle.separation(H.points[l])
        if delta_scale < 1:
            assert 2 * q >= delta[l]          # the case the widening search exists for
        assert abs(info.q[l] - q) <= 1e-15 * q, (l, info.q[l], q)
