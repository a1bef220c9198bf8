"""Parity at BASELINE.json's full size (config C3: 6 levels, 11.4M points,
~1.06e8 nonzeros, 10^7 evaluation points), in the launch configuration
bench.py times (device buffers, PRUNED schedule, tol 1e-12): sampled outputs
checked one by one against the oracle.

* alpha: rows of eq:mas recomputed by brute force in the oracle
  (mo_mas_row_residual: sum over every point of the levels <= l, no cell
  list) from the GPU coefficients -- the residual must be at solver level;
* s_L: sampled evaluation points against oracle.evaluate from the same
  coefficients (1e-12 relative to the absolute kernel sum).
"""
import numpy as np
import pytest

import oracle
from workloads import config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solved():
    import torch
    import paper_2503_04914_b200 as msk
    msk.load()
    H = config("C3")
    dev = torch.device("cuda", 0)
    ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream)
    h = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k)
    h.assemble()
    f = H.f()
    a, info = h.solve([torch.from_numpy(v).to(dev) for v in f], tol=1e-12)
    s, einfo = h.evaluate(torch.from_numpy(H.eval_points).to(dev))
    out = (H, f, [v.cpu().numpy() for v in a], s.cpu().numpy(), info, einfo)
    h.close()
    ctx.close()
    return out


def test_full_size_counts(solved):
    H, f, a, s, info, einfo = solved
    assert H.L == 6 and sum(H.n) == 11_428_527
    assert all(0 < it < 200 for it in info.cg_iters[:6])
    assert all(r <= 1e-12 for r in info.rel_res[:6])
    assert 1.0e8 < einfo.nnz < 1e9


@pytest.mark.parametrize("level", range(6))
def test_full_size_mas_rows(solved, level):
    H, f, a, s, info, einfo = solved
    rng = np.random.default_rng(level)
    rows = rng.choice(H.n[level], size=6 if level == 5 else 12, replace=False)
    fn = np.linalg.norm(f[level])
    for j in rows:
        r, absrow = oracle.mas_row_residual(H.points, H.delta, a, level, int(j), float(f[level][j]), k=H.k)
        # CG stops at ||r||_2 <= 1e-12 ||beta_l||_2 <~ 1e-12 ||f_l||_2 (reading C-9): the
        # residual of any one row is below that; 10x margin plus the rounding of the row sum
        assert abs(r) <= 1e-11 * fn + 1e-13 * absrow, (level, j, r, absrow, fn)


def test_full_size_evaluation_samples(solved):
    H, f, a, s, info, einfo = solved
    rng = np.random.default_rng(7)
    idx = rng.choice(H.eval_points.shape[0], size=64, replace=False)
    x = H.eval_points[idx]
    ref = oracle.evaluate(H.points, H.delta, a, x, k=H.k)
    # rounding scale of each kernel sum: the same sum with |alpha| (Phi >= 0)
    scale = oracle.evaluate(H.points, H.delta, [np.abs(v) for v in a], x, k=H.k)
    err = np.abs(s[idx] - ref)
    assert np.all(err <= 1e-12 * scale), (err.max(), scale[err.argmax()])
