"""Local-patch Lagrange factor vs the exact one (msk_assemble vs msk_assemble_ex)
on a hierarchy: max |X~_patch - X~_exact| / max |X~_exact| per block, and the
solve difference.

    python tools/patch_check.py [--config C3P4] [--T 3] [--R 6 8 10 12]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3P4")
    ap.add_argument("--T", type=float, default=3.0)
    ap.add_argument("--R", type=float, nargs="+", default=[6, 8, 10, 12])
    args = ap.parse_args()
    import paper_2503_04914_b200 as msk
    from workloads import config, grid_hierarchy
    H = grid_hierarchy(7) if args.config == "grid7" else config(args.config, m_eval=0)
    ctx = msk.Context(0)
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
    t0 = time.perf_counter()
    h.assemble(T=args.T, lagrange_tol=1e-14)
    t_exact = time.perf_counter() - t0
    ref = {(k, l): h.export_factor(k, l) for k in range(1, H.L) for l in range(k)}
    a_ref, _ = h.solve(H.f())
    for R in args.R:
        t0 = time.perf_counter()
        h.assemble(T=args.T, lagrange_tol=1e-14, patch_R=R, patch_min_n=0)
        t_patch = time.perf_counter() - t0
        err = {}
        for (k, l), (rp, col, val, _) in ref.items():
            rp2, col2, val2, _ = h.export_factor(k, l)
            assert np.array_equal(rp, rp2) and np.array_equal(col, col2)
            err[f"{k}{l}"] = float(np.abs(val2 - val).max() / max(np.abs(val).max(), 1e-300))
        a, _ = h.solve(H.f())
        serr = [float(np.linalg.norm(a[l] - a_ref[l]) / np.linalg.norm(a_ref[l])) for l in range(H.L)]
        print(json.dumps({"config": args.config, "T": args.T, "R": R, "max_rel_err_per_block": err,
                          "alpha_rel_err": serr, "t_exact_s": round(t_exact, 3), "t_patch_s": round(t_patch, 3)}))
    h.close()
    ctx.close()


if __name__ == "__main__":
    main()
