"""Figures 2 and 3 on the GPU at L = 3..Lmax (the dense oracle stops at 6):
||M - M~(T)||_2 / ||M||_2 (msk_m_norm_ex) and nnz(M~(T)) / nnz(M) with the
entries counted as |v| > 1e-8 (reading C-6) from the stored factor
(msk_export_factor; T = 1e9 keeps every entry: the denominator), next to the
printed values.

    python tools/fig23_extend.py [--Lmax 7]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def count_entries(h, L, eps=1e-8):
    tot = 0
    for k in range(1, L):
        for l in range(k):
            _, _, val, _ = h.export_factor(k, l)
            tot += int(np.count_nonzero(np.abs(val) > eps))
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Lmin", type=int, default=3)
    ap.add_argument("--Lmax", type=int, default=7)
    args = ap.parse_args()
    import paper_2503_04914_b200 as msk
    from workloads import grid_hierarchy
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    golden = json.load(open(os.path.join(root, "tests", "golden", "paper_values.json")))
    ctx = msk.Context(0)
    for L in range(args.Lmin, args.Lmax + 1):
        t0 = time.perf_counter()
        H = grid_hierarchy(L)
        h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
        h.assemble(T=1e9, lagrange_tol=1e-14)      # every entry of X: the Figure 3 denominator
        den = count_entries(h, L)
        m, _ = h.m_norm(max_iter=3000, rel_tol=1e-11)
        fig2, fig3 = [], []
        for T in range(1, 7):
            h.assemble(T=float(T), lagrange_tol=1e-14)
            d, _ = h.m_diff_norm(max_iter=3000, rel_tol=1e-11)
            fig2.append(d / m)
            fig3.append(count_entries(h, L) / den)
        row = {"L": L, "points": int(sum(H.n)), "norm_M": m, "nnz_M_eps1e-8": den,
               "fig2": fig2, "fig2_paper": golden["figure2"].get(str(L)),
               "fig3": fig3, "fig3_paper": golden["figure3"].get(str(L)),
               "seconds": round(time.perf_counter() - t0, 2)}
        print(json.dumps(row), flush=True)
        h.close()
    ctx.close()


if __name__ == "__main__":
    main()
