"""Figure 1 on the GPU, extended beyond the paper's L = 7 (the paper's
Python analysis stopped there): ||M_L||_2 by msk_m_norm on the paper grids
(Table 1, nu = 4, phi_(3,1)), next to the printed values and the bound curve
sqrt(L) 2^(L-1) (reading C-23).

    python tools/fig1_extend.py [--Lmax 10]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Lmax", type=int, default=10)
    args = ap.parse_args()
    import paper_2503_04914_b200 as msk
    from workloads import grid_hierarchy
    golden = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "tests", "golden", "paper_values.json")))["figure1"]
    ctx = msk.Context(0)
    rows = []
    for L in range(2, args.Lmax + 1):
        H = grid_hierarchy(L)
        h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k)
        h.assemble()
        t0 = time.perf_counter()
        nrm, it = h.m_norm(max_iter=5000, rel_tol=1e-10)
        dt = time.perf_counter() - t0
        row = {"L": L, "points": int(sum(H.n)), "norm": nrm, "power_iters": it, "seconds": round(dt, 3),
               "paper": golden["numerical"].get(str(L)), "bound_sqrtL_2^(L-1)": math.sqrt(L) * 2.0 ** (L - 1),
               "ratio_to_previous": nrm / rows[-1]["norm"] if rows else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
        h.close()
    ctx.close()


if __name__ == "__main__":
    main()
