"""Config C4 science outputs on ALL of C3 (local-patch Lagrange build, NEXT-4):
for T = 1..Tmax the thresholded solve against the exact one -- nnz of the
stored factor, build and solve time, per-level relative alpha error,
||s~_L - s_L||_inf and ||f - s~_L||_inf vs ||f - s_L||_inf on uniform
evaluation points (SURVEY §8(c) "What to expect in C4") -- and the Theorem
decayerror quantities: ||beta - beta~||_2 (beta_l = A_l alpha_l,
by msk_apply_block), ||M||_2, ||M - M~(T)||_2, ||M~(T)||_2 (msk_m_norm_ex) and
the corrected Lemma pert1 bound (reading C-22)
    ||beta - beta~|| <= ||f|| ||M - M~|| sum_{k=1}^{L-1} k max(||M||, ||M~||)^(k-1).

    python tools/c4_sweep.py [--Tmax 4] [--m-eval 1000000]
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
    ap.add_argument("--config", default="C4F")
    ap.add_argument("--Tmax", type=int, default=4)
    ap.add_argument("--m-eval", type=int, default=1_000_000)
    ap.add_argument("--norms", action="store_true", help="also the power-iteration norms and the pert1 bound")
    ap.add_argument("--norm-iters", type=int, default=60)
    args = ap.parse_args()
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config, franke, uniform_points
    H = config(args.config, m_eval=0)
    dev = torch.device("cuda", 0)
    ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream)
    h = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k)
    xe = uniform_points(args.m_eval, H.d, seed=2503)
    fe = franke(xe)
    x = torch.from_numpy(xe).to(dev)
    f = [torch.from_numpy(v).to(dev) for v in H.f()]
    h.assemble()
    a0t, _ = h.solve(f)
    a0 = [v.cpu().numpy() for v in a0t]
    fnorm = float(np.sqrt(sum(float((v * v).sum()) for v in f)))

    def beta_of(alpha):  # beta_l = A_l alpha_l (eq:split: alpha = D_L^{-1} beta)
        return np.concatenate([h.apply_block(l, l, alpha[l])[0].cpu().numpy() for l in range(H.L)])

    b0 = beta_of(a0t)
    nM = h.m_norm(max_iter=args.norm_iters, rel_tol=1e-6)[0] if args.norms else None
    s0, _ = h.evaluate(x)
    s0 = s0.cpu().numpy()
    base = {"config": args.config, "T": 0, "err_f_inf": float(np.abs(fe - s0).max())}
    print(json.dumps(base), flush=True)
    for T in range(1, args.Tmax + 1):
        R = T + 8.0  # patches beyond ~730 points run from a global workspace
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.assemble(T=float(T), lagrange_tol=1e-14, patch_R=R, patch_min_n=20000)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        a, si = h.solve(f)
        s, _ = h.evaluate(x)
        s = s.cpu().numpy()
        rel = [float(np.linalg.norm(a[l].cpu().numpy() - a0[l]) / np.linalg.norm(a0[l])) for l in range(H.L)]
        db = float(np.linalg.norm(beta_of(a) - b0))
        extra = {"beta_err": db, "beta_rel_err": db / float(np.linalg.norm(b0)), "f_norm": fnorm}
        if args.norms:
            nD = h.m_diff_norm(max_iter=args.norm_iters, rel_tol=1e-6)[0]
            nMt = h.m_tilde_norm(max_iter=args.norm_iters, rel_tol=1e-6)[0]
            bound = fnorm * nD * sum(k * max(nM, nMt) ** (k - 1) for k in range(1, H.L))
            extra.update({"M_norm": nM, "M_minus_Mt_norm": nD, "Mt_norm": nMt, "pert1_bound": bound,
                          "bound_holds": bool(db <= bound)})
        row = {"config": args.config, "T": T, "patch_R": R, "nnz_factor": float(si.nnz_gather),
               "build_s": round(tb, 3), "solve_ms": round(si.t_total_ms, 3), "alpha_rel_err": rel,
               "s_diff_inf": float(np.abs(s - s0).max()), "err_f_inf": float(np.abs(fe - s).max()),
               "err_f_inf_exact": base["err_f_inf"], **extra}
        print(json.dumps(row), flush=True)
    h.close()
    ctx.close()


if __name__ == "__main__":
    main()
