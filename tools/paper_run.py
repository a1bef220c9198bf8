"""One full multiscale solve of a paper grid hierarchy (Table 1 / Figure 4,
PAPER.md:1594-1684) on one B200: grids l = 1..L, nu = 4, phi_(3,1), Franke.

    python tools/paper_run.py --levels 14 [--schedule pruned|literal]

Prints one JSON line with per-phase device times (CUDA events inside the
library), CG iterations and nonzero counts.  The paper reports 92.6 s for
L = 11 and ~2.5 h for L = 14 (A100, 3456 warps, CPU clock incl. data
management) -- context, not a like-for-like comparison.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, default=11)
    ap.add_argument("--schedule", default="pruned")
    ap.add_argument("--tol", type=float, default=1e-12)
    ap.add_argument("--m-eval", type=int, default=100_000)
    ap.add_argument("--matrix-free", action="store_true",
                    help="MSK_FLAG_MATRIX_FREE (the paper's mode: no stored matrices, P:1559)")
    args = ap.parse_args()
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config
    t0 = time.time()
    H = config(f"P{args.levels}", m_eval=args.m_eval)
    dev = torch.device("cuda", 0)
    pts = [torch.from_numpy(p).to(dev) for p in H.points]
    f = [torch.from_numpy(x).to(dev) for x in H.f()]
    xe = torch.from_numpy(H.eval_points).to(dev)
    t_gen = time.time() - t0
    ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    t1 = time.time()
    h = msk.Hierarchy(ctx, pts, H.delta, H.q, k=1,
                      flags=msk.MSK_FLAG_MATRIX_FREE if args.matrix_free else 0)
    h.assemble()
    alpha, si = h.solve(f, tol=args.tol, schedule=args.schedule)
    s, ei = h.evaluate(xe)
    torch.cuda.synchronize()
    wall = time.time() - t1
    hi = h.info()
    # interpolation check on a sample of the finest level (f_L = f on X_L)
    idx = torch.arange(0, H.n[-1], max(1, H.n[-1] // 1000), device=dev)
    sL, _ = h.evaluate(pts[-1][idx].contiguous())
    err = float((sL - f[-1][idx]).abs().max() / f[-1].abs().max())
    L = H.L
    out = {"levels": L, "points": int(sum(H.n)), "schedule": args.schedule, "tol": args.tol,
           "matrix_free": bool(args.matrix_free),
           "wall_s": wall, "gen_s": t_gen,
           "t_create_ms": hi.t_create_ms, "t_assemble_ms": hi.t_assemble_ms,
           "t_solve_ms": si.t_total_ms, "t_cg_ms": si.t_cg_ms, "t_b_ms": si.t_gather_ms,
           "t_eval_ms": ei.t_total_ms, "cg_iters": [int(si.cg_iters[l]) for l in range(L)],
           "nnz_A": int(sum(hi.nnz_A[l] for l in range(L))), "nnz_cg": si.nnz_cg,
           "nnz_b": si.nnz_gather, "interp_rel_err_sampled": err,
           "mem_gb": torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
