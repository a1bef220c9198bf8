"""Isolated-kernel timings on the C3 finest level (device-resident inputs).

    python tools/microbench.py [--config C3] [--reps 5]
Prints JSON: standalone CSR SpMV (k_spmv) GB/s on algorithmic bytes, one CG
solve of the finest level, the finest B product and the evaluation kernel.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--level", type=int, default=-1, help="level of the CG / SpMV timings (default finest)")
    ap.add_argument("--eval", action="store_true",
                    help="only time s_L at 1e7 uniform points (first k_gather launch = evaluation)")
    args = ap.parse_args()
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config
    H = config(args.config, m_eval=0)
    dev = torch.device("cuda", 0)
    ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream)
    h = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k)
    h.assemble()
    info = h.info()
    if args.eval:
        from workloads import uniform_points
        f = H.f()
        h.solve(f)
        x = torch.from_numpy(uniform_points(10_000_000, H.d, seed=7)).to(dev)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # ncu --profile-from-start off captures from here
        ts = []
        for _ in range(args.reps + 1):
            _, einfo = h.evaluate(x)
            ts.append(einfo.t_eval_ms)
        print(json.dumps({"config": args.config, "m": 10_000_000, "eval_kernel_ms": ts[1:]}))
        return
    L = H.L
    lf = L - 1 if args.level < 0 else args.level
    n, nnz = H.n[lf], int(info.nnz_A[lf])
    out = {"config": args.config, "n": n, "nnz": nnz}
    v = torch.rand(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    ts = []
    for _ in range(args.reps + 1):
        _, t = h.apply_block(lf, lf, v, y)
        ts.append(t)
    t = float(np.median(ts[1:]))
    byts = 12.0 * nnz + 8.0 * (n + 1) + 8.0 * n + 8.0 * n   # val+col, row_ptr, x (once), y
    out["spmv_ms"] = t
    out["spmv_GBs"] = byts / (t * 1e-3) / 1e9
    out["spmv_GNNZs"] = nnz / (t * 1e-3) / 1e9
    # matrix-free y = A v of the same level (kernel sum over the cell list)
    hm = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k,
                       flags=msk.MSK_FLAG_MATRIX_FREE)
    hm.assemble()
    ts = []
    for _ in range(args.reps + 1):
        _, t = hm.apply_block(lf, lf, v, y)
        ts.append(t)
    t = float(np.median(ts[1:]))
    out["spmv_mf_ms"] = t
    out["spmv_mf_GNNZs"] = nnz / (t * 1e-3) / 1e9
    hm.close()
    b = torch.from_numpy(H.f()[lf]).to(dev)
    ts, its = [], []
    for _ in range(2):
        x, it, rr, t = h.cg_level(lf, b, tol=1e-12)
        ts.append(t)
        its.append(it)
    t = ts[-1]
    it = its[-1]
    cgb = it * (12.0 * nnz + 88.0 * n) + 16.0 * n   # DESIGN.md §7 (k_cg algorithmic bytes)
    out.update(cg_ms=t, cg_iters=it, cg_ms_per_iter=t / max(it, 1), cg_GBs=cgb / (t * 1e-3) / 1e9)
    if lf > 0:
        vc = torch.rand(H.n[lf - 1], dtype=torch.float64, device=dev)
        ts = []
        for _ in range(3):
            _, t = h.apply_block(lf, lf - 1, vc, y)
            ts.append(t)
        out["B_finest_from_next_coarser_ms"] = float(np.median(ts))
    print(json.dumps(out))
    h.close()
    ctx.close()


if __name__ == "__main__":
    main()
