"""One end-to-end pass of the hot path for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \
        python tools/sanitize_run.py C1|C2|C2P4 [--mf] [--thresh] [--multi]

create -> assemble -> solve (pruned and literal) -> evaluate, device buffers,
plus optional matrix-free A_l, thresholded factor (T=3, exact and local-patch
Lagrange functions) and multi-RHS.  Exits 0 and prints "sanitize ok" when
every call returned MSK_OK; the sanitizer reports its own error summary.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--mf", action="store_true")
    ap.add_argument("--thresh", action="store_true")
    ap.add_argument("--multi", action="store_true")
    ap.add_argument("--m-eval", type=int, default=20_000)
    args = ap.parse_args()
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config, halton_hierarchy
    if args.config == "C2P4":
        H = halton_hierarchy("C2P4", 2, [1024 * 4 ** l for l in range(4)], 4.0, m_eval=args.m_eval)
    else:
        H = config(args.config, m_eval=args.m_eval)
    dev = torch.device("cuda", 0)
    ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream)
    flags = msk.MSK_FLAG_MATRIX_FREE if args.mf else 0
    h = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k, flags=flags)
    h.assemble()
    f = [torch.from_numpy(v).to(dev) for v in H.f()]
    a, info = h.solve(f, tol=1e-12)
    if not args.mf:
        h.solve(f, tol=1e-12, schedule="literal")
    x = torch.from_numpy(H.eval_points).to(dev)
    s, _ = h.evaluate(x)
    s_host, _ = h.evaluate(H.eval_points)          # host-buffer (pipelined) path
    assert np.array_equal(s.cpu().numpy(), s_host)
    if args.multi and not args.mf:
        F = [torch.stack([v, 2 * v, -v], dim=1).contiguous() for v in f]
        h.solve_multi(F, tol=1e-12)
    if args.thresh and not args.mf:
        h.assemble(T=3.0, lagrange_tol=1e-13)
        h.solve(f, tol=1e-12)
        h.set_threshold(2.0)
        h.solve(f, tol=1e-12, schedule="literal")
        h.assemble(T=3.0, lagrange_tol=1e-13, patch_R=8.0, patch_min_n=500)
        h.solve(f, tol=1e-12)
    torch.cuda.synchronize()
    h.close()
    ctx.close()
    print(f"sanitize ok: {H.name} mf={args.mf} thresh={args.thresh} iters={list(info.cg_iters)[:H.L]}")


if __name__ == "__main__":
    main()
