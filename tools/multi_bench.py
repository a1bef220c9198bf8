"""Multi-RHS throughput on a config (device-resident inputs): msk_solve_multi
+ msk_evaluate_multi with R right-hand sides vs R separate single solves.

    python tools/multi_bench.py [--config C3] [--nrhs 1 2 4 8] [--m-eval 1000000]
Prints one JSON line per R: ms per call, ms per right-hand side.
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
    ap.add_argument("--nrhs", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--m-eval", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config, uniform_points
    H = config(args.config, m_eval=0)
    dev = torch.device("cuda", 0)
    ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream)
    h = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k)
    h.assemble()
    x = torch.from_numpy(uniform_points(args.m_eval, H.d, seed=3)).to(dev)
    f0 = H.f()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for R in args.nrhs:
        F = [torch.from_numpy(np.stack([f0[l] * (1.0 + 0.1 * r) + 0.01 * r for r in range(R)], 1)).to(dev)
             for l in range(H.L)]
        ts, ts1 = [], []
        for rep in range(args.reps + 1):
            torch.cuda.synchronize()
            ev0.record()
            _, it, _ = h.solve_multi(F)
            h.evaluate_multi(x)
            ev1.record()
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        # R single solves of the same columns
        for rep in range(2):
            torch.cuda.synchronize()
            ev0.record()
            for r in range(R):
                h.solve([F[l][:, r].contiguous() for l in range(H.L)])
                h.evaluate(x)
            ev1.record()
            torch.cuda.synchronize()
            ts1.append(ev0.elapsed_time(ev1))
        t, t1 = float(np.median(ts[1:])), float(ts1[-1])
        print(json.dumps({"config": args.config, "nrhs": R, "m_eval": args.m_eval, "multi_ms": t,
                          "multi_ms_per_rhs": t / R, "single_ms_per_rhs": t1 / R, "speedup": t1 / t,
                          "iters_finest": [int(v) for v in it[-1]]}))
    h.close()
    ctx.close()


if __name__ == "__main__":
    main()
