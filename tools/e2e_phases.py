"""Per-call times of the bench step from pinned host buffers (e2e) vs device buffers.

    python tools/e2e_phases.py [--config C3] [--reps 3]
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
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config
    H = config(args.config)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    ctx = msk.Context(0, st.cuda_stream)
    f = H.f()
    host = dict(pts=[torch.from_numpy(p).pin_memory() for p in H.points],
                f=[torch.from_numpy(x).pin_memory() for x in f],
                xe=torch.from_numpy(H.eval_points).pin_memory(),
                a=[torch.empty(n, dtype=torch.float64).pin_memory() for n in H.n],
                s=torch.empty(H.eval_points.shape[0], dtype=torch.float64).pin_memory())
    devb = dict(pts=[p.to(dev) for p in host["pts"]], f=[x.to(dev) for x in host["f"]],
                xe=host["xe"].to(dev), a=[torch.empty(n, dtype=torch.float64, device=dev) for n in H.n],
                s=torch.empty(H.eval_points.shape[0], dtype=torch.float64, device=dev))

    def step(b):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(st)
        h = msk.Hierarchy(ctx, b["pts"], H.delta, H.q, k=H.k)
        ev[1].record(st)
        h.assemble()
        ev[2].record(st)
        h.solve(b["f"], tol=1e-12, alpha=b["a"])
        ev[3].record(st)
        h.evaluate(b["xe"], out=b["s"])
        ev[4].record(st)
        h.close()
        torch.cuda.synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]

    out = {}
    for name, b in (("device", devb), ("host", host)):
        step(b)
        r = np.array([step(b) for _ in range(args.reps)]).mean(0)
        out[name] = dict(zip(["create", "assemble", "solve", "evaluate"], np.round(r, 3).tolist()))
        out[name]["total"] = round(float(r.sum()), 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
