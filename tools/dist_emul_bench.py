"""Per-level CG time of the partitioned solve in the single-GPU emulation:
k_pcg (one launch over "peer" stores, device-side cross-partition barriers)
against the host-driven phase kernels (MSK_DIST_P2P=0), world 1..8, on C3.
On one GPU the partitions share the SMs, so the difference to world 1 is the
cost of the partitioned machinery itself (barriers, pushes, launches).

    python tools/dist_emul_bench.py [--config C3] [--worlds 1,2,4,8]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(args):
    import numpy as np
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config
    H = config(args.config, m_eval=0)
    dev = torch.device("cuda", 0)
    pts = [torch.from_numpy(p).to(dev) for p in H.points]
    f = [torch.from_numpy(v).to(dev) for v in H.f()]
    ref = None
    for w in [int(x) for x in args.worlds.split(",")]:
        ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream) if w == 1 else \
            msk.Context(0, torch.cuda.current_stream().cuda_stream, rank=-1, world=w)
        h = msk.Hierarchy(ctx, pts, H.delta, H.q, k=H.k)
        h.assemble()
        ts = []
        for rep in range(args.reps + 1):
            a, info = h.solve(f, tol=1e-12)
            if rep:
                ts.append([info.t_cg_level_ms[l] for l in range(H.L)])
        a = [v.cpu().numpy() for v in a]
        if ref is None:
            ref = a
        same = all(np.array_equal(x, y) for x, y in zip(a, ref))
        med = np.median(np.array(ts), axis=0).tolist()
        print(json.dumps({"path": os.environ.get("MSK_DIST_P2P", "1"), "world": w, "cg_level_ms": med,
                          "iters": list(info.cg_iters)[:H.L], "bitwise_vs_world1": same}), flush=True)
        h.close()
        ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        child(args)
        return
    for p2p in ("1", "0"):
        env = dict(os.environ, MSK_DIST_P2P=p2p)
        r = subprocess.run([sys.executable, __file__, "--child", "--config", args.config, "--worlds", args.worlds,
                            "--reps", str(args.reps)], env=env, capture_output=True, text=True)
        sys.stdout.write(r.stdout)
        if r.returncode:
            sys.stdout.write(r.stderr[-3000:])


if __name__ == "__main__":
    main()
