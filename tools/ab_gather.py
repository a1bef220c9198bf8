"""A/B of the matrix-free kernel sums: per-thread (default) against the
warp-cooperative staged scan (MSK_GATHER_WARP=1).  Each variant runs in its own
process (the switch is read once); outputs must be bit-identical.

    python tools/ab_gather.py [--config C3] [--mf] [--m-eval 10000000]
Prints one JSON line per variant (B-product, evaluation-kernel and CG times)
and "bitwise: True/False".
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(args, out):
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config
    H = config(args.config, m_eval=args.m_eval)
    dev = torch.device("cuda", 0)
    ctx = msk.Context(0, torch.cuda.current_stream().cuda_stream)
    flags = msk.MSK_FLAG_MATRIX_FREE if args.mf else 0
    h = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k, flags=flags)
    h.assemble()
    f = [torch.from_numpy(v).to(dev) for v in H.f()]
    x = torch.from_numpy(H.eval_points).to(dev)
    rec = {"b": [], "eval": [], "cg": [], "cg_levels": None}
    for rep in range(args.reps + 1):
        a, info = h.solve(f, tol=1e-12)
        s, einfo = h.evaluate(x)
        if rep:
            rec["b"].append(info.t_gather_ms)
            rec["eval"].append(einfo.t_eval_ms)
            rec["cg"].append(info.t_cg_ms)
            rec["cg_levels"] = list(info.t_cg_level_ms)[:H.L]
    np.savez(out, *[v.cpu().numpy() for v in a], s=s.cpu().numpy())
    res = {"variant": "warp" if os.environ.get("MSK_GATHER_WARP") else "v1", "config": args.config,
           "mf": args.mf, "b_products_ms": float(np.median(rec["b"])), "eval_kernel_ms": float(np.median(rec["eval"])),
           "cg_ms": float(np.median(rec["cg"])), "cg_level_ms": rec["cg_levels"],
           "nnz_gather": info.nnz_gather, "nnz_eval": einfo.nnz}
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--mf", action="store_true")
    ap.add_argument("--m-eval", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--child", default=None)
    args = ap.parse_args()
    if args.child:
        child(args, args.child)
        return
    tmp = tempfile.mkdtemp()
    outs = []
    for v1 in (True, False):
        env = dict(os.environ)
        env.pop("MSK_GATHER_V1", None)
        env.pop("MSK_GATHER_WARP", None)
        if not v1:
            env["MSK_GATHER_WARP"] = "1"
        out = os.path.join(tmp, f"v{int(v1)}.npz")
        cmd = [sys.executable, __file__, "--config", args.config, "--reps", str(args.reps), "--child", out]
        if args.mf:
            cmd.append("--mf")
        if args.m_eval is not None:
            cmd += ["--m-eval", str(args.m_eval)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True)
        sys.stdout.write(r.stdout)
        if r.returncode:
            sys.stdout.write(r.stderr[-3000:])
            sys.exit(r.returncode)
        outs.append(np.load(out))
    same = all(np.array_equal(outs[0][k], outs[1][k]) for k in outs[0].files)
    print(json.dumps({"config": args.config, "mf": args.mf, "bitwise": bool(same)}))


if __name__ == "__main__":
    main()
