"""Host-buffer (pipelined) vs device-buffer evaluation on C3: per-phase times.

    MSK_EVAL_CHUNK=... python tools/eval_pipe.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2503_04914_b200 as msk
    from workloads import config
    H = config("C3")
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    ctx = msk.Context(0, st.cuda_stream)
    h = msk.Hierarchy(ctx, [torch.from_numpy(p).to(dev) for p in H.points], H.delta, H.q, k=H.k)
    h.assemble()
    h.solve([torch.from_numpy(x).to(dev) for x in H.f()], tol=1e-12)
    xh = torch.from_numpy(H.eval_points).pin_memory()
    sh = torch.empty(xh.shape[0], dtype=torch.float64).pin_memory()
    xd = xh.to(dev)
    sd = torch.empty(xh.shape[0], dtype=torch.float64, device=dev)
    res = {}
    for name, (x, s) in (("device", (xd, sd)), ("host", (xh, sh))):
        rows = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _, info = h.evaluate(x, out=s)
            e1.record(st)
            torch.cuda.synchronize()
            rows.append([e0.elapsed_time(e1), info.t_sort_ms, info.t_eval_ms, info.t_total_ms])
        res[name] = np.round(np.mean(rows[1:], 0), 3).tolist()
    res["chunk"] = os.environ.get("MSK_EVAL_CHUNK", "default")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
