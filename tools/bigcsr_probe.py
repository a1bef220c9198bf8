"""Probe: one level with > 2^31 nonzeros (2-D Halton, large delta), a few CG
iterations, to exercise the int64 paths of assembly and the CG kernel."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_04914_b200 as msk
from workloads import halton

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30_000_000
K = float(sys.argv[2]) if len(sys.argv) > 2 else 80.0
P = torch.from_numpy(halton(n, 2)).cuda()
delta = math.sqrt(K / (math.pi * n))
ctx = msk.Context(0)
h = msk.Hierarchy(ctx, [P], [delta])
h.assemble()
info = h.info()
print("nnz", info.nnz_A[0], "2^31 =", 2 ** 31, flush=True)
b = torch.ones(n, dtype=torch.float64, device="cuda")
try:
    x, it, rr, t = h.cg_level(0, b, tol=1e-14, max_iter=3)
except msk.MskError as e:
    print("cg:", e)
print("ok", flush=True)
