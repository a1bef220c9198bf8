"""Streaming bandwidth probes on one B200 (CUDA events, best of 10): pure read
(torch sum of 4.3 GB FP64), copy (read + write), and read of 4 streams at once
(sum of four 1 GB tensors), to put k_cg's mixed read stream in context."""
import json
import torch

def best(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[2:])

n = 1 << 29
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
out = {}
t = best(lambda: x.sum()); out["read_sum_GBs"] = 8 * n / t / 1e6
t = best(lambda: y.copy_(x)); out["copy_GBs"] = 16 * n / t / 1e6
xs = [torch.rand(n // 4, dtype=torch.float64, device="cuda") for _ in range(4)]
t = best(lambda: (xs[0] + xs[1]).add_(xs[2]).add_(xs[3]))
out["4stream_add_GBs (r+w approx)"] = 8 * (n // 4) * (4 + 1 + 2 + 2) / t / 1e6
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
