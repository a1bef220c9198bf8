#!/usr/bin/env python
"""Benchmark of the hot path: one STEP = the whole multiscale pipeline on one
synthetic workload through the C-ABI (libmsk.so):

  a0/a1 msk_hierarchy_create (ingest + cell lists)  ->  a2 msk_assemble
  -> a3-a5,a8 msk_solve (Jacobi on T'_L + block CG)  ->  a9 msk_evaluate

Default workload: config C3 of BASELINE.json (d=3, 6 Halton levels, 305 ...
10^7 points, phi_{3,1}, ~1.06e8 nonzeros in the A_l, Franke-type f,
s_L evaluated at 10^7 uniform points).  Metric: Wendland nonzeros processed
per second (GNNZ/s) -- every (row, column) pair inside the support that the
step reads (assembled SpMV) or evaluates (matrix-free products, assembly,
evaluation), DESIGN.md §Measurement.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl msk|reference]

N > 1 (torchrun): one rank per GPU solves the SAME problem partitioned across
the ranks (large levels -- a latency model decides, DESIGN.md §10 -- split into spatially sorted row blocks,
p halos exchanged and CG chunk partials all-reduced over NCCL; smaller levels
solved redundantly) -- strong scaling, DESIGN.md §Multi-GPU.  value = the
problem's Wendland nonzeros per step (identical for every N: the partitioned
solve reproduces the single-GPU iterations bit for bit) / max step time.
`--impl reference` times the CPU oracle (oracle/, plain C; OpenMP over rows on
the host's cores) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# C4F: coarse levels above this many points get local-patch Lagrange functions
# (C3: levels 3-6 -> 19,531 .. 1.25M columns; levels 1-2 exact).  Round 1 used
# 20000 (level 3 exact: 609 ms of the 1.96 s build).
PATCH_MIN_N = 4000

METRIC = "multiscale solve time & Wendland nonzeros/s (GNNZ/s, % HBM roofline) at 1/2/4/8 B200"
UNIT = "GNNZ/s"
WORKLOAD = ("C3: d=3, 6 nested Halton(2,3,5) levels N=305..1e7 (round(1e7*8^(l-6))), "
            "delta_l=1.5*(sqrt(3)/2)*N^(-1/3), phi_{3,1}, f=Franke-3D, tol=1e-12, "
            "pruned Jacobi schedule, s_L at 1e7 uniform points")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_msk(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2503_04914_b200 as msk
    from workloads import config, franke

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    H = config(args.config, m_eval=args.m_eval)
    L = H.L
    # inputs resident in HBM before the timed region
    pts_d = [torch.from_numpy(p).to(dev) for p in H.points]
    f_np = H.f()
    f_d = [torch.from_numpy(x).to(dev) for x in f_np]
    xe_d = torch.from_numpy(H.eval_points).to(dev)
    alpha_d = [torch.empty(n, dtype=torch.float64, device=dev) for n in H.n]
    s_d = torch.empty(H.eval_points.shape[0], dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.current_stream(dev)
    ctx = msk.Context.distributed(local_rank, stream.cuda_stream) if world > 1 else \
        msk.Context(local_rank, stream.cuda_stream)
    sched = args.schedule
    thr = args.threshold if args.threshold is not None else (3.0 if args.config in ("C4", "C4F") else 0.0)
    patch_R = args.patch_R if args.patch_R is not None else (11.0 if args.config == "C4F" else 0.0)

    hflags = msk.MSK_FLAG_MATRIX_FREE if args.matrix_free else 0
    if world > 1:  # each rank keeps its share of s_L (no all-gather of the 80 MB result)
        hflags |= msk.MSK_FLAG_OUTPUT_LOCAL

    def step(pts, f, xe, alpha, s):
        h = msk.Hierarchy(ctx, pts, H.delta, H.q, k=H.k, flags=hflags)
        h.assemble(T=thr, lagrange_tol=1e-14, patch_R=patch_R, patch_min_n=PATCH_MIN_N)
        _, sinfo = h.solve(f, tol=args.tol, max_iter=20000, schedule=sched, alpha=alpha)
        _, einfo = h.evaluate(xe, out=s)
        hinfo = h.info()
        h.close()
        return hinfo, sinfo, einfo

    def nnz_of(hinfo, sinfo, einfo):
        # assembly evaluates every entry of A once (not in matrix-free mode)
        assembled = 0.0 if args.matrix_free else float(sum(hinfo.nnz_A[l] for l in range(L)))
        return assembled + sinfo.nnz_cg + sinfo.nnz_gather + einfo.nnz

    def launches_of(hinfo, sinfo, einfo):
        return hinfo.launches_create + hinfo.launches_assemble + sinfo.launches + einfo.launches

    for _ in range(args.warmup):
        step(pts_d, f_d, xe_d, alpha_d, s_d)
    torch.cuda.synchronize()

    # ---- timed region (device events on the stream the library launches on)
    clocks = ClockSampler(local_rank)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    recs = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        recs.append(step(pts_d, f_d, xe_d, alpha_d, s_d))
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    times = [a.elapsed_time(b) for a, b in ev]
    ms_local = float(np.mean(times))
    nnz_local = float(np.mean([nnz_of(*r) for r in recs]))
    launches = int(sum(launches_of(*r) for r in recs))

    # ---- e2e: the same step from pinned HOST buffers, copies inside the region
    pts_h = [torch.from_numpy(p).pin_memory() for p in H.points]
    f_h = [torch.from_numpy(x).pin_memory() for x in f_np]
    xe_h = torch.from_numpy(H.eval_points).pin_memory()
    alpha_h = [torch.empty(n, dtype=torch.float64).pin_memory() for n in H.n]
    s_h = torch.empty(H.eval_points.shape[0], dtype=torch.float64).pin_memory()
    step(pts_h, f_h, xe_h, alpha_h, s_h)  # warm
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(max(1, min(args.steps, 3)))]
    e2e_nnz = []
    torch.cuda.synchronize()
    for a, b in e2e_ev:
        flush.zero_()
        a.record(stream)
        e2e_rec = step(pts_h, f_h, xe_h, alpha_h, s_h)
        e2e_nnz.append(nnz_of(*e2e_rec))
        b.record(stream)
    torch.cuda.synchronize()
    e2e_ms_local = float(np.mean([a.elapsed_time(b) for a, b in e2e_ev]))
    h2d = sum(p.numel() * 8 for p in pts_h) + sum(x.numel() * 8 for x in f_h) + xe_h.numel() * 8
    d2h = sum(x.numel() * 8 for x in alpha_h) + s_h.numel() * 8
    # correctness guard for the e2e path (same numbers as the device path)
    for l in range(L):
        assert torch.equal(alpha_h[l], alpha_d[l].cpu()), "e2e and device results differ"

    # ---- max over ranks
    if world > 1:
        t = torch.tensor([ms_local, e2e_ms_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms = float(t[0]), float(t[1])
        # the problem's nonzeros per step: counted by one untimed single-GPU
        # solve of the same inputs on rank 0 (the partitioned solve performs
        # the same iterations; per-rank counters see only owned rows)
        if rank == 0:
            c1 = msk.Context(local_rank, stream.cuda_stream)
            h1 = msk.Hierarchy(c1, pts_d, H.delta, H.q, k=H.k, flags=hflags)
            h1.assemble(T=thr, lagrange_tol=1e-14, patch_R=patch_R, patch_min_n=PATCH_MIN_N)
            _, si1 = h1.solve(f_d, tol=args.tol, max_iter=20000, schedule=sched)
            _, ei1 = h1.evaluate(xe_d)
            nnz_all = e2e_nnz_all = nnz_of(h1.info(), si1, ei1)
            h1.close()
            c1.close()
        else:
            nnz_all = e2e_nnz_all = nnz_local
        dist.barrier()
    else:
        ms, e2e_ms = ms_local, e2e_ms_local
        nnz_all, e2e_nnz_all = nnz_local, float(np.mean(e2e_nnz))

    # ---- roofline of the dominant kernel: the persistent CG launch of the
    # finest level (algorithmic bytes / its CUDA-event duration)
    hinfo, sinfo, einfo = recs[-1]
    lf = L - 1
    peak, peak_kind = _peaks()
    cg_ms = float(np.mean([r[1].t_cg_level_ms[lf] for r in recs]))
    cg_bytes = float(np.mean([r[1].bytes_cg_level[lf] for r in recs]))
    if cg_ms == 0.0:  # thresholded / literal: one batched CG launch over all levels
        cg_ms = float(np.mean([r[1].t_cg_ms for r in recs]))
        cg_bytes = float(np.mean([r[1].bytes_cg for r in recs]))
    achieved = cg_bytes / (cg_ms * 1e-3) / 1e9 if cg_ms > 0 else 0.0
    # ncu DRAM bytes of this kernel, only if captured for THIS configuration
    # (profiles/traffic_<round>.json, keyed by config and mode); else null
    traffic = None
    key = f"{args.config}{'_mf' if args.matrix_free else ''}_{sched}_T{thr:g}"
    for tp in sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")), reverse=True):
        with open(tp) as fh:
            d = json.load(fh)
        if key in d.get("cg_finest_level_bytes_per_launch_by_config", {}):
            traffic = d["cg_finest_level_bytes_per_launch_by_config"][key]
            break
    share = cg_ms / ms if ms > 0 else None
    if args.matrix_free:
        # FP64-ALU bound: algorithmic flops = 17 per Wendland nonzero (r^2 5, scale 1,
        # phi 5 + 1 FMA, accumulate 2, sqrt counted as 3); candidate
        # tests not counted.  Peak: measured DFMA rate (profiles/fp64_peak.json).
        fp = os.path.join(ROOT, "profiles", "fp64_peak.json")
        fpeak = json.load(open(fp))["fp64_fma_tflops"] if os.path.exists(fp) else 37.2
        nnz_f = float(np.mean([r[1].cg_iters[lf] for r in recs])) * float(hinfo.nnz_A[lf])
        ach = 17.0 * nnz_f / (cg_ms * 1e-3) / 1e12 if cg_ms > 0 else 0.0
        roof = {"bound": "alu", "achieved": ach, "peak": fpeak, "unit": "TFLOP/s", "frac": ach / fpeak,
                "traffic": None,
                "kernel": "k_mf_spmv + CG phase kernels (matrix-free finest level, per-launch average over the solve)",
                "peak_source": "profiles/fp64_peak.json (measured DFMA)" if os.path.exists(fp) else
                "derived 148 SM x 64 FP64 lanes x 2 x 1.965 GHz",
                "algorithmic_flops_per_solve": 17.0 * nnz_f, "launch_ms": cg_ms, "share_of_step": share}
    else:
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_cg (persistent cooperative CG, finest level: fused CSR SpMV + dots + updates)",
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_launch": cg_bytes, "launch_ms": cg_ms,
                "share_of_step": share}

    out = {
        "metric": METRIC, "value": nnz_all / (ms * 1e-3) / 1e9, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD if args.config == "C3" else args.config,
                   "config": args.config, "schedule": sched, "tol": args.tol, "threshold_T": thr,
                   "matrix_free": bool(args.matrix_free), "patch_R": patch_R,
                   "n_per_level": H.n, "nnz_A": [int(hinfo.nnz_A[l]) for l in range(L)],
                   "cg_iters": [int(sinfo.cg_iters[l]) for l in range(L)],
                   "kappa_est": [round(float(sinfo.kappa_est[l]), 2) for l in range(L)],
                   "m_eval": int(H.eval_points.shape[0]),
                   "nnz_per_step": nnz_local,
                   "l2": "inputs (274 MB points, 240 MB eval points) larger than the 126 MB L2, plus a 256 MB flush write between steps",
                   "parallelism": (f"partitioned x{world}: large levels split in row blocks, CG of each in one "
                                   f"k_pcg launch per rank over NVLink peer memory (partials + r halos stored "
                                   f"into the peers, device-side barrier); smaller levels redundant; s_L "
                                   f"rank-local (MSK_FLAG_OUTPUT_LOCAL)") if world > 1
                   else "single",
                   "phase_ms": {"create": hinfo.t_create_ms, "assemble": hinfo.t_assemble_ms,
                                "solve": sinfo.t_total_ms, "solve_cg": sinfo.t_cg_ms,
                                "solve_cg_per_level": [sinfo.t_cg_level_ms[l] for l in range(L)],
                                "solve_b_products": sinfo.t_gather_ms, "evaluate": einfo.t_total_ms,
                                "evaluate_sort": einfo.t_sort_ms, "evaluate_kernel": einfo.t_eval_ms}},
        "roofline": roof,
        "e2e": {"value": e2e_nnz_all / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                # the library's own phase clocks in the last e2e step (copies included where they sit)
                "phase_ms": {"create": e2e_rec[0].t_create_ms, "assemble": e2e_rec[0].t_assemble_ms,
                             "solve": e2e_rec[1].t_total_ms, "evaluate": e2e_rec[2].t_total_ms}},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args)
    ctx.close()
    return out


# ---------------------------------------------------------------------------
# oracle (CPU) -- cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------
def _oracle_sample(name, m_eval):
    from workloads import config
    return config(name, m_eval=m_eval)


def oracle_step(H):
    """One oracle pass over the sample: sequential eq:mas solve + evaluation.
    Returns (seconds, Wendland nonzeros processed)."""
    import oracle
    f = H.f()
    t0 = time.perf_counter()
    alpha, iters, _ = oracle.sequential(H.points, H.delta, f, tol=1e-12, direct_max_n=0, count=False)
    oracle.evaluate(H.points, H.delta, alpha, H.eval_points)
    dt = time.perf_counter() - t0
    # nonzero accounting outside the timed region (same unit as our arm):
    # assembly nnz(A_l) + CG iterations x nnz(A_l) + B products + evaluation
    nnz = 0.0
    for l, (P, dl) in enumerate(zip(H.points, H.delta)):
        nA = float(oracle.pattern(P, P, dl)[0][-1])
        nnz += nA * (1 + iters[l])
        for k in range(l):
            nnz += float(oracle.pattern(P, H.points[k], H.delta[k])[0][-1])
        nnz += float(oracle.pattern(H.eval_points, P, dl)[0][-1])
    return dt, nnz


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


_SAMPLES = {
    "C3P4": "4-level prefix of C3 (N=305..156250, 178,527 points)",
    "C3P5": "5-level prefix of C3 (N=305..1.25e6, 1,428,527 points)",
}


def _oracle_leg(name, m_eval, threads):
    """The oracle (same source as the tests' library) built -O3 -march=native
    -ffp-contract=off -fopenmp for this host, `threads` OpenMP threads over rows
    (reductions serial: bit-identical results for any thread count)."""
    import oracle
    used = oracle.use_native(threads)
    try:
        dt, nnz = oracle_step(_oracle_sample(name, m_eval))
    finally:
        oracle.use_plain()
    return {"value": nnz / dt / 1e9, "unit": UNIT, "cores": used, "seconds": dt,
            "sample": f"{name}: {_SAMPLES[name]}, sequential eq:mas solve (CG, tol 1e-12) + s_L at "
                      f"{m_eval:.0e} uniform points; oracle/msk_oracle.c gcc -O3 -march=native "
                      f"-ffp-contract=off -fopenmp, {used} thread(s)"}


def cpu_baseline(args):
    """the oracle as it stands on this host, 1 thread (C3P4) and
    OpenMP over rows on every core the job may use (C3P5); the reported value
    is the multi-core leg."""
    cores = _host_cores()
    one = _oracle_leg("C3P4", 100_000, 1)
    allc = _oracle_leg("C3P5", 1_000_000, cores)
    out = dict(allc)
    out.update({"kind": "oracle", "cpu_model": _cpu_model(), "host_cores": cores,
                "legs": [one, allc]})
    return out


def run_reference(args):
    """--impl reference: the oracle on this host's cores (OpenMP build, all
    affinity cores), each step one bounded sample (C3P4) of the workload."""
    import oracle
    cores = _host_cores()
    name = "C3P4"
    H = _oracle_sample(name, 100_000)
    used = oracle.use_native(cores)
    for _ in range(args.warmup):
        oracle_step(H)
    ts, ns = [], []
    for _ in range(args.steps):
        dt, nnz = oracle_step(H)
        ts.append(dt)
        ns.append(nnz)
    oracle.use_plain()
    ms = 1e3 * float(np.mean(ts))
    val = float(np.mean(ns)) / (ms * 1e-3) / 1e9
    sample = (f"{name}: {_SAMPLES[name]}, sequential eq:mas solve (CG, tol 1e-12) + s_L at 1e5 uniform "
              f"points; oracle/msk_oracle.c gcc -O3 -march=native -ffp-contract=off -fopenmp, {used} threads")
    return {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": used, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="msk", choices=["msk", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--m-eval", type=int, default=None)
    ap.add_argument("--schedule", default="pruned", choices=["pruned", "literal"])
    ap.add_argument("--tol", type=float, default=1e-12)
    ap.add_argument("--threshold", type=float, default=None,
                    help="T of the thresholded factor (C4 default 3; 0 = exact mode)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--patch-R", type=float, default=None,
                    help="local-patch Lagrange radius (units of q_l) for levels > 4000 points (T > 0; C4F: 11)")
    ap.add_argument("--matrix-free", action="store_true",
                    help="MSK_FLAG_MATRIX_FREE: A_l never stored, CG SpMVs evaluate Phi on the fly")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_msk(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
