"""TEST INFRASTRUCTURE (run by tests/test_gpu_rank_threads.py in a subprocess).

The rank >= 0 distributed path of libmsk -- one msk_ctx per rank created
with an NCCL unique id, halo plans from all-gathered column ranges, grouped
ncclSend/ncclRecv of r halos, zero-filled all-reduces -- run with `world`
ranks as THREADS of this process on one GPU.  The NCCL entry points come from
tests/nccl_shim (MSK_NCCL_LIBRARY, set by the caller before libmsk resolves
NCCL), which checks that every rank issues the same collectives and that
every receive matches a send.  Every rank's alpha, iteration counts and s_L
must equal the single-GPU solve bit for bit, exact and
thresholded (with the T sweep).

Usage: python tests/nccl_shim/threads_dist.py WORLD [--full]
(--full: the bench configuration instead, C3 with 10^7 points on the finest
level and 10^6 evaluation points, no DIST_ALL.)
Prints one line per case and "ALL OK" at the end; exits non-zero on failure.
"""
import ctypes
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from workloads import config, halton_hierarchy, uniform_points  # noqa: E402

import paper_2503_04914_b200 as msk  # noqa: E402

DIST_ALL = msk.MSK_FLAG_DIST_ALL
CASES = [  # (name, hierarchy, T, patch_R, flags of the rank contexts' hierarchies)
    ("C1", lambda: config("C1", m_eval=0), 0.0, 0.0, DIST_ALL),
    ("halton3d", lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5), 0.0, 0.0, DIST_ALL),
    ("C3P4", lambda: config("C3P4", m_eval=0), 0.0, 0.0, DIST_ALL),
    ("halton3d-T3", lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5), 3.0, 0.0, DIST_ALL),
    ("C3P4-T2", lambda: config("C3P4", m_eval=0), 2.0, 0.0, DIST_ALL),
    ("halton3d-T3-patch", lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5), 3.0, 9.0, DIST_ALL),
    # bench.py's setting (no DIST_ALL): the latency model partitions only the 1.25M-point level
    ("C3P5-default", lambda: config("C3P5", m_eval=0), 0.0, 0.0, 0),
    # the LITERAL schedule (Algorithm 2 as printed) with partitioned levels
    ("halton3d-literal", lambda: halton_hierarchy("h3", 3, [301, 2411, 9999], 1.5), 0.0, 0.0, DIST_ALL),
    ("C3P4-literal", lambda: config("C3P4", m_eval=0), 0.0, 0.0, DIST_ALL),
    # MSK_FLAG_OUTPUT_LOCAL: each rank writes only its share of s_L (no all-gather)
    ("C3P4-local", lambda: config("C3P4", m_eval=0), 0.0, 0.0, DIST_ALL | msk.MSK_FLAG_OUTPUT_LOCAL),
]
FULL = [("C3-default", lambda: config("C3", m_eval=0), 0.0, 0.0, 0)]


def run(ctx, H, f, x, T, patch_R, flags, schedule="pruned"):
    h = msk.Hierarchy(ctx, H.points, H.delta, H.q, k=H.k, flags=flags)
    h.assemble(T=T, lagrange_tol=1e-14, patch_R=patch_R, patch_min_n=1000)
    a, info = h.solve(f, tol=1e-12, schedule=schedule)
    out = {"alpha": a, "iters": list(info.cg_iters)[:H.L]}
    if T > 0:
        h.set_threshold(1.0)
        out["alpha_T1"], _ = h.solve(f, tol=1e-12)
    else:
        s = np.full(x.shape[0], np.nan)
        h.evaluate(x, out=s)
        out["s"] = s
    h.close()
    return out


def shim_stats():
    out = (ctypes.c_long * 5)()
    ctypes.CDLL(os.environ["MSK_NCCL_LIBRARY"]).msk_shim_stats(out)
    return dict(zip(("allreduce", "allgather", "send", "recv", "comm_init"), out))


def main(world: int, full: bool = False) -> None:
    msk.load()
    for name, mk, T, patch_R, flags in (FULL if full else CASES):
        H = mk()
        f = H.f()
        x = uniform_points(10 ** 6 if full else 5000, H.d, seed=4)
        c1 = msk.Context(0)
        sched = "literal" if name.endswith("-literal") else "pruned"
        ref = run(c1, H, f, x, T, patch_R, 0, sched)  # also initialises libmsk's per-process state
        c1.close()
        nid = msk.msk_nccl_unique_id()
        res, err = [None] * world, [None] * world

        def rank_main(r):
            try:
                ctx = msk.Context(0, None, r, world, nid)
                res[r] = run(ctx, H, f, x, T, patch_R, flags, sched)
                ctx.close()
            except BaseException as e:  # reported by the main thread
                err[r] = e

        th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
        s0 = shim_stats()
        for t in th:
            t.start()
        for t in th:
            t.join()
        s1 = {k: s1 - s0[k] for k, s1 in shim_stats().items()}
        for r in range(world):
            if err[r] is not None:
                raise RuntimeError(f"{name}: rank {r} failed: {err[r]!r}")
            got = res[r]
            for l in range(H.L):
                assert np.array_equal(got["alpha"][l], ref["alpha"][l]), \
                    (name, r, l, float(np.abs(got["alpha"][l] - ref["alpha"][l]).max()))
            assert got["iters"] == ref["iters"], (name, r, got["iters"], ref["iters"])
            if T > 0:
                for l in range(H.L):
                    assert np.array_equal(got["alpha_T1"][l], ref["alpha_T1"][l]), (name, r, l, "T=1")
            elif flags & msk.MSK_FLAG_OUTPUT_LOCAL:
                w = ~np.isnan(got["s"])  # this rank's share only, each value exact
                assert w.any() and np.array_equal(got["s"][w], ref["s"][w]), (name, r, "s_L share")
            else:
                assert np.array_equal(got["s"], ref["s"]), (name, r, "s_L")
        if flags & msk.MSK_FLAG_OUTPUT_LOCAL:  # the shares partition the points
            cover = sum((~np.isnan(res[r]["s"])).astype(int) for r in range(world))
            assert np.all(cover == 1), (name, "shares")
        # the transport really carried the solve: per-rank init, halos, reductions
        assert s1["comm_init"] == world and s1["allgather"] > 0 and s1["allreduce"] > 0, s1
        assert s1["send"] > 0 and s1["send"] == s1["recv"], s1
        print(f"{name} world={world}: {world} ranks bit-identical to one GPU, iters {ref['iters']}, "
              f"shim calls {s1}", flush=True)
    print("ALL OK", flush=True)


if __name__ == "__main__":
    if not os.environ.get("MSK_NCCL_LIBRARY"):
        sys.exit("set MSK_NCCL_LIBRARY to the built tests/nccl_shim library")
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2, "--full" in sys.argv)
