"""world_size-2 CPU tests (torch.distributed gloo) of the host logic of the
partitioned path: the row partition (msk_partition_rows), the halo plan
(msk_halo_plan) used to exchange p between SpMVs, and the deterministic
reduction scheme (zero-filled per-chunk partials all-reduced, then summed in
chunk order), each checked against the single-process result.  The library's
host functions are called directly (no device needed); the vector data path
is emulated with numpy over gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _banded(n, w, seed=0):
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in range(max(0, i - w), min(n, i + w + 1)):
            if rng.random() < 0.6 or i == j:
                rows.append(i)
                cols.append(j)
                vals.append(rng.standard_normal())
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, np.asarray(rows) + 1, 1)
    return np.cumsum(rp), np.asarray(cols), np.asarray(vals)


def _worker(rank, world, port, n, w, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2503_04914_b200 as msk
    try:
        bounds = msk.msk_partition_rows(n, world)
        allb = [None] * world
        dist.all_gather_object(allb, bounds)
        assert all(b == bounds for b in allb)
        lo, hi = bounds[rank], bounds[rank + 1]
        rp, col, val = _banded(n, w)
        v = np.sin(np.arange(n) * 0.37)
        # referenced column range of my rows, shared with everyone
        mycols = col[rp[lo]:rp[hi]]
        hr = [int(mycols.min()), int(mycols.max()) + 1] if len(mycols) else [lo, hi]
        allh = [None] * world
        dist.all_gather_object(allh, hr)
        hlo = [h[0] for h in allh]
        hhi = [h[1] for h in allh]
        slo, shi, rlo, rhi = msk.msk_halo_plan(world, rank, bounds, hlo, hhi)
        # local copy: only my rows are valid, the rest NaN until received
        loc = np.full(n, np.nan)
        loc[lo:hi] = v[lo:hi]
        reqs = []
        for s in range(world):
            if shi[s] > slo[s]:
                reqs.append(dist.isend(torch.from_numpy(loc[slo[s]:shi[s]].copy()), dst=s))
        bufs = {}
        for s in range(world):
            if rhi[s] > rlo[s]:
                bufs[s] = torch.empty(rhi[s] - rlo[s], dtype=torch.float64)
                reqs.append(dist.irecv(bufs[s], src=s))
        for r in reqs:
            r.wait()
        for s, b in bufs.items():
            loc[rlo[s]:rhi[s]] = b.numpy()
        y = np.array([np.dot(val[rp[i]:rp[i + 1]], loc[col[rp[i]:rp[i + 1]]]) for i in range(lo, hi)])
        assert np.all(np.isfinite(y)), "a needed halo value was not received"
        # deterministic dot: per-chunk partials, zero elsewhere, all-reduce, ordered sum
        rpc = 256  # rows per chunk for this n (cg_chunk_tiles == 1)
        nch = (n + rpc - 1) // rpc
        part = torch.zeros(nch, dtype=torch.float64)
        for c in range(lo // rpc, (hi + rpc - 1) // rpc):
            a, b = c * rpc, min((c + 1) * rpc, n)
            part[c] = float(np.sum(y[a - lo:b - lo] ** 2))
        dist.all_reduce(part)
        yy = 0.0
        for c in range(nch):
            yy += float(part[c])
        full = [None] * world
        dist.all_gather_object(full, (lo, y.tolist(), yy))
        if rank == 0:
            out.put(full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,w", [(2, 5000, 40), (3, 2000, 300), (2, 1025, 900)])
def test_gloo_partition_halo_and_reduction(world, n, w):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), n, w, q), nprocs=world, join=True,
                       start_method="spawn")
    parts = q.get(timeout=60)
    rp, col, val = _banded(n, w)
    v = np.sin(np.arange(n) * 0.37)
    y_ref = np.array([np.dot(val[rp[i]:rp[i + 1]], v[col[rp[i]:rp[i + 1]]]) for i in range(n)])
    y = np.zeros(n)
    for lo, yl, _ in parts:
        y[lo:lo + len(yl)] = yl
    assert np.array_equal(y, y_ref)
    # single-process chunk-ordered reduction == distributed one, bit for bit
    yy_ref = 0.0
    for c in range((n + 255) // 256):
        yy_ref += float(np.sum(y_ref[c * 256:(c + 1) * 256] ** 2))
    assert all(p[2] == yy_ref for p in parts)


def test_partition_rows_properties():
    import paper_2503_04914_b200 as msk
    for n in (1, 255, 256, 257, 10_000, 1_250_000, 10_000_000):
        for world in (1, 2, 3, 8):
            b = msk.msk_partition_rows(n, world)
            assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
            tiles = (n + 255) // 256
            rpc = (4 if tiles >= 1024 else 2 if tiles >= 512 else 1) * 256
            assert all(x % rpc == 0 for x in b[:-1])
