"""paper_2503_04914_b200 -- B200-native (sm_100a, FP64) hot path of Lot & Rieger's
monolithic kernel-based multiscale method (arXiv 2503.04914).

The compute lives in ``libmsk.so`` (CUDA kernels behind the C-ABI declared in
``include/msk.h``).  This package is the thin Python binding: the functions
``msk_*`` mirror the C entry points one to one, and ``Context`` /
``Hierarchy`` wrap the handles.  Buffers may be numpy arrays (host memory) or
torch tensors (host or CUDA): the library detects which and copies host data
through its stream.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from ._lib import (EXPORTED, MSK_FLAG_DIST_ALL, MSK_FLAG_MATRIX_FREE, MSK_FLAG_OUTPUT_LOCAL, MSK_SCHED_LITERAL, MSK_SCHED_PRUNED, EvalInfo, HierarchyInfo,
                   MskError, SolveInfo, check, load)

__all__ = ["Context", "Hierarchy", "MskError", "SolveInfo", "HierarchyInfo", "EvalInfo",
           "MSK_SCHED_PRUNED", "MSK_SCHED_LITERAL", "load"] + EXPORTED

_vp = ctypes.c_void_p


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a):
    """Raw data pointer of a contiguous numpy array / torch tensor (FP64 or ints)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if _is_torch(a):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)}")


def _f64(a):
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.float64)
    if _is_torch(a):
        import torch
        if a.dtype != torch.float64:
            raise TypeError("tensors must be float64")
        return a.contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _empty_like_kind(ref, n):
    if _is_torch(ref):
        import torch
        return torch.empty(n, dtype=torch.float64, device=ref.device)
    return np.empty(n, dtype=np.float64)


def _ptr_array(bufs):
    arr = (_vp * len(bufs))(*[_ptr(b) for b in bufs])
    return ctypes.cast(arr, ctypes.POINTER(_vp)), arr


# ----------------------------------------------------------------- C-ABI mirror
def msk_ctx_create(device=0, cuda_stream=None, rank=0, world_size=1, nccl_unique_id=None):
    out = _vp()
    check(load().msk_ctx_create(device, cuda_stream, rank, world_size, nccl_unique_id,
                                ctypes.byref(out)))
    return out


def msk_ctx_destroy(ctx):
    load().msk_ctx_destroy(ctx)


def msk_hierarchy_create(ctx, d, L, n, points, delta, q, wendland_k, flags=0):
    nn = (ctypes.c_int64 * L)(*n)
    pp, keep = _ptr_array(points)
    dl = (ctypes.c_double * L)(*delta)
    qq = (ctypes.c_double * L)(*q) if q is not None else None
    out = _vp()
    check(load().msk_hierarchy_create(ctx, d, L, nn, pp, dl, qq, wendland_k, flags, ctypes.byref(out)))
    return out


def msk_hierarchy_destroy(h):
    load().msk_hierarchy_destroy(h)


def msk_hierarchy_info_get(h):
    info = HierarchyInfo()
    check(load().msk_hierarchy_info_get(h, ctypes.byref(info)))
    return info


def msk_assemble(h, T=0.0, lagrange_tol=1e-13):
    check(load().msk_assemble(h, float(T), float(lagrange_tol)))


def msk_set_threshold(h, T):
    check(load().msk_set_threshold(h, float(T)))


def msk_assemble_ex(h, T, lagrange_tol, patch_R, patch_min_n):
    check(load().msk_assemble_ex(h, float(T), float(lagrange_tol), float(patch_R), int(patch_min_n)))


def msk_solve(h, f, tol, max_iter, schedule, alpha):
    fp, k1 = _ptr_array(f)
    ap, k2 = _ptr_array(alpha)
    info = SolveInfo()
    check(load().msk_solve(h, fp, float(tol), int(max_iter), int(schedule), ap, ctypes.byref(info)))
    return info


def msk_solve_multi(h, nrhs, f, tol, max_iter, alpha, iters=None):
    """iters: optional int32 array [L * nrhs]; returns the device time (ms)."""
    fp, k1 = _ptr_array(f)
    ap, k2 = _ptr_array(alpha)
    t = ctypes.c_double(0.0)
    check(load().msk_solve_multi(h, int(nrhs), fp, float(tol), int(max_iter), ap, _ptr(iters), ctypes.byref(t)))
    return t.value


def msk_evaluate_multi(h, m, x, s):
    check(load().msk_evaluate_multi(h, int(m), _ptr(x), _ptr(s)))


def msk_m_norm(h, max_iter=500, rel_tol=1e-9, cg_tol=1e-13):
    """||M_L||_2 by power iteration (returns (norm, iterations))."""
    nrm = ctypes.c_double(0.0)
    it = ctypes.c_int32(0)
    check(load().msk_m_norm(h, int(max_iter), float(rel_tol), float(cg_tol), ctypes.byref(nrm), ctypes.byref(it)))
    return nrm.value, it.value


def msk_m_norm_ex(h, which, max_iter=500, rel_tol=1e-9, cg_tol=1e-13):
    nrm = ctypes.c_double(0.0)
    it = ctypes.c_int32(0)
    check(load().msk_m_norm_ex(h, int(which), int(max_iter), float(rel_tol), float(cg_tol), ctypes.byref(nrm),
                               ctypes.byref(it)))
    return nrm.value, it.value


def msk_evaluate(h, m, x, s):
    check(load().msk_evaluate(h, int(m), _ptr(x), _ptr(s)))


def msk_evaluate_ex(h, m, x, s):
    info = EvalInfo()
    check(load().msk_evaluate_ex(h, int(m), _ptr(x), _ptr(s), ctypes.byref(info)))
    return info


def msk_export_block(h, row_level, col_level, row_ptr, col, val):
    check(load().msk_export_block(h, row_level, col_level, _ptr(row_ptr), _ptr(col), _ptr(val)))


def msk_export_factor(h, row_level, col_level, row_ptr, col, val):
    T = ctypes.c_double(0.0)
    check(load().msk_export_factor(h, row_level, col_level, _ptr(row_ptr), _ptr(col), _ptr(val),
                                   ctypes.byref(T)))
    return T.value


def msk_export_cells(h, level, perm, cell_start, cell_key, lo, cell, dims):
    check(load().msk_export_cells(h, level, _ptr(perm), _ptr(cell_start), _ptr(cell_key), _ptr(lo),
                                  _ptr(cell), _ptr(dims)))


def msk_export_grid(h, level, lo, inv_cell, dims):
    check(load().msk_export_grid(h, level, _ptr(lo), _ptr(inv_cell), _ptr(dims)))


def msk_apply_block(h, row_level, col_level, v, y):
    t = ctypes.c_double(0.0)
    check(load().msk_apply_block(h, row_level, col_level, _ptr(v), _ptr(y), ctypes.byref(t)))
    return t.value


def msk_cg_level(h, level, b, x, tol, max_iter):
    it = ctypes.c_int32(0)
    rr = ctypes.c_double(0.0)
    t = ctypes.c_double(0.0)
    check(load().msk_cg_level(h, level, _ptr(b), _ptr(x), float(tol), int(max_iter), ctypes.byref(it),
                              ctypes.byref(rr), ctypes.byref(t)))
    return it.value, rr.value, t.value


def msk_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(load().msk_nccl_unique_id(ctypes.cast(buf, _vp)))
    return buf.raw


def msk_partition_rows(n, world):
    b = (ctypes.c_int64 * (world + 1))()
    check(load().msk_partition_rows(int(n), int(world), b))
    return list(b)


def msk_halo_plan(world, rank, rows, hlo, hhi):
    arr = lambda v: (ctypes.c_int64 * len(v))(*[int(x) for x in v])
    out = [(ctypes.c_int64 * world)() for _ in range(4)]
    check(load().msk_halo_plan(int(world), int(rank), arr(rows), arr(hlo), arr(hhi), *out))
    return [list(o) for o in out]  # send_lo, send_hi, recv_lo, recv_hi


def msk_last_error():
    return load().msk_last_error().decode()


def msk_version():
    return load().msk_version().decode()


# ----------------------------------------------------------------- handles
class Context:
    """A libmsk context on one CUDA device.

    world == 1: single GPU.  world > 1 with rank >= 0: one partition per rank
    over NCCL; `nccl_id` is the 128-byte id from msk_nccl_unique_id() on rank
    0 (``Context.distributed`` broadcasts it with torch.distributed).
    world > 1 with rank == -1: single-process emulation of `world` partitions
    on this device (tests).
    """

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1, nccl_id=None):
        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        self.rank, self.world = rank, world
        self.handle = msk_ctx_create(device, stream, rank, world,
                                     ctypes.cast(idbuf, _vp) if idbuf is not None else None)
        self._children = weakref.WeakSet()

    @classmethod
    def distributed(cls, device: int, stream=None):
        """One rank of a torch.distributed job: rank 0 creates the NCCL id and
        broadcasts it through the process group (plumbing only)."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        if world == 1:
            return cls(device, stream)
        obj = [msk_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(device, stream, rank, world, obj[0])

    def close(self):
        if self.handle:
            for h in list(self._children):   # hierarchies die before their context
                h.close()
            msk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Hierarchy:
    """Point hierarchy X_1..X_L on the device with its cell lists (a0, a1).

    points: list of (N(l), d) FP64 arrays/tensors (row-major), coarse to fine.
    delta:  support radii; q: separation values or None; k: Wendland phi_{d,k}.
    """

    def __init__(self, ctx: Context, points, delta, q=None, k: int = 1, flags: int = 0):
        pts = [_f64(p) for p in points]
        self.ctx = ctx
        self.d = int(pts[0].shape[1])
        self.L = len(pts)
        self.n = [int(p.shape[0]) for p in pts]
        self.handle = msk_hierarchy_create(ctx.handle, self.d, self.L, self.n, pts, list(delta),
                                           None if q is None else list(q), int(k), int(flags))
        self.last_solve = None
        ctx._children.add(self)

    def close(self):
        if self.handle and self.ctx.handle:
            msk_hierarchy_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> HierarchyInfo:
        return msk_hierarchy_info_get(self.handle)

    def assemble(self, T: float = 0.0, lagrange_tol: float = 1e-13, patch_R: float = 0.0, patch_min_n: int = 0):
        """patch_R > 0: local-patch Lagrange functions of radius patch_R * q_l on the
        coarse levels with more than patch_min_n points (msk_assemble_ex)."""
        if patch_R > 0.0:
            msk_assemble_ex(self.handle, T, lagrange_tol, patch_R, patch_min_n)
        else:
            msk_assemble(self.handle, T, lagrange_tol)

    def solve(self, f, tol=1e-12, max_iter=20000, schedule="pruned", alpha=None):
        f = [_f64(x) for x in f]
        if alpha is None:
            alpha = [_empty_like_kind(f[l], self.n[l]) for l in range(self.L)]
        sch = MSK_SCHED_LITERAL if schedule == "literal" else MSK_SCHED_PRUNED
        info = msk_solve(self.handle, f, tol, max_iter, sch, alpha)
        self.last_solve = info
        return alpha, info

    def set_threshold(self, T: float):
        """Use the entries of the stored factor within T q_l (T integer <= the
        build's T, or the build's T): the T sweep of one build."""
        msk_set_threshold(self.handle, T)

    def solve_multi(self, F, tol=1e-12, max_iter=20000):
        """F: per level an (n_l, nrhs) array (numpy or CUDA tensor).  Returns
        (alpha list of (n_l, nrhs), iterations (L, nrhs), device ms)."""
        F = [_f64(x) for x in F]
        nrhs = int(F[0].shape[1]) if len(F[0].shape) == 2 else 1
        alpha = []
        for l in range(self.L):
            if _is_torch(F[l]):
                import torch
                alpha.append(torch.empty((self.n[l], nrhs), dtype=torch.float64, device=F[l].device))
            else:
                alpha.append(np.empty((self.n[l], nrhs), dtype=np.float64))
        iters = np.zeros(self.L * nrhs, dtype=np.int32)
        t = msk_solve_multi(self.handle, nrhs, F, tol, max_iter, alpha, iters)
        self.nrhs = nrhs
        return alpha, iters.reshape(self.L, nrhs), t

    def m_norm(self, max_iter=500, rel_tol=1e-9, cg_tol=1e-13):
        """||M_L||_2 (Figure 1) by power iteration on the GPU: (norm, iterations)."""
        return msk_m_norm(self.handle, max_iter, rel_tol, cg_tol)

    def m_diff_norm(self, max_iter=500, rel_tol=1e-9, cg_tol=1e-13):
        """||M_L - M~_L(T)||_2 (Figure 2) with the stored factor: (norm, iterations)."""
        return msk_m_norm_ex(self.handle, 1, max_iter, rel_tol, cg_tol)

    def m_tilde_norm(self, max_iter=500, rel_tol=1e-9, cg_tol=1e-13):
        """||M~_L(T)||_2 of the stored factor alone: (norm, iterations)."""
        return msk_m_norm_ex(self.handle, 2, max_iter, rel_tol, cg_tol)

    def evaluate_multi(self, x):
        x = _f64(x)
        m = int(x.shape[0])
        nrhs = getattr(self, "nrhs", 1)  # before solve_multi the library reports MSK_ERR_STATE
        if _is_torch(x):
            import torch
            s = torch.empty((m, nrhs), dtype=torch.float64, device=x.device)
        else:
            s = np.empty((m, nrhs), dtype=np.float64)
        msk_evaluate_multi(self.handle, m, x, s)
        return s

    def evaluate(self, x, out=None):
        x = _f64(x)
        m = int(x.shape[0])
        s = out if out is not None else _empty_like_kind(x, m)
        info = msk_evaluate_ex(self.handle, m, x, s)
        return s, info

    def export_block(self, row_level: int, col_level: int):
        n = self.n[row_level]
        rp = np.zeros(n + 1, dtype=np.int64)
        msk_export_block(self.handle, row_level, col_level, rp, None, None)
        nnz = int(rp[-1])
        col = np.zeros(max(nnz, 1), dtype=np.int32)
        val = np.zeros(max(nnz, 1), dtype=np.float64)
        msk_export_block(self.handle, row_level, col_level, rp, col, val)
        return rp, col[:nnz], val[:nnz]

    def export_factor(self, row_level: int, col_level: int):
        """Entries of X~_{row_level,col_level}(T) (caller indices, CSR)."""
        n = self.n[row_level]
        rp = np.zeros(n + 1, dtype=np.int64)
        msk_export_factor(self.handle, row_level, col_level, rp, None, None)
        nnz = int(rp[-1])
        col = np.zeros(max(nnz, 1), dtype=np.int32)
        val = np.zeros(max(nnz, 1), dtype=np.float64)
        T = msk_export_factor(self.handle, row_level, col_level, rp, col, val)
        return rp, col[:nnz], val[:nnz], T

    def export_cells(self, level: int):
        info = self.info()
        n, nc = self.n[level], int(info.ncells[level])
        perm = np.zeros(n, dtype=np.int32)
        cs = np.zeros(nc + 1, dtype=np.int32)
        keys = np.zeros(n, dtype=np.int64)
        lo = np.zeros(3)
        cell = np.zeros(1)
        dims = np.zeros(3, dtype=np.int64)
        msk_export_cells(self.handle, level, perm, cs, keys, lo, cell, dims)
        inv = np.zeros(3)
        msk_export_grid(self.handle, level, None, inv, None)
        return dict(perm=perm, cell_start=cs, keys=keys, lo=lo[:self.d], cell=float(cell[0]),
                    inv_cell=inv[:self.d].copy(), dims=dims[:self.d])

    def apply_block(self, row_level: int, col_level: int, v, y=None):
        v = _f64(v)
        y = y if y is not None else _empty_like_kind(v, self.n[row_level])
        t = msk_apply_block(self.handle, row_level, col_level, v, y)
        return y, t

    def cg_level(self, level: int, b, tol=1e-12, max_iter=20000, x=None):
        b = _f64(b)
        x = x if x is not None else _empty_like_kind(b, self.n[level])
        it, rr, t = msk_cg_level(self.handle, level, b, x, tol, max_iter)
        return x, it, rr, t
