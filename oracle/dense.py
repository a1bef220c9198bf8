"""Dense numpy oracle for SMALL hierarchies — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py may import this module.

Writes out, densely and literally, the matrices of PAPER.md §3-§4:

* B_{l2,l1} = (Phi_{l1}(x^{(l2)} - x^{(l1)}))            P:274-279 (reading C-1)
* T_L (eq:bigt P:297-319), D_L, T'_L (eq:matrix_decomposition P:320-351)
* X_{kl} = B_{kl} A_l^{-1} (eq:mathfrakXkell P:463-466)
* M = id - T'_L (eq:M P:718-738; blocks -X_{kl}, reading C-7)
* M~(T): X~_{kl}(T) keeps entries with ||x_j^{(k)} - x_i^{(l)}|| < T q_l
  (eq:perturbedmatrix P:846-861; readings C-5, C-24)
* the path-sum inverse of Theorem reformulation (eq:explicit_inverse_T
  P:501-583; reading C-27) and the Neumann series (eq:TinvNeumann P:490-493)
* the quantities plotted in Figures 1-3 (readings C-6, C-23).

Library primitives used as steps: numpy.linalg.solve / inv / norm(.,2).
"""
from __future__ import annotations

import itertools

import numpy as np


def phi(d: int, k: int, r):
    """phi_{d,k} closed form, l = floor(d/2)+k+1 (reading C-3)."""
    r = np.asarray(r, dtype=np.float64)
    l = d // 2 + k + 1
    s = np.where(r < 1.0, 1.0 - r, 0.0)
    if k == 0:
        return s ** l
    if k == 1:
        return s ** (l + 1) * ((l + 1) * r + 1.0)
    if k == 2:
        return s ** (l + 2) * ((l * l + 4 * l + 3) * r * r + (3 * l + 6) * r + 3.0) / 3.0
    raise ValueError(k)


def dist2(Xr: np.ndarray, Xc: np.ndarray) -> np.ndarray:
    """r^2 summed over coordinates left to right (elementwise, no FMA; C-4)."""
    s = np.zeros((Xr.shape[0], Xc.shape[0]))
    for a in range(Xr.shape[1]):
        t = Xr[:, None, a] - Xc[None, :, a]
        s = s + t * t
    return s


def kernel_matrix(Xr, Xc, delta, k=1):
    """(Phi_delta(x_j - y_n))_{j,n}; Phi_delta = delta^-d phi(r/delta)."""
    d = Xr.shape[1]
    r2 = dist2(Xr, Xc)
    inside = r2 < delta * delta
    v = delta ** (-d) * phi(d, k, np.sqrt(r2) / delta)
    return np.where(inside, v, 0.0)


def offsets(points):
    return np.cumsum([0] + [p.shape[0] for p in points])


def blocks(points, delta, k=1):
    """B[(kk, l)] for kk >= l (0-based), column level's delta (reading C-1)."""
    L = len(points)
    return {(a, b): kernel_matrix(points[a], points[b], delta[b], k)
            for a in range(L) for b in range(a + 1)}


def T_matrix(points, delta, k=1):
    """Dense T_L of eq:bigt."""
    o = offsets(points)
    B = blocks(points, delta, k)
    T = np.zeros((o[-1], o[-1]))
    for (a, b), blk in B.items():
        T[o[a]:o[a + 1], o[b]:o[b + 1]] = blk
    return T


def D_matrix(points, delta, k=1):
    o = offsets(points)
    D = np.zeros((o[-1], o[-1]))
    for l, p in enumerate(points):
        D[o[l]:o[l + 1], o[l]:o[l + 1]] = kernel_matrix(p, p, delta[l], k)
    return D


def Xi_blocks(points, delta, k=1):
    """X_{kl} = B_{kl} A_l^{-1} for kk > l (eq:mathfrakXkell)."""
    L = len(points)
    Ainv = [np.linalg.inv(kernel_matrix(points[l], points[l], delta[l], k)) for l in range(L)]
    return {(a, b): kernel_matrix(points[a], points[b], delta[b], k) @ Ainv[b]
            for a in range(L) for b in range(a)}


def Tprime_matrix(points, delta, k=1, Xi=None):
    """T'_L of eq:T_n_prime: identity diagonal, X_{kl} below."""
    o = offsets(points)
    Xi = Xi if Xi is not None else Xi_blocks(points, delta, k)
    Tp = np.eye(o[-1])
    for (a, b), blk in Xi.items():
        Tp[o[a]:o[a + 1], o[b]:o[b + 1]] = blk
    return Tp


def M_matrix(points, delta, k=1, Xi=None):
    """M = id - T'_L (blocks -X_{kl}; reading C-7)."""
    return np.eye(offsets(points)[-1]) - Tprime_matrix(points, delta, k, Xi)


def truncation_mask(points, q, T):
    """Geometric mask of X~_{kl}(T): ||x_j^{(k)} - x_i^{(l)}||^2 < (T q_l)^2
    (strict; coarse column level's q, reading C-5)."""
    L = len(points)
    return {(a, b): dist2(points[a], points[b]) < (T * q[b]) * (T * q[b])
            for a in range(L) for b in range(a)}


def Mtilde_matrix(points, delta, q, T, k=1, Xi=None):
    """M~(T) (eq:perturbedmatrix), blocks -X~_{kl}(T)."""
    o = offsets(points)
    Xi = Xi if Xi is not None else Xi_blocks(points, delta, k)
    mask = truncation_mask(points, q, T)
    Mt = np.zeros((o[-1], o[-1]))
    for (a, b), blk in Xi.items():
        Mt[o[a]:o[a + 1], o[b]:o[b + 1]] = -np.where(mask[(a, b)], blk, 0.0)
    return Mt


def split(v, points):
    o = offsets(points)
    return [v[o[l]:o[l + 1]].copy() for l in range(len(points))]


def solve_dense(points, delta, f, k=1):
    """O8: alpha = T_L^{-1} f by dense LU (eq:bigt)."""
    T = T_matrix(points, delta, k)
    return split(np.linalg.solve(T, np.concatenate(f)), points)


def path_sum_inverse(points, delta, k=1, Xi=None):
    """(T'_L)^{-1} from Theorem reformulation (eq:explicit_inverse_T):
    block (kk, j) = sum over strictly decreasing paths p = (kk=p_1 > ... > p_m = j)
    of (-1)^{|p|-1} X_{p1 p2} X_{p2 p3} ... X_{p_{m-1} p_m}   (reading C-27)."""
    L = len(points)
    o = offsets(points)
    Xi = Xi if Xi is not None else Xi_blocks(points, delta, k)
    inv = np.eye(o[-1])
    for a in range(L):
        for b in range(a):
            acc = np.zeros((points[a].shape[0], points[b].shape[0]))
            inner = list(range(b + 1, a))
            for r in range(len(inner) + 1):
                for mid in itertools.combinations(sorted(inner, reverse=True), r):
                    path = (a,) + tuple(sorted(mid, reverse=True)) + (b,)
                    prod = Xi[(path[0], path[1])]
                    for t in range(1, len(path) - 1):
                        prod = prod @ Xi[(path[t], path[t + 1])]
                    acc += (-1.0) ** (len(path) - 1) * prod
            inv[o[a]:o[a + 1], o[b]:o[b + 1]] = acc
    return inv


def neumann_inverse(M, L):
    """(T'_L)^{-1} = sum_{t=0}^{L-1} (id - T'_L)^t (eq:TinvNeumann)."""
    acc = np.eye(M.shape[0])
    P = np.eye(M.shape[0])
    for _ in range(1, L):
        P = P @ M
        acc = acc + P
    return acc


def jacobi(Mop, f, L, beta0=None):
    """beta_{m+1} = f + M beta_m, L sweeps (eq:jacobi, Theorem jacobi)."""
    fv = np.concatenate(f)
    beta = fv.copy() if beta0 is None else np.concatenate(beta0)
    for _ in range(L):
        beta = fv + Mop @ beta
    return beta


def thresholded_solve(points, delta, q, f, T, k=1, Xi=None):
    """O7: (id - M~(T)) beta~ = f by L Jacobi sweeps, then D_L alpha~ = beta~
    (eq:perturbed_split P:865-869).  Returns (alpha~ list, beta~ list)."""
    Mt = Mtilde_matrix(points, delta, q, T, k, Xi)
    beta = jacobi(Mt, f, len(points))
    bl = split(beta, points)
    alpha = [np.linalg.solve(kernel_matrix(p, p, delta[l], k), bl[l])
             for l, p in enumerate(points)]
    return alpha, bl


# ---------------------------------------------------------------------------
# Figures 1-3
# ---------------------------------------------------------------------------
def fig1_norm(points, delta, k=1):
    """||M_L||_2 (Figure 1 'numerical value')."""
    return float(np.linalg.norm(M_matrix(points, delta, k), 2))


def fig1_bound(L):
    """Figure 1 'theoretical bound' curve = sqrt(L) 2^(L-1) (reading C-23):
    eq:Mbound with C C_Sigma sqrt(2) c_q^{-d} = 1 ... evaluated as printed."""
    return float(np.sqrt(L) * 2.0 ** (L - 1))


def fig2_ratio(points, delta, q, T, k=1, Xi=None):
    """||M - M~(T)||_2 / ||M||_2 (Figure 2; reading C-24)."""
    Xi = Xi if Xi is not None else Xi_blocks(points, delta, k)
    M = M_matrix(points, delta, k, Xi)
    Mt = Mtilde_matrix(points, delta, q, T, k, Xi)
    return float(np.linalg.norm(M - Mt, 2) / np.linalg.norm(M, 2))


def fig3_ratio(points, delta, q, T, k=1, Xi=None, eps=1e-8):
    """nnz(M~(T)) / nnz(M), counting |v| > 1e-8 (Figure 3; reading C-6)."""
    Xi = Xi if Xi is not None else Xi_blocks(points, delta, k)
    mask = truncation_mask(points, q, T)
    num = sum(int(np.count_nonzero((np.abs(b) > eps) & mask[key])) for key, b in Xi.items())
    den = sum(int(np.count_nonzero(np.abs(b) > eps)) for b in Xi.values())
    return num / den
