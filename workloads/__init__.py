"""Seeded / deterministic synthetic inputs shared by the oracle tests, the GPU
tests and bench.py.

This module holds NO arithmetic of the multiscale method (no kernel, no
solver, no pattern logic).  It only produces

* point hierarchies X_1 ... X_L  (Assumption "pointset";
  Table 1 grids PAPER.md:1260-1272; Halton families),
* the support radii delta_l and separation values q_l handed to the API
  (the recipe is DESIGN.md "Input recipe"; PAPER.md:105-107 eq:deltadef),
* the target function samples f^{(l)} = f|_{X_l}  (the Franke
  function eq:Franke PAPER.md:1277-1279 and its 3-D extension, reading C-16),
* evaluation points (numpy PCG64, seed 2503).

Every generator is deterministic; nothing here depends on the CUDA path or on
the oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

EVAL_SEED = 2503
PRIMES = (2, 3, 5)


# ----------------------------------------------------------------------------
# point families
# ----------------------------------------------------------------------------
def halton(n: int, d: int, start: int = 1) -> np.ndarray:
    """Unscrambled Halton points, indices start..start+n-1 (origin skipped).

    Radical inverse in bases (2, 3, 5)[:d]; the digit loop accumulates in a
    fixed order so the result is bit-reproducible.  Row-major (n, d) float64.
    Nested by construction: halton(m, d)[:n] == halton(n, d) for n <= m.
    """
    out = np.empty((n, d), dtype=np.float64)
    idx0 = np.arange(start, start + n, dtype=np.int64)
    for a in range(d):
        b = PRIMES[a]
        i = idx0.copy()
        r = np.zeros(n, dtype=np.float64)
        f = 1.0 / b
        while np.any(i > 0):
            r += f * (i % b)
            i //= b
            f /= b
        out[:, a] = r
    return out


def grid_level(level: int, d: int = 2) -> np.ndarray:
    """Regular grid on [0,1]^d with spacing 2^-level (Table 1).

    N(level) = (2^level + 1)^d; ravelled with meshgrid(indexing='ij')
    (x-major), so x = i * 2^-level exactly.
    """
    m = 2 ** level + 1
    ax = np.arange(m, dtype=np.float64) * (2.0 ** -level)
    mesh = np.meshgrid(*([ax] * d), indexing="ij")
    return np.stack([g.ravel() for g in mesh], axis=1)


def uniform_points(m: int, d: int, seed: int = EVAL_SEED) -> np.ndarray:
    """m i.i.d. uniform points in [0,1]^d (numpy PCG64, fixed seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.random((m, d), dtype=np.float64)


# ----------------------------------------------------------------------------
# target functions (inputs, not method arithmetic)
# ----------------------------------------------------------------------------
def franke2(p: np.ndarray) -> np.ndarray:
    """Franke function, PAPER.md:1277-1279 (eq:Franke), verbatim (reading C-16)."""
    x, y = p[:, 0], p[:, 1]
    return (0.75 * np.exp(-((9 * x - 2) ** 2 + (9 * y - 2) ** 2) / 4.0)
            + 0.75 * np.exp(-((9 * x + 1) ** 2) / 49.0 - (9 * y + 1) / 10.0)
            + 0.5 * np.exp(-((9 * x - 7) ** 2 + (9 * y - 3) ** 2) / 4.0)
            - 0.2 * np.exp(-(9 * x - 4) ** 2 - (9 * y - 7) ** 2))


def franke3(p: np.ndarray) -> np.ndarray:
    """3-D extension of eq:Franke (the paper is silent on d=3; reading C-16)."""
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    return (0.75 * np.exp(-((9 * x - 2) ** 2 + (9 * y - 2) ** 2 + (9 * z - 2) ** 2) / 4.0)
            + 0.75 * np.exp(-((9 * x + 1) ** 2) / 49.0 - (9 * y + 1) / 10.0 - (9 * z + 1) / 10.0)
            + 0.5 * np.exp(-((9 * x - 7) ** 2 + (9 * y - 3) ** 2 + (9 * z - 5) ** 2) / 4.0)
            - 0.2 * np.exp(-(9 * x - 4) ** 2 - (9 * y - 7) ** 2 - (9 * z - 5) ** 2))


def franke(p: np.ndarray) -> np.ndarray:
    return franke2(p) if p.shape[1] == 2 else franke3(p)


# ----------------------------------------------------------------------------
# hierarchies
# ----------------------------------------------------------------------------
@dataclass
class Hierarchy:
    name: str
    d: int
    k: int                      # Wendland smoothness: phi_{d,k}
    points: list                # L arrays (N(l), d) float64, row-major
    delta: list                 # L support radii
    q: list                     # L separation values handed to the API
    eval_points: np.ndarray = field(default=None)

    @property
    def L(self) -> int:
        return len(self.points)

    @property
    def n(self) -> list:
        return [int(p.shape[0]) for p in self.points]

    def f(self) -> list:
        return [franke(p) for p in self.points]


def halton_hierarchy(name, d, sizes, nu, k=1, m_eval=0):
    """Nested Halton hierarchy: X_l = first N(l) Halton points.

    delta_l = nu * (sqrt(d)/2) * N(l)^(-1/d)  (grid-equivalent fill distance
    times nu, reading C-15); q_l = 0.5 * N(l)^(-1/d) (reading C-14).
    """
    allp = halton(max(sizes), d)
    pts = [np.ascontiguousarray(allp[:n]) for n in sizes]
    delta = [nu * (math.sqrt(d) / 2.0) * n ** (-1.0 / d) for n in sizes]
    q = [0.5 * n ** (-1.0 / d) for n in sizes]
    ev = uniform_points(m_eval, d) if m_eval else None
    return Hierarchy(name, d, k, pts, delta, q, ev)


def grid_hierarchy(L, d=2, nu=4.0, k=1, first=1, m_eval=0):
    """Paper P-series (Table 1): grids l=first..first+L-1, mu=0.5, nu=4.

    h_l = sqrt(d) * 2^-(l+1), delta_l = nu*h_l, q_l = 2^-(l+1)
    (Figure 1 reproduces with exactly these, SURVEY C-15).
    """
    levels = range(first, first + L)
    pts = [grid_level(l, d) for l in levels]
    delta = [nu * math.sqrt(d) * 2.0 ** -(l + 1) for l in levels]
    q = [2.0 ** -(l + 1) for l in levels]
    ev = uniform_points(m_eval, d) if m_eval else None
    return Hierarchy(f"grid{d}d_L{L}", d, k, pts, delta, q, ev)


def config(name: str, m_eval=None) -> Hierarchy:
    """The BASELINE.json configs as concrete inputs.

    C1: d=2, Halton 100/400/1600, nu=4.
    C2: d=2, 6 levels N = 1024*4^(l-1) up to 1,048,576, nu=4.
    C3: d=3, 6 levels N = round(1e7 * 8^(l-6)) (305 ... 1e7), nu=1.5.
    C3P4/C3P5: the 4-/5-level prefixes of C3 (oracle-sized parity cases).
    C2P5: the 5-level prefix of C2 (oracle-sized parity case).
    C5: d=2, 8 levels N = round(5e7 * 4^(l-8)), nu=4.
    """
    if name == "C1":
        return halton_hierarchy("C1", 2, [100, 400, 1600], 4.0,
                                m_eval=10_000 if m_eval is None else m_eval)
    if name in ("C2", "C2P5"):
        # C2P5: the 5-level prefix of C2 (finest level 262,144 points; oracle-sized)
        L = 6 if name == "C2" else 5
        return halton_hierarchy(name, 2, [1024 * 4 ** l for l in range(L)], 4.0,
                                m_eval=(10_000 if name == "C2" else 100_000) if m_eval is None else m_eval)
    if name in ("C3", "C3P4", "C3P5", "C4", "C4F"):
        # C4 = the thresholded-factor study on the 4-level prefix of C3 (the
        # exact Lagrange build costs sum_l N(l)^2); C4F = the
        # same on all of C3 with local-patch Lagrange functions (NEXT-4)
        L = {"C3": 6, "C3P4": 4, "C3P5": 5, "C4": 4, "C4F": 6}[name]
        sizes = [int(round(1e7 * 8.0 ** (l - 6))) for l in range(1, 7)][:L]
        return halton_hierarchy(name, 3, sizes, 1.5,
                                m_eval=(10_000_000 if name in ("C3", "C4F") else 1_000_000 if name == "C4"
                                        else 100_000) if m_eval is None else m_eval)
    if name.startswith("P") and name[1:].isdigit():
        # paper workload (Table 1 / Figure 4): grids l=1..L, nu=4, phi_(3,1)
        L = int(name[1:])
        H = grid_hierarchy(L, m_eval=(100_000 if m_eval is None else m_eval))
        H.name = name
        return H
    if name == "C5":
        sizes = [int(round(5e7 * 4.0 ** (l - 8))) for l in range(1, 9)]
        return halton_hierarchy("C5", 2, sizes, 4.0,
                                m_eval=10_000_000 if m_eval is None else m_eval)
    raise ValueError(f"unknown config {name}")
