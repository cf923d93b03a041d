"""1D building blocks -- restatement of reference ``speckern/bases.py``.

TEST INFRASTRUCTURE (see ``oracle/__init__.py``).
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

GLL = "gll"  # Gauss-Lobatto-Legendre                      (bases.py:52)
GRJ1 = "grj1"  # Gauss-Radau-Jacobi, weight (1-z), z=-1 node   (bases.py:54)
GRJ2 = "grj2"  # Gauss-Radau-Jacobi, weight (1-z)^2            (bases.py:56)


def jacobi(n: int, a: float, b: float, z) -> np.ndarray:
    """P_n^{(a,b)}(z) by the standard three-term recurrence (bases.py:146-166)."""
    z = np.asarray(z, dtype=float)
    prev = np.ones_like(z)
    if n == 0:
        return prev
    cur = 0.5 * ((a + b + 2.0) * z + (a - b))
    for k in range(2, n + 1):
        s = 2.0 * k + a + b
        c1 = 2.0 * k * (k + a + b) * (s - 2.0)
        c2 = (s - 1.0) * (a * a - b * b)
        c3 = (s - 2.0) * (s - 1.0) * s
        c4 = 2.0 * (k + a - 1.0) * (k + b - 1.0) * s
        cur, prev = ((c2 + c3 * z) * cur - c4 * prev) / c1, cur
    return cur


def jacobi_d(n: int, a: float, b: float, z) -> np.ndarray:
    """dP_n^{(a,b)}/dz (bases.py:169-174)."""
    z = np.asarray(z, dtype=float)
    if n == 0:
        return np.zeros_like(z)
    return 0.5 * (n + a + b + 1.0) * jacobi(n - 1, a + 1.0, b + 1.0, z)


def _roots(n: int, a: float, b: float) -> np.ndarray:
    """Deflated Newton for the roots of P_n^{(a,b)} (bases.py:177-208)."""
    out = np.empty(n)
    for k in range(n):
        x = -math.cos(math.pi * (2.0 * k + 1.0) / (2.0 * n))
        if k:
            x = 0.5 * (x + out[k - 1])
        for _ in range(100):
            f = float(jacobi(n, a, b, x))
            fp = float(jacobi_d(n, a, b, x))
            s = float(np.sum(1.0 / (x - out[:k]))) if k else 0.0
            step = -f / (fp - s * f)
            x += step
            if abs(step) < 1e-15:
                break
        out[k] = x
    return out


@lru_cache(maxsize=None)
def quad_rule(kind: str, q: int) -> tuple[np.ndarray, np.ndarray]:
    """(points, weights) of a Q-point rule (bases.py:235-270)."""
    if kind == GLL:
        inner = _roots(q - 2, 1.0, 1.0) if q > 2 else np.empty(0)
        z = np.concatenate(([-1.0], inner, [1.0]))
        p = jacobi(q - 1, 0.0, 0.0, z)
        w = 2.0 / (q * (q - 1) * p * p)
        return z, w
    alpha = 1 if kind == GRJ1 else 2
    z = np.concatenate(([-1.0], _roots(q - 1, float(alpha), 1.0)))
    # moments of Legendre polynomials against (1-z)^alpha (bases.py:215-232)
    mom = np.zeros(q)
    if alpha == 1:
        mom[0] = 2.0
        if q > 1:
            mom[1] = -2.0 / 3.0
    else:
        mom[0] = 8.0 / 3.0
        if q > 1:
            mom[1] = -4.0 / 3.0
        if q > 2:
            mom[2] = 4.0 / 15.0
    vand = np.stack([jacobi(k, 0.0, 0.0, z) for k in range(q)])
    return z, np.linalg.solve(vand, mom)


def psi_a(p: int, z) -> np.ndarray:
    """Modified principal function (bases.py:277-290)."""
    z = np.asarray(z, dtype=float)
    if p == 0:
        return 0.5 * (1.0 - z)
    if p == 1:
        return 0.5 * (1.0 + z)
    return 0.25 * (1.0 - z) * (1.0 + z) * jacobi(p - 2, 1.0, 1.0, z)


def psi_a_d(p: int, z) -> np.ndarray:
    """d psi_a / dz (bases.py:293-304)."""
    z = np.asarray(z, dtype=float)
    if p == 0:
        return np.full_like(z, -0.5)
    if p == 1:
        return np.full_like(z, 0.5)
    return -0.5 * z * jacobi(p - 2, 1.0, 1.0, z) + 0.25 * (1.0 - z) * (
        1.0 + z
    ) * jacobi_d(p - 2, 1.0, 1.0, z)


def psi_b(p: int, q: int, z) -> np.ndarray:
    """Warped function psi^b_{pq} (bases.py:307-322)."""
    z = np.asarray(z, dtype=float)
    if p == 0:
        return psi_a(q, z)
    lead = (0.5 * (1.0 - z)) ** p
    if q == 0:
        return lead
    return lead * 0.5 * (1.0 + z) * jacobi(q - 1, 2.0 * p - 1.0, 1.0, z)


def psi_b_d(p: int, q: int, z) -> np.ndarray:
    """d psi^b_{pq} / dz (bases.py:325-340)."""
    z = np.asarray(z, dtype=float)
    if p == 0:
        return psi_a_d(q, z)
    lead = (0.5 * (1.0 - z)) ** p
    dlead = -0.5 * p * (0.5 * (1.0 - z)) ** (p - 1)
    if q == 0:
        return dlead
    j = jacobi(q - 1, 2.0 * p - 1.0, 1.0, z)
    dj = jacobi_d(q - 1, 2.0 * p - 1.0, 1.0, z)
    tail = 0.5 * (1.0 + z) * j
    return dlead * tail + lead * (0.5 * j + 0.5 * (1.0 + z) * dj)


def diff_matrix(z: np.ndarray) -> np.ndarray:
    """Barycentric collocation derivative matrix (bases.py:468-477, 399-402)."""
    dz = z[:, None] - z[None, :]
    np.fill_diagonal(dz, 1.0)
    lam = 1.0 / np.prod(dz, axis=1)
    d = (lam[None, :] / lam[:, None]) / dz
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, -np.sum(d, axis=1))
    return d
