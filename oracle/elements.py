"""Reference elements: quadrature composition, modes, sum-fac tables, Duffy G.

Restatement of reference ``speckern/shapes.py`` for the four 3D shapes of the
hot path.  TEST INFRASTRUCTURE (see ``oracle/__init__.py``).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from oracle.basis1d import GLL, GRJ1, GRJ2, diff_matrix, psi_a, psi_a_d, psi_b, psi_b_d, quad_rule

#: shapes in the reference ``Shape`` enum order (shapes.py:57-65); the enum
#: index is part of the bench seed key (bench.py:261)
SHAPES = ("quad", "tri", "hex", "prism", "pyr", "tet")
SHAPE_INDEX = {s: i for i, s in enumerate(SHAPES)}

# per-direction rule kinds (shapes.py:76-98) and Duffy scale (shapes.py:102-109)
_KINDS = {
    "hex": (GLL, GLL, GLL),
    "prism": (GLL, GLL, GRJ1),
    "pyr": (GLL, GLL, GRJ2),
    "tet": (GLL, GRJ1, GRJ2),
}
_SCALE = {
    "hex": (1.0, 1.0, 1.0),
    "prism": (1.0, 1.0, 0.5),
    "pyr": (1.0, 1.0, 0.25),
    "tet": (1.0, 0.5, 0.25),
}


def mode_count(shape: str, P: int) -> int:
    """shapes.py:112-129."""
    return {
        "hex": (P + 1) ** 3,
        "prism": (P + 1) ** 2 * (P + 2) // 2,
        "pyr": (P + 1) * (P + 2) * (2 * P + 3) // 6,
        "tet": (P + 1) * (P + 2) * (P + 3) // 6,
    }[shape]


def qcounts(shape: str, P: int) -> tuple[int, int, int]:
    """P+2 Lobatto points, P+1 Radau points per direction (shapes.py:132-139)."""
    return tuple(P + 2 if k == GLL else P + 1 for k in _KINDS[shape])


def mode_set(shape: str, P: int) -> list[tuple[int, int, int]]:
    """Lexicographic admissible (p, q, r), p slowest (shapes.py:142-179)."""
    out = []
    for p in range(P + 1):
        for q in range(P + 1 - p if shape == "tet" else P + 1):
            if shape == "hex":
                nr = P + 1
            elif shape == "prism":
                nr = P + 1 - p
            elif shape == "pyr":
                nr = P + 1 - max(p, q)
            else:
                nr = P + 1 - p - q
            out.extend((p, q, r) for r in range(nr))
    return out


def _factor_fns(shape: str, m: tuple[int, int, int]):
    """Per-direction (value, derivative) factor of one mode, including the
    collapsed-vertex special cases (shapes.py:374-405)."""
    p, q, r = m
    one = (lambda z: np.ones_like(z), lambda z: np.zeros_like(z))
    A = lambda i: (lambda z: psi_a(i, z), lambda z: psi_a_d(i, z))  # noqa: E731
    Bf = lambda i, j: (lambda z: psi_b(i, j, z), lambda z: psi_b_d(i, j, z))  # noqa: E731
    if shape == "hex":
        return [A(p), A(q), A(r)]
    if shape == "prism":
        if p == 0 and r == 1:
            return [one, A(q), Bf(0, 1)]
        return [A(p), A(q), Bf(p, r)]
    if shape == "pyr":
        if (p, q, r) == (0, 0, 1):
            return [one, one, Bf(0, 1)]
        return [A(p), A(q), Bf(max(p, q), r)]
    if (p, q, r) == (0, 0, 1):
        return [one, one, Bf(0, 1)]
    if (p, q) == (0, 1):
        return [one, Bf(0, 1), Bf(1, r)]
    return [A(p), Bf(p, q), Bf(p + q, r)]


@dataclass(frozen=True)
class RefElement:
    """Everything per (shape, P) the operators consume (shapes.py:412-456)."""

    shape: str
    P: int
    q: tuple[int, int, int]
    nq: int
    nm: int
    modes: list
    z: tuple  # 1D points per direction (collapsed coordinates eta)
    w: tuple  # 1D weights per direction (unscaled)
    refw: np.ndarray  # (nq,) tensor weights incl. Duffy scale
    D: tuple  # collocation matrices per direction
    G: np.ndarray  # (nq, 3, 3) dense chain-rule factors, grad_xi = G grad_eta
    a: tuple  # per direction (vals, ders) Q_d x (P+1), or None when warped
    b2: tuple | None  # warped family dir 1: per p (vals, ders) Q2 x (P+1-p)
    c3: tuple | None  # warped family dir 2: per k (vals, ders) Q3 x (P+1-k)
    bmat: np.ndarray  # dense (nq, nm)
    dbmat: tuple  # dense (nq, nm) collocation derivatives per direction


def _g_dense(shape: str, z: tuple, q: tuple) -> np.ndarray:
    """Duffy chain-rule factors on the tensor grid (shapes.py:265-323)."""
    e1, e2, e3 = (g.ravel() for g in np.meshgrid(*z, indexing="ij"))
    n = e1.size
    g = np.zeros((n, 3, 3))
    if shape == "hex":
        g[:, 0, 0] = g[:, 1, 1] = g[:, 2, 2] = 1.0
    elif shape == "prism":
        g[:, 0, 0] = 2.0 / (1.0 - e3)
        g[:, 1, 1] = 1.0
        g[:, 2, 0] = (1.0 + e1) / (1.0 - e3)
        g[:, 2, 2] = 1.0
    elif shape == "pyr":
        g[:, 0, 0] = 2.0 / (1.0 - e3)
        g[:, 1, 1] = 2.0 / (1.0 - e3)
        g[:, 2, 0] = (1.0 + e1) / (1.0 - e3)
        g[:, 2, 1] = (1.0 + e2) / (1.0 - e3)
        g[:, 2, 2] = 1.0
    else:
        g[:, 0, 0] = 4.0 / ((1.0 - e2) * (1.0 - e3))
        g[:, 1, 0] = 2.0 * (1.0 + e1) / ((1.0 - e2) * (1.0 - e3))
        g[:, 1, 1] = 2.0 / (1.0 - e3)
        g[:, 2, 0] = 2.0 * (1.0 + e1) / ((1.0 - e2) * (1.0 - e3))
        g[:, 2, 1] = (1.0 + e2) / (1.0 - e3)
        g[:, 2, 2] = 1.0
    return g


def _a_pair(P: int, z: np.ndarray):
    return (
        np.stack([psi_a(p, z) for p in range(P + 1)], axis=1),
        np.stack([psi_a_d(p, z) for p in range(P + 1)], axis=1),
    )


def _warped(P: int, z: np.ndarray):
    """Per-leading-index slices of the psi^b family (bases.py:445-465)."""
    return tuple(
        (
            np.stack([psi_b(p, q, z) for q in range(P + 1 - p)], axis=1),
            np.stack([psi_b_d(p, q, z) for q in range(P + 1 - p)], axis=1),
        )
        for p in range(P + 1)
    )


@lru_cache(maxsize=None)
def element(shape: str, P: int, q: tuple | None = None) -> RefElement:
    """Assemble the per-(shape, P) bundle (shapes.py:466-518, 555-583);
    ``q`` overrides the per-direction point counts (build_shape_basis
    qpoints, shapes.py:521-541)."""
    q = qcounts(shape, P) if q is None else tuple(int(v) for v in q)
    rules = [quad_rule(k, n) for k, n in zip(_KINDS[shape], q)]
    z = tuple(r[0] for r in rules)
    w = tuple(r[1] for r in rules)
    ws = [wd * s for wd, s in zip(w, _SCALE[shape])]
    refw = np.multiply.outer(np.multiply.outer(ws[0], ws[1]), ws[2]).ravel()
    D = tuple(diff_matrix(zd) for zd in z)
    modes = mode_set(shape, P)
    cols = []
    for m in modes:
        f = _factor_fns(shape, m)
        v = np.multiply.outer(np.multiply.outer(f[0][0](z[0]), f[1][0](z[1])), f[2][0](z[2]))
        cols.append(v.ravel())
    bmat = np.stack(cols, axis=1)
    dbmat = []
    for d in range(3):
        full = bmat.reshape(*q, -1)
        t = np.moveaxis(np.tensordot(D[d], full, axes=([1], [d])), 0, d)
        dbmat.append(np.ascontiguousarray(t.reshape(bmat.shape)))
    a = [None, None, None]
    b2 = c3 = None
    a[0] = _a_pair(P, z[0])
    if shape in ("hex", "prism", "pyr"):
        a[1] = _a_pair(P, z[1])
    if shape == "hex":
        a[2] = _a_pair(P, z[2])
    if shape == "tet":
        b2 = _warped(P, z[1])
    if shape != "hex":
        c3 = _warped(P, z[2])
    return RefElement(
        shape=shape,
        P=P,
        q=q,
        nq=int(np.prod(q)),
        nm=len(modes),
        modes=modes,
        z=z,
        w=w,
        refw=refw,
        D=D,
        G=_g_dense(shape, z, q),
        a=tuple(a),
        b2=b2,
        c3=c3,
        bmat=bmat,
        dbmat=tuple(dbmat),
    )
