"""Dense quadrature-sum elemental matrices (independent route).

Restatement of reference ``speckern/oracle.py``.  TEST INFRASTRUCTURE.
"""

from __future__ import annotations

import numpy as np

from oracle.elements import RefElement
from oracle.geom import Geometry


def _pointwise(el: RefElement, geo: Geometry, e: int):
    """(w|J| per point, dxi per point) of one element (oracle.py:81-93)."""
    if geo.deformed:
        return geo.jac[e], geo.dxi[e]
    return el.refw * geo.jac[e], np.broadcast_to(geo.dxi[e], (el.nq, 3, 3))


def _grad_xi(el: RefElement) -> np.ndarray:
    """d phi / d xi_i (3, nq, nm) by collocation + chain rule (oracle.py:61-78)."""
    deta = np.stack(el.dbmat)
    return np.einsum("lij,jlm->ilm", el.G, deta)


def dense_mass(el: RefElement, geo: Geometry, e: int = 0) -> np.ndarray:
    """oracle.py:101-107."""
    wj, _ = _pointwise(el, geo, e)
    return np.einsum("lm,l,ln->mn", el.bmat, wj, el.bmat)


def dense_helmholtz(el: RefElement, geo: Geometry, lam: float, e: int = 0) -> np.ndarray:
    """Literal quadrature double sum, Eq. 7 (oracle.py:110-127)."""
    wj, dxi = _pointwise(el, geo, e)
    gx = np.einsum("lij,ilm->jlm", dxi, _grad_xi(el))
    h = lam * np.einsum("lm,l,ln->mn", el.bmat, wj, el.bmat)
    return h + np.einsum("jlm,l,jln->mn", gx, wj, gx)


def _tensor_d(el: RefElement, d: int) -> np.ndarray:
    mats = [np.eye(q) for q in el.q]
    mats[d] = el.D[d]
    return np.kron(np.kron(mats[0], mats[1]), mats[2])


def dense_helmholtz_factored(el: RefElement, geo: Geometry, lam: float, e: int = 0) -> np.ndarray:
    """B^T { sum_j E_j^T W E_j + lam W } B, Eq. 20 (oracle.py:130-157)."""
    wj, dxi = _pointwise(el, geo, e)
    t = np.einsum("lij,lim->ljm", dxi, el.G)
    dfull = [_tensor_d(el, k) for k in range(3)]
    core = lam * np.diag(wj)
    for j in range(3):
        ej = sum(t[:, j, m, None] * dfull[m] for m in range(3))
        core = core + ej.T @ (wj[:, None] * ej)
    return el.bmat.T @ core @ el.bmat
