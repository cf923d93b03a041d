"""Geometric factors and the seeded synthetic meshes.

Restatement of reference ``speckern/geometry.py`` (3D shapes) and the payload
construction of ``speckern/field_block.py:331-363``, element-major.
TEST INFRASTRUCTURE (see ``oracle/__init__.py``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle.elements import RefElement

# reference vertices (geometry.py:47-81) and edge vertices (geometry.py:84-91)
REF_VERTS = {
    "hex": np.array(
        [[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]],
        dtype=float,
    ),
    "prism": np.array(
        [[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1], [-1, 1, 1]], dtype=float
    ),
    "pyr": np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float),
    "tet": np.array([[-1, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float),
}
EDGE_VERTS = {"hex": (1, 3, 4), "prism": (1, 3, 4), "pyr": (1, 3, 4), "tet": (1, 2, 3)}


@dataclass(frozen=True)
class Geometry:
    """GeometricFactors (geometry.py:94-116): ``dxi`` is (E,3,3) regular or
    (E,NQ,3,3) deformed with ``dxi[...,i,j] = d xi_i / d x_j``; ``jac`` is
    (E,) |J| (regular) or (E,NQ) w|J| (deformed)."""

    deformed: bool
    dxi: np.ndarray
    jac: np.ndarray

    @property
    def n(self) -> int:
        return self.jac.shape[0]


def affine_geometry(shape: str, verts: np.ndarray) -> Geometry:
    """Affine factors from vertices (geometry.py:119-158)."""
    verts = np.asarray(verts, dtype=float)
    if verts.ndim == 2:
        verts = verts[None]
    edges = np.stack([verts[:, k, :] - verts[:, 0, :] for k in EDGE_VERTS[shape]], axis=-1)
    jm = 0.5 * edges
    det = np.linalg.det(jm)
    if np.any(det <= 0.0):
        raise ValueError("nonpositive Jacobian")
    return Geometry(False, np.linalg.inv(jm), det)


def deformed_geometry_from_coords(el: RefElement, coords: np.ndarray, either_orientation: bool = False) -> Geometry:
    """Iso-parametric factors (geometry.py:161-212): collocation derivatives
    on the collapsed grid, Duffy chain rule, pointwise det/inverse.
    ``either_orientation`` (assembled tet mesh only): w|det J| for reflected
    elements instead of the reference's rejection."""
    coords = np.asarray(coords, dtype=float)
    ne = coords.shape[0]
    full = coords.reshape(ne, *el.q, 3)
    dxdeta = np.empty((ne, el.nq, 3, 3))
    for m in range(3):
        t = np.moveaxis(np.tensordot(el.D[m], full, axes=([1], [m + 1])), 0, m + 1)
        dxdeta[..., m] = t.reshape(ne, el.nq, 3)
    if el.shape == "hex":
        jm = dxdeta
    else:
        # J[.., i, j] = sum_m G[j][m] dx_i/deta_m, only over structural nonzeros
        jm = np.zeros_like(dxdeta)
        for j in range(3):
            for m in range(3):
                g = el.G[:, j, m]
                if not np.any(g):
                    continue
                if np.all(g == 1.0):
                    jm[..., j] += dxdeta[..., m]
                else:
                    jm[..., j] += dxdeta[..., m] * g[None, :, None]
    det = np.linalg.det(jm)
    if either_orientation:
        det = np.abs(det)
    if np.any(det <= 0.0):
        raise ValueError("nonpositive Jacobian")
    return Geometry(True, np.linalg.inv(jm), el.refw[None, :] * det)


def quadrature_xi(el: RefElement) -> np.ndarray:
    """Standard-region coordinates of the tensor points (geometry.py:234-238;
    Duffy inverse shapes.py:218-239)."""
    e = np.stack([g.ravel() for g in np.meshgrid(*el.z, indexing="ij")], axis=-1)
    xi = e.copy()
    if el.shape == "prism":
        xi[:, 0] = 0.5 * (1.0 + e[:, 0]) * (1.0 - e[:, 2]) - 1.0
    elif el.shape == "pyr":
        xi[:, 0] = 0.5 * (1.0 + e[:, 0]) * (1.0 - e[:, 2]) - 1.0
        xi[:, 1] = 0.5 * (1.0 + e[:, 1]) * (1.0 - e[:, 2]) - 1.0
    elif el.shape == "tet":
        xi[:, 1] = 0.5 * (1.0 + e[:, 1]) * (1.0 - e[:, 2]) - 1.0
        xi[:, 0] = 0.25 * (1.0 + e[:, 0]) * (1.0 - e[:, 1]) * (1.0 - e[:, 2]) - 1.0
    return xi


def synthetic_affine_vertices(shape: str, n: int, seed: int = 0, jitter: float = 0.15) -> np.ndarray:
    """Per-element seeded affine images (geometry.py:256-272)."""
    ref = REF_VERTS[shape]
    out = np.empty((n, ref.shape[0], 3))
    for e in range(n):
        rng = np.random.default_rng(seed * 1_000_003 + e)
        mat = np.eye(3) + jitter * (rng.random((3, 3)) - 0.5)
        if np.linalg.det(mat) <= 0.0:
            mat[:, 0] = -mat[:, 0]
        out[e] = ref @ mat.T + rng.random(3)
    return out


def deformation_params(n: int, seed: int = 0, amplitude: float = 0.05, first: int = 0) -> np.ndarray:
    """Per-element draws of the sinusoidal deformation (geometry.py:275-300):
    columns amp[3], phase[3], perm[3] (as floats), shift[3]."""
    amplitude = min(amplitude, 0.1)
    out = np.empty((n, 12))
    for i in range(n):
        e = first + i
        rng = np.random.default_rng(seed * 9_999_991 + 7 * e + 1)
        out[i, 0:3] = amplitude * (0.5 + 0.5 * rng.random(3))
        out[i, 3:6] = 2.0 * np.pi * rng.random(3)
        out[i, 6:9] = rng.permutation(3)
        out[i, 9:12] = rng.random(3)
    return out


def deformed_coords(el: RefElement, params: np.ndarray) -> np.ndarray:
    """x = xi + shift + amp * sin(pi * xi[perm] + phase) at every point."""
    xi = quadrature_xi(el)
    ne = params.shape[0]
    x = np.empty((ne, el.nq, 3))
    for i in range(3):
        perm = params[:, 6 + i].astype(int)
        arg = np.pi * xi[:, perm].T + params[:, 3 + i, None]
        x[:, :, i] = (xi[None, :, i] + params[:, 9 + i, None]) + params[:, i, None] * np.sin(arg)
    return x


def synthetic_geometry(el: RefElement, deformed: bool, n: int, seed: int = 0) -> Geometry:
    """make_synthetic_factors (geometry.py:303-315)."""
    if not deformed:
        return affine_geometry(el.shape, synthetic_affine_vertices(el.shape, n, seed))
    return deformed_geometry_from_coords(el, deformed_coords(el, deformation_params(n, seed)))


# -- metric payloads, element-major (field_block.py:331-363) ----------------


def payload_lam(el: RefElement, geo: Geometry) -> list:
    """lam[i][j] = (sum_k dxi[i,k] dxi[j,k]) * jac as (n, E) arrays (n=NQ
    deformed, 1 regular); symmetric entries alias."""
    lam = [[None] * 3 for _ in range(3)]
    for i in range(3):
        for j in range(i, 3):
            prod = np.einsum("...k,...k->...", geo.dxi[..., i, :], geo.dxi[..., j, :]) * geo.jac
            arr = prod.T if geo.deformed else prod[None, :]
            lam[i][j] = lam[j][i] = np.ascontiguousarray(arr)
    return lam


def payload_w(el: RefElement, geo: Geometry) -> np.ndarray:
    """Diagonal W as (NQ, E): wj (deformed) or ref_w * |J| (regular)
    (operators.py:493-499)."""
    if geo.deformed:
        return np.ascontiguousarray(geo.jac.T)
    return el.refw[:, None] * geo.jac[None, :]


def payload_dxi(el: RefElement, geo: Geometry) -> list:
    """dxi[i][j] as (n, E) arrays."""
    out = [[None] * 3 for _ in range(3)]
    for i in range(3):
        for j in range(3):
            e = geo.dxi[..., i, j]
            out[i][j] = np.ascontiguousarray(e.T if geo.deformed else e[None, :])
    return out
