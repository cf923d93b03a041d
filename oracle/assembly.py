"""CPU oracle of the assembled C0 operator on a conforming hex mesh.

The reference stops at elemental operators (global assembly is out of its
scope), so this restatement is the checker for the
assembled variant: y = A^T H_e A x, where A gathers element modal
coefficients from global C0 DOFs and H_e is the reference's elemental
collocated Helmholtz (oracle.ops.helmholtz_coll, pinned to speckern).
"parity unpinned" against the reference itself (it has no assembly); it is
pinned through the elemental operator and checked by C0 invariants (the
assembled stiffness annihilates constants, the assembled operator is
symmetric).  TEST INFRASTRUCTURE.

Mesh: nx x ny x nz hexes of the box [0, nx] x [0, ny] x [0, nz], all
elements aligned with the global axes (so shared vertex/edge/face modes
need no orientation signs), mapped by a smooth global deformation.
Global DOFs form a tensor product of 1D C0 numberings: along x, the modal
index p of element ex maps to ex*P + (0 if p == 0 else P if p == 1 else p-1).
"""

from __future__ import annotations

import numpy as np

from oracle.elements import element
from oracle.geom import deformed_geometry_from_coords, quadrature_xi
from oracle.ops import helmholtz_coll


def dof_1d(e: int, p: int, P: int) -> int:
    return e * P + (0 if p == 0 else P if p == 1 else p - 1)


def local_to_global(nx: int, ny: int, nz: int, P: int, first: int = 0, count: int | None = None) -> np.ndarray:
    """(E, NM) global DOF of every local mode, elements e = (ez*ny+ey)*nx+ex
    in [first, first + count)."""
    E = nx * ny * nz if count is None else count
    P1 = P + 1
    Nx, Ny = nx * P + 1, ny * P + 1
    out = np.empty((E, P1**3), dtype=np.int64)
    pm = np.array([0 if p == 0 else P if p == 1 else p - 1 for p in range(P1)])
    for i in range(E):
        e = first + i
        ex, rest = e % nx, e // nx
        ey, ez = rest % ny, rest // ny
        gx = ex * P + pm
        gy = ey * P + pm
        gz = ez * P + pm
        out[i] = ((gz[None, None, :] * Ny + gy[None, :, None]) * Nx + gx[:, None, None]).ravel()
    return out


def mesh_coords(nx: int, ny: int, nz: int, P: int, amp: float = 0.05, first: int = 0, count: int | None = None):
    """Quadrature-point coordinates (E, NQ, 3) of the conforming deformed
    mesh: element (ex,ey,ez) maps xi in [-1,1]^3 to the global point
    X = g + 0.5 (xi + 1), g = (ex, ey, ez), then x = X + amp sin(pi X_perm / 2)
    (one smooth global map, so neighbouring elements share faces)."""
    el = element("hex", P)
    xi = quadrature_xi(el)
    E = nx * ny * nz if count is None else count
    out = np.empty((E, el.nq, 3))
    for i in range(E):
        e = first + i
        ex, rest = e % nx, e // nx
        ey, ez = rest % ny, rest // ny
        X = np.array([ex, ey, ez], dtype=float)[None, :] + 0.5 * (xi + 1.0)
        out[i] = X + amp * np.sin(0.5 * np.pi * X[:, [1, 2, 0]])
    return out


def assembled_helmholtz(nx: int, ny: int, nz: int, P: int, x: np.ndarray, lam: float, amp: float = 0.05):
    """y = A^T H_e A x on the whole mesh (numpy)."""
    el = element("hex", P)
    geo = deformed_geometry_from_coords(el, mesh_coords(nx, ny, nz, P, amp))
    l2g = local_to_global(nx, ny, nz, P)
    xe = x[l2g].T  # (NM, E)
    ye = helmholtz_coll(el, geo, xe, lam)
    y = np.zeros_like(x)
    np.add.at(y, l2g.T.ravel(), ye.ravel())
    return y


def n_global(nx: int, ny: int, nz: int, P: int) -> int:
    return (nx * P + 1) * (ny * P + 1) * (nz * P + 1)
