"""CPU oracle of the assembled C0 operators on conforming hex, prism, tet and
pyramid meshes (the hex section first; the others below).

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

from oracle.elements import element, mode_set
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


# ---------------------------------------------------------------------------
# Assembled C0 on a conforming prism mesh: a triangulated nx x nw grid of
# unit squares in the (x, z) plane (two triangles per square), extruded along
# y in nz element layers.  The prism's collapsed pair (xi1, xi3) spans the
# triangle, xi2 the extrusion (shapes.py:374-405: modes (p, q, r), r <= P-p,
# psi_a(p)(eta1) psi_a(q)(eta2) psi_b(p, r)(eta3), (0, q, 1) the collapsed
# vertex).  The triangle's modal set is a hierarchical C0 basis: vertex
# modes (0,0) V0, (1,0) V1, (0,1) V2; edge modes of degree k = 2..P on
# V0V1 (p=k, r=0), V1V2 (p=1, r=k-1) and V0V2 (p=0, r=k), each tracing
# psi_a(k) along its edge parameter from the lower to the higher local vertex;
# interior modes p >= 2, r >= 1.  A shared edge traversed against its global
# direction (lower global vertex id -> higher) flips the sign of its odd
# modes; triangular faces between layers and the extrusion direction need no
# orientation (every prism of a column uses the same triangle).


def _tri_topology(nx: int, nw: int):
    """Triangles as global vertex ids (V0, V1, V2) and 2D corner points;
    square (ix, iw) -> lower (c00, c10, c01), upper (c11, c01, c10)."""
    vid = lambda ix, iw: iw * (nx + 1) + ix  # noqa: E731
    tris, pts = [], []
    for iw in range(nw):
        for ix in range(nx):
            c00, c10, c01, c11 = (ix, iw), (ix + 1, iw), (ix, iw + 1), (ix + 1, iw + 1)
            for v in ((c00, c10, c01), (c11, c01, c10)):
                tris.append(tuple(vid(*c) for c in v))
                pts.append(np.array(v, dtype=float))
    return tris, pts


def _tri_dofs(nx: int, nw: int, P: int):
    """Per triangle: {(p, r): (2D global dof, sign)} and the 2D dof count."""
    tris, _ = _tri_topology(nx, nw)
    nv = (nx + 1) * (nw + 1)
    edges: dict = {}
    for t in tris:
        for a, b in ((t[0], t[1]), (t[1], t[2]), (t[0], t[2])):
            key = (min(a, b), max(a, b))
            edges.setdefault(key, len(edges))
    ni = (P - 1) * (P - 2) // 2
    base_e, base_i = nv, nv + len(edges) * (P - 1)
    out = []
    for ti, t in enumerate(tris):
        d = {(0, 0): (t[0], 1.0), (1, 0): (t[1], 1.0), (0, 1): (t[2], 1.0)}

        def edge(a, b, k):
            eid = edges[(min(a, b), max(a, b))]
            sign = 1.0 if a < b else (-1.0) ** k
            return base_e + eid * (P - 1) + (k - 2), sign

        for k in range(2, P + 1):
            d[(k, 0)] = edge(t[0], t[1], k)  # V0V1
            d[(1, k - 1)] = edge(t[1], t[2], k)  # V1V2
            d[(0, k)] = edge(t[0], t[2], k)  # V0V2
        j = 0
        for p in range(2, P + 1):
            for r in range(1, P + 1 - p):
                d[(p, r)] = (base_i + ti * ni + j, 1.0)
                j += 1
        out.append(d)
    return out, base_i + len(tris) * ni


def prism_n_global(nx: int, nw: int, nz: int, P: int) -> int:
    return _tri_dofs(nx, nw, P)[1] * (nz * P + 1)


def prism_local_to_global(nx: int, nw: int, nz: int, P: int, first_layer: int = 0, n_layers: int | None = None):
    """(l2g, sign), both (E, NM), for elements e = ez_local * NT + t of the
    layers [first_layer, first_layer + n_layers); global dofs of the slab
    vector (layer-major: extrusion node * N2D + 2D dof)."""
    tri, n2d = _tri_dofs(nx, nw, P)
    nl = nz - first_layer if n_layers is None else n_layers
    modes = mode_set("prism", P)
    E = nl * len(tri)
    l2g = np.empty((E, len(modes)), dtype=np.int64)
    sgn = np.empty((E, len(modes)))
    for ez in range(nl):
        for t, d in enumerate(tri):
            e = ez * len(tri) + t
            for m, (p, q, r) in enumerate(modes):
                layer = dof_1d(ez, q, P)  # slab-relative extrusion node
                g2, s = d[(p, r)]
                l2g[e, m] = layer * n2d + g2
                sgn[e, m] = s
    return l2g, sgn


def prism_mesh_coords(nx: int, nw: int, P: int, ez_first: int, n_layers: int, amp: float = 0.05):
    """(E, NQ, 3) quadrature coordinates: triangle point from barycentrics
    (1 - l1 - l2, l1 = (1 + xi1)/2, l2 = (1 + xi3)/2) in the (x, z) plane,
    y = layer + (1 + xi2)/2, then the global map x = X + amp sin(pi X_perm / 2)."""
    el = element("prism", P)
    xi = quadrature_xi(el)
    _, pts = _tri_topology(nx, nw)
    l1, l2 = 0.5 * (1.0 + xi[:, 0]), 0.5 * (1.0 + xi[:, 2])
    l0 = 1.0 - l1 - l2
    out = np.empty((n_layers * len(pts), el.nq, 3))
    for ez in range(n_layers):
        for t, v in enumerate(pts):
            X = np.empty((el.nq, 3))
            xz = l0[:, None] * v[0] + l1[:, None] * v[1] + l2[:, None] * v[2]
            X[:, 0], X[:, 2] = xz[:, 0], xz[:, 1]
            X[:, 1] = ez_first + ez + 0.5 * (1.0 + xi[:, 1])
            out[ez * len(pts) + t] = X + amp * np.sin(0.5 * np.pi * X[:, [1, 2, 0]])
    return out


def assembled_helmholtz_prism(nx: int, nw: int, nz: int, P: int, x: np.ndarray, lam: float, amp: float = 0.05):
    """y = sum_e A_e^T H_e A_e x with signed local-to-global maps (numpy)."""
    el = element("prism", P)
    geo = deformed_geometry_from_coords(el, prism_mesh_coords(nx, nw, P, 0, nz, amp))
    l2g, sgn = prism_local_to_global(nx, nw, nz, P)
    xe = (x[l2g] * sgn).T
    ye = helmholtz_coll(el, geo, xe, lam)
    y = np.zeros_like(x)
    np.add.at(y, l2g.T.ravel(), (ye * sgn.T).ravel())
    return y


def prism_eval(P: int, coeffs: np.ndarray, eta: np.ndarray) -> np.ndarray:
    """Expansion sum_m coeffs[m] phi_m at collapsed points eta (n, 3)
    (shapes.py:374-405 mode factors)."""
    from oracle.elements import _factor_fns

    out = np.zeros(eta.shape[0])
    for c, m in zip(coeffs, mode_set("prism", P)):
        f = _factor_fns("prism", m)
        out += c * f[0][0](eta[:, 0]) * f[1][0](eta[:, 1]) * f[2][0](eta[:, 2])
    return out


# ---------------------------------------------------------------------------
# Assembled C0 on a conforming tet mesh: nx x ny x nz unit cubes, each split
# into the six Kuhn tets along its main diagonal; every tet takes its
# vertices in global-id order (= the diagonal path order), so on every shared
# edge and face both tets use the same vertex correspondence and the modified
# basis (shapes.py:374-405) conforms with no signs or permutations: edge
# modes of degree k trace psi_a(k) from the lower to the higher vertex, face
# modes trace psi_a(a)(s) psi_b(a, b)(t) collapsed towards the face's highest
# vertex.  Half of the tets are reflected: their factors use w|det J|
# (deformed_geometry_from_coords(..., either_orientation=True)).
# Global dofs are ordered by geometric level -- plane z=0, the entities
# between z=0 and z=1, plane z=1, ... -- so a slab of cube layers owns one
# contiguous range whose first / last plane is shared with its neighbours;
# within a level, vertices, edges and faces in ascending sorted global
# vertex ids, then the tets' interior modes.

_KUHN = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def _tet_topology(nx: int, ny: int, nz: int):
    """Tets (e = ((iz*ny + iy)*nx + ix)*6 + kuhn) as ascending global vertex
    id 4-tuples, their vertex coordinates (4, 3) and the z of every vertex."""
    vid = lambda x, y, z: (z * (ny + 1) + y) * (nx + 1) + x  # noqa: E731
    tets, pts = [], []
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                for perm in _KUHN:
                    c = [ix, iy, iz]
                    vs = [tuple(c)]
                    for ax in perm:
                        c = list(c)
                        c[ax] += 1
                        vs.append(tuple(c))
                    tets.append(tuple(vid(*v) for v in vs))
                    pts.append(np.array(vs, dtype=float))
    return tets, pts


def _tet_mode_entity(P: int):
    """Per local tet mode (p, q, r): ('v', i) | ('e', (i, j), k) | ('f', (i, j, l), idx) | ('i', idx)
    with local vertex indices and the canonical face-mode index."""
    face_ab = [(a, b) for a in range(2, P + 1) for b in range(1, P + 1 - a)]
    fidx = {ab: i for i, ab in enumerate(face_ab)}
    out, ni = [], 0
    for p, q, r in mode_set("tet", P):
        if (p, q, r) in ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)):
            out.append(("v", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)].index((p, q, r))))
        elif q == 0 and r == 0:
            out.append(("e", (0, 1), p))
        elif p == 0 and r == 0:
            out.append(("e", (0, 2), q))
        elif p == 1 and r == 0:
            out.append(("e", (1, 2), q + 1))
        elif p == 0 and q == 0:
            out.append(("e", (0, 3), r))
        elif p == 1 and q == 0:
            out.append(("e", (1, 3), r + 1))
        elif p == 0 and q == 1:
            out.append(("e", (2, 3), r + 1))
        elif r == 0:
            out.append(("f", (0, 1, 2), fidx[(p, q)]))
        elif q == 0:
            out.append(("f", (0, 1, 3), fidx[(p, r)]))
        elif p == 0:
            out.append(("f", (0, 2, 3), fidx[(q, r)]))
        elif p == 1:
            out.append(("f", (1, 2, 3), fidx[(q + 1, r)]))
        else:
            out.append(("i", ni))
            ni += 1
    return out, len(face_ab), ni


def _tet_numbering(nx: int, ny: int, nz: int, P: int):
    """Global dof of every (tet, local mode), the per-level dof offsets and
    the plane size (dofs of one z = const plane)."""
    tets, _ = _tet_topology(nx, ny, nz)
    ent, nf, ni = _tet_mode_entity(P)
    zof = lambda v: v // ((nx + 1) * (ny + 1))  # noqa: E731
    size = {"v": 1, "e": P - 1, "f": nf}
    levels: dict = {}  # level -> {(kind, verts): None}
    for t in tets:
        for kind, k in (("v", 1), ("e", 2), ("f", 3)):
            for sub in _subsets(t, k):
                zs = [zof(v) for v in sub]
                lev = 2 * min(zs) + (0 if min(zs) == max(zs) else 1)
                levels.setdefault(lev, {})[(kind, sub)] = None
    order = {"v": 0, "e": 1, "f": 2}
    start, offs = 0, {}
    level_start = {}
    for lev in range(2 * nz + 1):
        level_start[lev] = start
        ents = sorted(levels.get(lev, {}), key=lambda x: (order[x[0]], x[1]))
        for kind, sub in ents:
            offs[(kind, sub)] = start
            start += size[kind]
        if lev % 2 == 1:  # interiors of the tets of cube layer lev // 2
            iz = lev // 2
            for e in range(iz * nx * ny * 6, (iz + 1) * nx * ny * 6):
                offs[("i", e)] = start
                start += ni
    level_start[2 * nz + 1] = start
    l2g = np.empty((len(tets), len(ent)), dtype=np.int64)
    for e, t in enumerate(tets):
        for m, en in enumerate(ent):
            if en[0] == "v":
                l2g[e, m] = offs[("v", (t[en[1]],))]
            elif en[0] == "e":
                l2g[e, m] = offs[("e", tuple(t[i] for i in en[1]))] + en[2] - 2
            elif en[0] == "f":
                l2g[e, m] = offs[("f", tuple(t[i] for i in en[1]))] + en[2]
            else:
                l2g[e, m] = offs[("i", e)] + en[1]
    plane = level_start[1] - level_start[0]
    return l2g, level_start, plane


def _subsets(t, k):
    import itertools

    return [tuple(c) for c in itertools.combinations(t, k)]


def tet_n_global(nx: int, ny: int, nz: int, P: int) -> int:
    return _tet_numbering(nx, ny, nz, P)[1][2 * nz + 1]


def tet_mesh_coords(nx: int, ny: int, nz: int, P: int, amp: float = 0.05):
    """(E, NQ, 3): affine image of the reference tet on each Kuhn tet
    (x = v0 + sum_i (1 + xi_i)/2 (v_i - v0)), then the global deformation."""
    el = element("tet", P)
    xi = quadrature_xi(el)
    _, pts = _tet_topology(nx, ny, nz)
    lam = 0.5 * (1.0 + xi)  # (NQ, 3)
    out = np.empty((len(pts), el.nq, 3))
    for e, v in enumerate(pts):
        X = v[0][None, :] + lam @ (v[1:] - v[0][None, :])
        out[e] = X + amp * np.sin(0.5 * np.pi * X[:, [1, 2, 0]])
    return out


def assembled_helmholtz_tet(nx: int, ny: int, nz: int, P: int, x: np.ndarray, lam: float, amp: float = 0.05):
    """y = sum_e A_e^T H_e A_e x (numpy), factors with w|det J|."""
    el = element("tet", P)
    geo = deformed_geometry_from_coords(el, tet_mesh_coords(nx, ny, nz, P, amp), either_orientation=True)
    l2g, _, _ = _tet_numbering(nx, ny, nz, P)
    ye = helmholtz_coll(el, geo, x[l2g].T, lam)
    y = np.zeros_like(x)
    np.add.at(y, l2g.T.ravel(), ye.ravel())
    return y


def tet_eval(P: int, coeffs: np.ndarray, eta: np.ndarray) -> np.ndarray:
    """Tet expansion at collapsed points eta (n, 3)."""
    from oracle.elements import _factor_fns

    out = np.zeros(eta.shape[0])
    for c, m in zip(coeffs, mode_set("tet", P)):
        f = _factor_fns("tet", m)
        out += c * f[0][0](eta[:, 0]) * f[1][0](eta[:, 1]) * f[2][0](eta[:, 2])
    return out


TET_REF = np.array([[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])


def tet_collapse(xi: np.ndarray) -> np.ndarray:
    """Duffy map xi -> eta of the tet (shapes.py:218-239), away from the
    collapsed points."""
    eta = np.empty_like(xi)
    eta[:, 0] = 2.0 * (1.0 + xi[:, 0]) / (-xi[:, 1] - xi[:, 2]) - 1.0
    eta[:, 1] = 2.0 * (1.0 + xi[:, 1]) / (1.0 - xi[:, 2]) - 1.0
    eta[:, 2] = xi[:, 2]
    return eta


# ---------------------------------------------------------------------------
# Assembled C0 on a conforming pyramid mesh: nx x ny x nz unit cubes, each
# split into six pyramids with the cube centre as apex and a cube face as
# base.  Every pyramid's base axes (eta1, eta2) run along the face's two
# global axes (lower axis first) in increasing direction from the face's
# minimum corner (V0), so shared base quads, shared triangular faces (base
# edge + apex) and every edge are parameterised alike on both sides
# (shapes.py:374-405 pyramid modes: psi_a(p) psi_a(q) psi_b(max(p,q), r),
# (0,0,1) the apex); reflected pyramids use w|det J|.  Dofs are ordered by
# level like the tet mesh (corner z = iz, cube centres between).

_PYR_FACES = ((0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1))  # (normal axis, side)


def _pyr_topology(nx: int, ny: int, nz: int):
    """Pyramids (e = cube * 6 + face) as vertex id 5-tuples (V0..V3 base,
    V4 apex; corners (z*(ny+1)+y)*(nx+1)+x, centres n_corners + cube),
    their doubled-z levels and vertex coordinates (5, 3)."""
    nc = (nx + 1) * (ny + 1) * (nz + 1)
    vid = lambda c: (c[2] * (ny + 1) + c[1]) * (nx + 1) + c[0]  # noqa: E731
    pyrs, pts, z2 = [], [], []
    cube = 0
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                o = np.array([ix, iy, iz])
                for n, side in _PYR_FACES:
                    a, b = [ax for ax in range(3) if ax != n]
                    v0 = o.copy()
                    v0[n] += side
                    ea, eb = np.eye(3, dtype=int)[a], np.eye(3, dtype=int)[b]
                    base = [v0, v0 + ea, v0 + ea + eb, v0 + eb]
                    pyrs.append(tuple(vid(c) for c in base) + (nc + cube,))
                    pts.append(np.array([*base, o + 0.5], dtype=float))
                    z2.append(tuple(2 * c[2] for c in base) + (2 * iz + 1,))
                cube += 1
    return pyrs, pts, z2


def _pyr_mode_entity(P: int):
    """Per local pyramid mode: ('v', i) | ('e', (i, j), degree) |
    ('q', canonical quad index) | ('t', (i, j, k), canonical triangle index) | ('i', idx)."""
    tri = {ab: i for i, ab in enumerate((a, b) for a in range(2, P + 1) for b in range(1, P + 1 - a))}
    quad = {pq: i for i, pq in enumerate((p, q) for p in range(2, P + 1) for q in range(2, P + 1))}
    vert = {(0, 0, 0): 0, (1, 0, 0): 1, (1, 1, 0): 2, (0, 1, 0): 3, (0, 0, 1): 4}
    out, ni = [], 0
    for p, q, r in mode_set("pyr", P):
        if (p, q, r) in vert:
            out.append(("v", vert[(p, q, r)]))
        elif r == 0 and q in (0, 1) and p >= 2:
            out.append(("e", (0, 1) if q == 0 else (3, 2), p))
        elif r == 0 and p in (0, 1) and q >= 2:
            out.append(("e", (0, 3) if p == 0 else (1, 2), q))
        elif r == 0:
            out.append(("q", quad[(p, q)]))
        elif p in (0, 1) and q in (0, 1):
            base = {(0, 0): 0, (1, 0): 1, (1, 1): 2, (0, 1): 3}[(p, q)]
            out.append(("e", (base, 4), r + (1 if (p, q) != (0, 0) else 0)))
        elif q in (0, 1):  # p >= 2: faces V0 V1 V4 (eta2 = -1) / V3 V2 V4 (eta2 = 1)
            out.append(("t", (0, 1, 4) if q == 0 else (3, 2, 4), tri[(p, r)]))
        elif p in (0, 1):  # q >= 2: faces V0 V3 V4 (eta1 = -1) / V1 V2 V4 (eta1 = 1)
            out.append(("t", (0, 3, 4) if p == 0 else (1, 2, 4), tri[(q, r)]))
        else:
            out.append(("i", ni))
            ni += 1
    return out, len(quad), len(tri), ni


def _pyr_numbering(nx: int, ny: int, nz: int, P: int):
    pyrs, _, z2 = _pyr_topology(nx, ny, nz)
    ent, nq, nt, ni = _pyr_mode_entity(P)
    size = {"v": 1, "e": P - 1, "q": nq, "t": nt}
    levels: dict = {}
    zmap = {}
    for t, zz in zip(pyrs, z2):
        for v, z in zip(t, zz):
            zmap[v] = z

    def level(sub):
        zs = [zmap[v] for v in sub]
        if min(zs) == max(zs) and min(zs) % 2 == 0:
            return min(zs)
        return 2 * (min(zs) // 2) + 1

    for t in pyrs:
        subs = [("v", (v,)) for v in t]
        subs += [("e", tuple(sorted((t[i], t[j])))) for i, j in ((0, 1), (3, 2), (0, 3), (1, 2), (0, 4), (1, 4), (2, 4), (3, 4))]
        subs += [("q", tuple(sorted(t[:4])))]
        subs += [("t", tuple(sorted(t[i] for i in f))) for f in ((0, 1, 4), (3, 2, 4), (0, 3, 4), (1, 2, 4))]
        for kind, sub in subs:
            levels.setdefault(level(sub), {})[(kind, sub)] = None
    order = {"v": 0, "e": 1, "q": 2, "t": 3}
    start, offs, level_start = 0, {}, {}
    per_layer = nx * ny * 6
    for lev in range(2 * nz + 1):
        level_start[lev] = start
        for kind, sub in sorted(levels.get(lev, {}), key=lambda x: (order[x[0]], x[1])):
            offs[(kind, sub)] = start
            start += size[kind]
        if lev % 2 == 1:
            for e in range((lev // 2) * per_layer, (lev // 2 + 1) * per_layer):
                offs[("i", e)] = start
                start += ni
    level_start[2 * nz + 1] = start
    l2g = np.empty((len(pyrs), len(ent)), dtype=np.int64)
    for e, t in enumerate(pyrs):
        for m, en in enumerate(ent):
            k = en[0]
            if k == "v":
                l2g[e, m] = offs[("v", (t[en[1]],))]
            elif k == "e":
                l2g[e, m] = offs[("e", tuple(sorted(t[i] for i in en[1])))] + en[2] - 2
            elif k == "q":
                l2g[e, m] = offs[("q", tuple(sorted(t[:4])))] + en[1]
            elif k == "t":
                l2g[e, m] = offs[("t", tuple(sorted(t[i] for i in en[1])))] + en[2]
            else:
                l2g[e, m] = offs[("i", e)] + en[1]
    return l2g, level_start, level_start[1] - level_start[0]


def pyr_n_global(nx: int, ny: int, nz: int, P: int) -> int:
    return _pyr_numbering(nx, ny, nz, P)[1][2 * nz + 1]


def pyr_mesh_coords(nx: int, ny: int, nz: int, P: int, amp: float = 0.05):
    """(E, NQ, 3): x = V0 + l1 (V1 - V0) + l2 (V3 - V0) + l3 (V4 - V0),
    l_i = (1 + xi_i)/2 (the reference pyramid's apex is xi = (-1,-1,1)), then
    the global deformation."""
    el = element("pyr", P)
    xi = quadrature_xi(el)
    _, pts, _ = _pyr_topology(nx, ny, nz)
    lam = 0.5 * (1.0 + xi)
    out = np.empty((len(pts), el.nq, 3))
    for e, v in enumerate(pts):
        X = v[0][None, :] + lam @ np.stack([v[1] - v[0], v[3] - v[0], v[4] - v[0]])
        out[e] = X + amp * np.sin(0.5 * np.pi * X[:, [1, 2, 0]])
    return out


def assembled_helmholtz_pyr(nx: int, ny: int, nz: int, P: int, x: np.ndarray, lam: float, amp: float = 0.05):
    el = element("pyr", P)
    geo = deformed_geometry_from_coords(el, pyr_mesh_coords(nx, ny, nz, P, amp), either_orientation=True)
    l2g, _, _ = _pyr_numbering(nx, ny, nz, P)
    ye = helmholtz_coll(el, geo, x[l2g].T, lam)
    y = np.zeros_like(x)
    np.add.at(y, l2g.T.ravel(), ye.ravel())
    return y


PYR_REF = np.array([[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [1.0, 1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])


def pyr_collapse(xi: np.ndarray) -> np.ndarray:
    eta = np.empty_like(xi)
    eta[:, 0] = 2.0 * (1.0 + xi[:, 0]) / (1.0 - xi[:, 2]) - 1.0
    eta[:, 1] = 2.0 * (1.0 + xi[:, 1]) / (1.0 - xi[:, 2]) - 1.0
    eta[:, 2] = xi[:, 2]
    return eta


def pyr_eval(P: int, coeffs: np.ndarray, eta: np.ndarray) -> np.ndarray:
    from oracle.elements import _factor_fns

    out = np.zeros(eta.shape[0])
    for c, m in zip(coeffs, mode_set("pyr", P)):
        f = _factor_fns("pyr", m)
        out += c * f[0][0](eta[:, 0]) * f[1][0](eta[:, 1]) * f[2][0](eta[:, 2])
    return out
