"""Assembled C0 Helmholtz on a conforming hex mesh, sharded by z-slabs
(BASELINE configs[4] "with assembled C0 variant").

y = A^T H_e A x: the elemental collocated Helmholtz kernel with the gather
(global C0 DOFs -> element modal coefficients) fused into its tile load
(sk_helmholtz_apply_c0; the stand-alone sk_c0_gather serves lam = 0), then a
deterministic device scatter (sk_c0_scatter).  Each rank owns
a contiguous slab of element layers; the two DOF layers on a slab boundary
are shared with the neighbouring ranks and are summed by one neighbour
exchange over NCCL (``torch.distributed`` P2P: send/recv of one
(nx*P+1) x (ny*P+1) layer to each neighbour) -- the only communication in
any operator of this package.

The reference has no global assembly; parity is against
the CPU restatement ``oracle/assembly.py`` built on the reference's
elemental operator.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from paper_2604_04644_b200 import _lib
from paper_2604_04644_b200.field_block import AccessQualifier, Block, FieldState
from paper_2604_04644_b200.geometry import deformed_factors_from_coords, quadrature_coords
from paper_2604_04644_b200.operators import helmholtz_apply
from paper_2604_04644_b200.sharding import partition
from paper_2604_04644_b200.shapes import Shape, build_shape_basis

__all__ = ["C0HexMesh", "C0PrismMesh", "C0TetMesh", "C0PyrMesh", "exchange_interfaces"]


def exchange_interfaces(y, layer: int, group=None) -> None:
    """Sum the shared first/last DOF layers of a z-slab vector ``y`` with the
    neighbouring ranks (in place).  Works on CUDA tensors (NCCL) and CPU
    tensors (gloo)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return
    world = dist.get_world_size(group)
    if world == 1:
        return
    rank = dist.get_rank(group)
    if y.is_cuda and dist.get_backend(group) == "gloo":
        # gloo point-to-point moves host tensors: exchange host copies of the
        # two boundary layers and add the neighbours' sums back on the device
        h = torch.cat([y[:layer], y[-layer:]]).cpu()
        lo_h, hi_h = h[:layer].clone(), h[layer:].clone()
        _exchange(lo_h, hi_h, rank, world, group)
        y[:layer] = lo_h.to(y.device)
        y[-layer:] = hi_h.to(y.device)
        return
    _exchange(y[:layer], y[-layer:], rank, world, group)


def _exchange(lo, hi, rank: int, world: int, group) -> None:
    """lo += lower neighbour's hi layer, hi += upper neighbour's lo layer."""
    import torch
    import torch.distributed as dist

    recv_lo = torch.empty_like(lo) if rank > 0 else None
    recv_hi = torch.empty_like(hi) if rank < world - 1 else None
    ops = []
    if rank > 0:
        peer = dist.get_global_rank(group, rank - 1) if group is not None else rank - 1
        ops += [dist.P2POp(dist.isend, lo.contiguous(), peer, group), dist.P2POp(dist.irecv, recv_lo, peer, group)]
    if rank < world - 1:
        peer = dist.get_global_rank(group, rank + 1) if group is not None else rank + 1
        ops += [dist.P2POp(dist.isend, hi.contiguous(), peer, group), dist.P2POp(dist.irecv, recv_hi, peer, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if recv_lo is not None:
        lo += recv_lo
    if recv_hi is not None:
        hi += recv_hi


class C0HexMesh:
    """This rank's slab of an nx x ny x nz conforming hex mesh of order P,
    deformed by one smooth global map x = X + amp sin(pi X_perm / 2)
    (X = global box coordinates), with its elemental Helmholtz payload on
    the device."""

    def __init__(self, nx: int, ny: int, nz: int, order: int, amp: float = 0.05, rank: int = 0, world: int = 1):
        import torch

        if nz < world:
            # an empty slab would leave its scatter output unwritten, and the
            # one-hop exchange cannot sum a layer shared by ranks r-1 and r+1
            raise ValueError(f"need at least one element layer per rank: nz={nz} < world={world}")
        self.nx, self.ny, self.nz, self.P, self.amp = nx, ny, nz, order, amp
        self.z0, self.nzl = partition(nz, world, rank)
        self.first = self.z0 * nx * ny
        self.E = self.nzl * nx * ny
        self.layer = (nx * order + 1) * (ny * order + 1)
        self.n_dofs = self.layer * (self.nzl * order + 1)  # slab DOFs incl. both end layers
        self.basis = build_shape_basis(Shape.HEX, order)
        dev = torch.device("cuda", torch.cuda.current_device())
        xi = torch.as_tensor(quadrature_coords(self.basis), device=dev)
        e = torch.arange(self.first, self.first + self.E, device=dev)
        g = torch.stack([e % nx, (e // nx) % ny, e // (nx * ny)], dim=-1).to(torch.float64)
        X = g[:, None, :] + 0.5 * (xi[None] + 1.0)
        coords = X + amp * torch.sin(0.5 * np.pi * X[..., [1, 2, 0]])
        self.factors = deformed_factors_from_coords(self.basis, coords)
        del coords, X
        self.block = Block(self.basis, self.factors, FieldState.COEFF, 1, 1)
        self.out = self.block.like(FieldState.COEFF)

    def helmholtz(self, x, lam: float, group=None):
        """y = A^T H_e A x for this slab's DOF vector x (CUDA, length
        n_dofs, end layers holding the shared values); returns y with the
        shared layers summed across ranks."""
        import torch

        lib = _lib.load()
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        W = 1
        if lam > 0.0:
            # gather fused into the Helmholtz tile load (no A x round trip through
            # HBM).  SK_C0_HEX_MODEMAJOR=1 stores the elemental result mode-major
            # ([mode][element], W = E) for a scatter coalesced along x: measured
            # 4 % slower than element-major + the tiled scatter
            pay = self.block.payload(_lib.SK_PAYLOAD_HELMHOLTZ)
            out = self.out.device(AccessQualifier.WRITE_ONLY)
            W = self.E if os.environ.get("SK_C0_HEX_MODEMAJOR", "0") == "1" else 1
            _lib.check(
                lib.sk_helmholtz_apply_c0_w(self.basis.handle, _lib.SK_GEO_DEFORMED, self.nx, self.ny, self.nzl,
                                            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(pay.data_ptr()),
                                            float(lam), ctypes.c_void_p(out.data_ptr()), W, s),
                "sk_helmholtz_apply_c0_w",
            )
        else:
            local = self.block.device(AccessQualifier.WRITE_ONLY)
            _lib.check(
                lib.sk_c0_gather(self.P, self.nx, self.ny, self.nzl, ctypes.c_void_p(x.data_ptr()), 1,
                                 ctypes.c_void_p(local.data_ptr()), s),
                "sk_c0_gather",
            )
            helmholtz_apply(self.block, lam, out=self.out)
        y = torch.empty(self.n_dofs, dtype=torch.float64, device=x.device)
        loc = self.out.device(AccessQualifier.READ_ONLY)
        _lib.check(
            lib.sk_c0_scatter(self.P, self.nx, self.ny, self.nzl, ctypes.c_void_p(loc.data_ptr()), W,
                              ctypes.c_void_p(y.data_ptr()), s),
            "sk_c0_scatter",
        )
        exchange_interfaces(y, self.layer, group)
        return y

    def slab_slice(self) -> slice:
        """This slab's range in the global DOF vector."""
        start = self.z0 * self.P * self.layer
        return slice(start, start + self.n_dofs)


def _prism_tri_maps(nx: int, nw: int, P: int):
    """2D part of the prism C0 numbering on the triangulated nx x nw grid of
    unit squares (two triangles per square, lower (c00, c10, c01), upper
    (c11, c01, c10); prism local (xi1, xi3) span the triangle).  Returns the
    triangles' global vertex ids (NT, 3), their corner points (NT, 3, 2), the
    2D dof and sign of every triangle mode (p, r) as dicts of (NT,) arrays,
    and the 2D dof count.  Edge modes of degree k (V0V1: (k, 0), V1V2:
    (1, k-1), V0V2: (0, k)) trace psi_a(k) from the lower to the higher local
    vertex; against the global edge direction (lower -> higher global vertex
    id) odd degrees flip sign.  Edges are numbered by first appearance."""
    ix, iw = np.meshgrid(np.arange(nx), np.arange(nw), indexing="xy")
    ix, iw = ix.ravel(), iw.ravel()
    vid = lambda a, b: b * (nx + 1) + a  # noqa: E731
    low = np.stack([vid(ix, iw), vid(ix + 1, iw), vid(ix, iw + 1)], axis=1)
    up = np.stack([vid(ix + 1, iw + 1), vid(ix, iw + 1), vid(ix + 1, iw)], axis=1)
    tris = np.stack([low, up], axis=1).reshape(-1, 3)
    c = lambda a, b: np.stack([a, b], axis=-1).astype(float)  # noqa: E731
    pts = np.stack([np.stack([c(ix, iw), c(ix + 1, iw), c(ix, iw + 1)], axis=1),
                    np.stack([c(ix + 1, iw + 1), c(ix, iw + 1), c(ix + 1, iw)], axis=1)], axis=1).reshape(-1, 3, 2)
    nt, nv = tris.shape[0], (nx + 1) * (nw + 1)
    pairs = ((0, 1), (1, 2), (0, 2))
    a = np.stack([tris[:, i] for i, _ in pairs], axis=1)  # (NT, 3) local edge start vertex
    b = np.stack([tris[:, j] for _, j in pairs], axis=1)
    key = (np.minimum(a, b) * nv + np.maximum(a, b)).ravel()
    _, first, inv = np.unique(key, return_index=True, return_inverse=True)
    rank = np.empty_like(first)
    rank[np.argsort(first, kind="stable")] = np.arange(first.size)
    eid = rank[inv].reshape(nt, 3)
    fwd = a < b
    ni = (P - 1) * (P - 2) // 2
    base_e, base_i = nv, nv + first.size * (P - 1)
    dof, sgn = {}, {}
    for k, (p, r) in enumerate(((0, 0), (1, 0), (0, 1))):
        dof[(p, r)], sgn[(p, r)] = tris[:, k], np.ones(nt)
    for k in range(2, P + 1):
        for le, (p, r) in enumerate(((k, 0), (1, k - 1), (0, k))):
            dof[(p, r)] = base_e + eid[:, le] * (P - 1) + (k - 2)
            sgn[(p, r)] = np.where(fwd[:, le], 1.0, (-1.0) ** k)
    j = 0
    for p in range(2, P + 1):
        for r in range(1, P + 1 - p):
            dof[(p, r)], sgn[(p, r)] = base_i + np.arange(nt) * ni + j, np.ones(nt)
            j += 1
    return tris, pts, dof, sgn, base_i + nt * ni


class _MappedC0Mesh:
    """Assembled C0 slab applied through explicit maps: signed gather
    (sk_c0_gather_map) -> the elemental collocated Helmholtz of the shape ->
    deterministic CSR scatter (sk_c0_scatter_map) -> exchange of the two
    shared end layers / planes (``layer`` DOFs each) with the neighbouring
    ranks.  Subclasses build the maps and the quadrature coordinates."""

    def _setup(self, shape: Shape, l2g: np.ndarray, sgn, coords, either_orientation: bool) -> None:
        """l2g (E, NM) slab-relative global DOFs, sgn (E, NM) or None (all +1),
        coords (E, NQ, 3) CUDA tensor of quadrature-point coordinates."""
        import torch

        self.basis = build_shape_basis(shape, self.P)
        assert l2g.shape == (self.E, self.basis.n_modes)
        flat = l2g.reshape(-1)
        order_ = np.argsort(flat, kind="stable")
        ptr = np.zeros(self.n_dofs + 1, dtype=np.int64)
        np.cumsum(np.bincount(flat, minlength=self.n_dofs), out=ptr[1:])
        dev = coords.device
        self._l2g = torch.as_tensor(flat, device=dev)
        self._ptr = torch.as_tensor(ptr, device=dev)
        self._loc = torch.as_tensor(order_.astype(np.int64), device=dev)
        if sgn is None:
            self._sgn = self._csgn = torch.ones(flat.size, dtype=torch.float64, device=dev)
        else:
            sg = sgn.reshape(-1)
            self._sgn = torch.as_tensor(sg, device=dev)
            self._csgn = torch.as_tensor(sg[order_], device=dev)
        # compact int32 maps ((index << 1) | negative sign): a third of the map
        # traffic (sk_c0_gather_map32 / sk_c0_scatter_map32); the int64 / double
        # maps stay for meshes beyond their index range
        self._map32 = None
        nm = self.basis.n_modes
        if self.n_dofs < (1 << 30) and flat.size < (1 << 31) and os.environ.get("SK_C0_MAP32", "1") != "0":
            neg = np.zeros(flat.size, dtype=np.int64) if sgn is None else (sgn.reshape(-1) < 0).astype(np.int64)
            l2gs = ((flat.astype(np.int64) << 1) | neg).astype(np.int32)
            locs = ((order_.astype(np.int64) << 1) | neg[order_]).astype(np.int32)
            self._map32 = (torch.as_tensor(l2gs, device=dev), torch.as_tensor(ptr.astype(np.int32), device=dev),
                           torch.as_tensor(locs, device=dev))
        self.factors = deformed_factors_from_coords(self.basis, coords, either_orientation=either_orientation)
        self.block = Block(self.basis, self.factors, FieldState.COEFF, 1, 1)
        self.out = self.block.like(FieldState.COEFF)

    def slab_slice(self) -> slice:
        """This slab's range in the global DOF vector.  Level-ordered meshes
        (tet, pyramid): cube layers [z0, z0 + nzl) own every level from plane
        z0 to plane z0 + nzl, and every cube layer holds the same number of
        plane + between-level DOFs."""
        per_layer = (self.n_dofs - self.layer) // self.nzl
        start = self.z0 * per_layer
        return slice(start, start + self.n_dofs)

    def helmholtz(self, x, lam: float, group=None):
        """y = A^T H_e A x for this slab's DOF vector x (CUDA, length
        n_dofs); the shared end layers are summed across ranks."""
        import torch

        lib = _lib.load()
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        nm = self.basis.n_modes
        m32 = self._map32
        if m32 is not None and os.environ.get("SK_C0_FUSED", "1") != "0":
            # gather fused into the elemental kernel's tile load
            pay = self.block.payload(_lib.SK_PAYLOAD_HELMHOLTZ)
            dout = self.out.device(AccessQualifier.WRITE_ONLY)
            _lib.check(lib.sk_helmholtz_apply_c0_mapped(self.basis.handle, _lib.SK_GEO_DEFORMED, self.E, vp(m32[0]),
                                                        vp(x), vp(pay), float(lam), vp(dout), s),
                       "sk_helmholtz_apply_c0_mapped")
        else:
            local = self.block.device(AccessQualifier.WRITE_ONLY)
            if m32 is not None:
                _lib.check(lib.sk_c0_gather_map32(self.E, nm, vp(m32[0]), vp(x), 1, vp(local), s),
                           "sk_c0_gather_map32")
            else:
                _lib.check(lib.sk_c0_gather_map(self.E, nm, vp(self._l2g), vp(self._sgn), vp(x), 1, vp(local), s),
                           "sk_c0_gather_map")
            helmholtz_apply(self.block, lam, out=self.out)
        y = torch.empty(self.n_dofs, dtype=torch.float64, device=x.device)
        loc = self.out.device(AccessQualifier.READ_ONLY)
        if m32 is not None:
            _lib.check(lib.sk_c0_scatter_map32(self.n_dofs, nm, vp(m32[1]), vp(m32[2]), vp(loc), 1, vp(y), s),
                       "sk_c0_scatter_map32")
        else:
            _lib.check(lib.sk_c0_scatter_map(self.n_dofs, nm, vp(self._ptr), vp(self._loc), vp(self._csgn), vp(loc),
                                             1, vp(y), s), "sk_c0_scatter_map")
        exchange_interfaces(y, self.layer, group)
        return y


class C0PrismMesh(_MappedC0Mesh):
    """This rank's slab of a conforming prism mesh: the triangulated nx x nw
    grid of unit squares in the (x, z) plane extruded along y in nz element
    layers (the slab axis), deformed by the same smooth global map as
    C0HexMesh.  y = A^T H_e A x with signed maps: sk_c0_gather_map -> the
    elemental collocated Helmholtz (prism kernels) -> sk_c0_scatter_map
    (a deterministic per-DOF gather over a CSR list), then the exchange of
    the two shared DOF layers with the neighbouring ranks.  Parity:
    oracle/assembly.py (prism section), whose map is checked for
    conformity on CPU."""

    def __init__(self, nx: int, nw: int, nz: int, order: int, amp: float = 0.05, rank: int = 0, world: int = 1):
        import torch

        if nz < world:
            raise ValueError(f"need at least one element layer per rank: nz={nz} < world={world}")
        P = order
        self.nx, self.nw, self.nz, self.P, self.amp = nx, nw, nz, P, amp
        self.z0, self.nzl = partition(nz, world, rank)
        tris, pts, dof2, sgn2, n2d = _prism_tri_maps(nx, nw, P)
        nt = tris.shape[0]
        self.layer = n2d  # DOFs of one extrusion node (the exchanged interface)
        self.n_dofs = n2d * (self.nzl * P + 1)
        self.E = self.nzl * nt
        modes = build_shape_basis(Shape.PRISM, P).modes
        nm = len(modes)
        pm = np.array([0 if q == 0 else P if q == 1 else q - 1 for q in range(P + 1)])
        ez = np.arange(self.nzl)
        l2g = np.empty((self.nzl, nt, nm), dtype=np.int64)
        sgn = np.empty((self.nzl, nt, nm))
        for m, (p, q, r) in enumerate(modes):
            l2g[:, :, m] = (ez[:, None] * P + pm[q]) * n2d + dof2[(p, r)][None, :]
            sgn[:, :, m] = sgn2[(p, r)][None, :]
        # quadrature coordinates: barycentrics of the triangle in (x, z),
        # y = layer + (1 + xi2) / 2, then the global deformation
        dev = torch.device("cuda", torch.cuda.current_device())
        xi = torch.as_tensor(quadrature_coords(build_shape_basis(Shape.PRISM, P)), device=dev)
        l1, l2 = 0.5 * (1.0 + xi[:, 0]), 0.5 * (1.0 + xi[:, 2])
        lw = torch.stack([1.0 - l1 - l2, l1, l2], dim=1)  # (NQ, 3)
        xz = torch.einsum("qk,tkc->tqc", lw, torch.as_tensor(pts, device=dev))  # (NT, NQ, 2)
        X = torch.empty((self.nzl, nt, xi.shape[0], 3), dtype=torch.float64, device=dev)
        X[..., 0] = xz[None, ..., 0]
        X[..., 2] = xz[None, ..., 1]
        X[..., 1] = (self.z0 + torch.arange(self.nzl, device=dev, dtype=torch.float64))[:, None, None] \
            + 0.5 * (1.0 + xi[None, None, :, 1])
        X = X.reshape(self.E, xi.shape[0], 3)
        self._setup(Shape.PRISM, l2g.reshape(self.E, nm), sgn.reshape(self.E, nm),
                    X + amp * torch.sin(0.5 * np.pi * X[..., [1, 2, 0]]), either_orientation=False)

    def slab_slice(self) -> slice:
        """This slab's range in the global DOF vector."""
        start = self.z0 * self.P * self.layer
        return slice(start, start + self.n_dofs)


_KUHN = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_TET_EDGES = ((0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (2, 3))
_TET_FACES = ((0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3))


def _tet_mode_table(P: int):
    """Entity of every local tet mode (p, q, r) (shapes.py:374-405 modes):
    (kind, local index, sub-index) with kind 0 vertex (index into the 4
    vertices), 1 edge (into _TET_EDGES; sub-index degree - 2), 2 face (into
    _TET_FACES; sub-index of the face's canonical (a, b) mode, a >= 2,
    b >= 1), 3 interior.  Edge / face modes trace psi_a along the edge from
    the lower vertex, psi_a(a) psi_b(a, b) on the face collapsed towards its
    highest vertex, so elements whose vertices are in global-id order agree
    on every shared entity."""
    face_ab = {ab: i for i, ab in enumerate((a, b) for a in range(2, P + 1) for b in range(1, P + 1 - a))}
    out, ni = [], 0
    for p in range(P + 1):
        for q in range(P + 1 - p):
            for r in range(P + 1 - p - q):
                verts = {(0, 0, 0): 0, (1, 0, 0): 1, (0, 1, 0): 2, (0, 0, 1): 3}
                if (p, q, r) in verts:
                    out.append((0, verts[(p, q, r)], 0))
                elif q == 0 and r == 0:
                    out.append((1, 0, p - 2))
                elif p == 0 and r == 0:
                    out.append((1, 1, q - 2))
                elif p == 1 and r == 0:
                    out.append((1, 2, q - 1))
                elif p == 0 and q == 0:
                    out.append((1, 3, r - 2))
                elif p == 1 and q == 0:
                    out.append((1, 4, r - 1))
                elif p == 0 and q == 1:
                    out.append((1, 5, r - 1))
                elif r == 0:
                    out.append((2, 0, face_ab[(p, q)]))
                elif q == 0:
                    out.append((2, 1, face_ab[(p, r)]))
                elif p == 0:
                    out.append((2, 2, face_ab[(q, r)]))
                elif p == 1:
                    out.append((2, 3, face_ab[(q + 1, r)]))
                else:
                    out.append((3, 0, ni))
                    ni += 1
    return out, len(face_ab), ni


def _tet_maps(nx: int, ny: int, nz: int, z0: int, nzl: int, P: int):
    """Numbering of the C0 tet mesh slab of cube layers [z0, z0 + nzl) (see
    C0TetMesh): vertex coordinates (E, 4, 3) of its Kuhn tets, the
    slab-relative global dof of every (tet, local mode), the slab's dof
    count and the dofs of one z plane."""
    nxy = (nx + 1) * (ny + 1)
    nv = nxy * (nz + 1)
    # Kuhn tets of the slab (cubes x fastest, then y, then z), vertices
    # ascending = the path along the cube's main diagonal
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), z0 + np.arange(nzl), indexing="ij")
    base = np.stack([ix.T.ravel(), iy.T.ravel(), iz.T.ravel()], axis=1)  # (cubes, 3)
    steps = np.eye(3, dtype=np.int64)
    corners = []
    for perm in _KUHN:
        path = [np.zeros(3, dtype=np.int64)]
        for ax in perm:
            path.append(path[-1] + steps[ax])
        corners.append(np.stack(path))
    pts = (base[:, None, None, :] + np.stack(corners)[None]).reshape(-1, 4, 3)
    verts = (pts[..., 2] * (ny + 1) + pts[..., 1]) * (nx + 1) + pts[..., 0]
    E = verts.shape[0]
    # every entity occurrence as (level, kind, key): level 2z for entities in
    # the plane z, 2z+1 between z and z+1; key = sorted vertex ids
    recs = []
    for kind, subs in ((0, ((0,), (1,), (2,), (3,))), (1, _TET_EDGES), (2, _TET_FACES)):
        arr = np.stack([verts[:, list(sub)] for sub in subs], axis=1)  # (E, n, k)
        z = arr // nxy
        lev = 2 * z.min(axis=-1) + (z.min(axis=-1) != z.max(axis=-1))
        key = np.zeros(arr.shape[:2], dtype=np.int64)
        for c in range(arr.shape[-1]):
            key = key * nv + arr[..., c]
        recs.append((lev, np.full(arr.shape[:2], kind), key))
    cz = verts[:, 0] // nxy  # cube layer of each tet: its interior modes
    recs.append(((2 * cz + 1)[:, None], np.full((E, 1), 3), np.arange(E, dtype=np.int64)[:, None]))
    lev = np.concatenate([r[0].ravel() for r in recs])
    kind = np.concatenate([r[1].ravel() for r in recs])
    key = np.concatenate([r[2].ravel() for r in recs])
    order_ = np.lexsort((key, kind, lev))
    srt = np.stack([lev[order_], kind[order_], key[order_]], axis=1)
    new = np.ones(len(srt), dtype=bool)
    new[1:] = np.any(srt[1:] != srt[:-1], axis=1)
    uid = np.empty(len(srt), dtype=np.int64)
    uid[order_] = np.cumsum(new) - 1
    modes, nf, ni = _tet_mode_table(P)
    usize = np.array([1, P - 1, nf, ni])[srt[new, 1]]
    uoff = np.concatenate([[0], np.cumsum(usize)[:-1]])
    n_dofs = int(usize.sum())
    layer = nxy + (nx * (ny + 1) + (nx + 1) * ny + nx * ny) * (P - 1) + 2 * nx * ny * nf  # one z plane
    cut = np.cumsum([0, E * 4, E * 6, E * 4, E])
    ent = [uid[cut[k]:cut[k + 1]].reshape(E, -1) for k in range(4)]
    l2g = np.empty((E, len(modes)), dtype=np.int64)
    for m, (k, li, sub) in enumerate(modes):
        l2g[:, m] = uoff[ent[k][:, li]] + sub
    return pts, l2g, n_dofs, layer


class C0TetMesh(_MappedC0Mesh):
    """This rank's slab of a conforming tet mesh: nx x ny x nz unit cubes,
    each split into the six Kuhn tets along its main diagonal, every tet
    taking its vertices in global-id order (so shared edges and faces are
    parameterised alike on both sides; the reflected half gets w|det J|,
    sk_geometry_from_coords_oriented), deformed by the global map of
    C0HexMesh.  Global DOFs are ordered by geometric level (plane z, the
    entities between z and z+1, ...; within a level vertices, edges, faces
    by sorted global vertex ids, then the tets' interior modes), so a slab of
    cube layers is one contiguous range whose end planes are shared with the
    neighbouring ranks.  y = A^T H_e A x by sk_c0_gather_map -> the tet
    kernels -> sk_c0_scatter_map, then the plane exchange.  Parity:
    oracle/assembly.py (tet section, conformity-checked on CPU)."""

    def __init__(self, nx: int, ny: int, nz: int, order: int, amp: float = 0.05, rank: int = 0, world: int = 1):
        import torch

        if nz < world:
            raise ValueError(f"need at least one element layer per rank: nz={nz} < world={world}")
        P = order
        self.nx, self.ny, self.nz, self.P, self.amp = nx, ny, nz, P, amp
        self.z0, self.nzl = partition(nz, world, rank)
        pts, l2g, self.n_dofs, self.layer = _tet_maps(nx, ny, nz, self.z0, self.nzl, P)
        self.E = pts.shape[0]
        # quadrature coordinates: affine image of the reference tet, then the
        # global deformation
        dev = torch.device("cuda", torch.cuda.current_device())
        xi = torch.as_tensor(quadrature_coords(build_shape_basis(Shape.TET, P)), device=dev)
        lam = 0.5 * (1.0 + xi)  # (NQ, 3)
        v = torch.as_tensor(pts, dtype=torch.float64, device=dev)  # (E, 4, 3)
        X = v[:, None, 0, :] + torch.einsum("qk,ekc->eqc", lam, v[:, 1:, :] - v[:, :1, :])
        self._setup(Shape.TET, l2g, None, X + amp * torch.sin(0.5 * np.pi * X[..., [1, 2, 0]]),
                    either_orientation=True)



_PYR_FACES = ((0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1))  # (normal axis, side) of the base
_PYR_EDGES = ((0, 1), (3, 2), (0, 3), (1, 2), (0, 4), (1, 4), (2, 4), (3, 4))
_PYR_TRIS = ((0, 1, 4), (3, 2, 4), (0, 3, 4), (1, 2, 4))


def _pyr_mode_table(P: int):
    """Entity of every local pyramid mode (p, q, r) (shapes.py:374-405):
    (kind, local index, sub-index); kinds 0 vertex, 1 edge (_PYR_EDGES,
    sub-index degree - 2), 2 base quad (canonical (p, q)), 3 triangular face
    (_PYR_TRIS, canonical (a, b): psi_a(a) along the base edge, psi_b(a, b)
    towards the apex), 4 interior."""
    tri = {ab: i for i, ab in enumerate((a, b) for a in range(2, P + 1) for b in range(1, P + 1 - a))}
    quad = {pq: i for i, pq in enumerate((p, q) for p in range(2, P + 1) for q in range(2, P + 1))}
    vert = {(0, 0, 0): 0, (1, 0, 0): 1, (1, 1, 0): 2, (0, 1, 0): 3, (0, 0, 1): 4}
    corner = {(0, 0): 0, (1, 0): 1, (1, 1): 2, (0, 1): 3}
    out, ni = [], 0
    for p in range(P + 1):
        for q in range(P + 1):
            for r in range(P + 1 - max(p, q)):
                if (p, q, r) in vert:
                    out.append((0, vert[(p, q, r)], 0))
                elif r == 0 and q <= 1 and p >= 2:
                    out.append((1, q, p - 2))  # edges V0V1 / V3V2
                elif r == 0 and p <= 1 and q >= 2:
                    out.append((1, 2 + p, q - 2))  # edges V0V3 / V1V2
                elif r == 0:
                    out.append((2, 0, quad[(p, q)]))
                elif p <= 1 and q <= 1:
                    c = corner[(p, q)]
                    out.append((1, 4 + c, r - 2 if c == 0 else r - 1))  # apex edges
                elif q <= 1:
                    out.append((3, q, tri[(p, r)]))
                elif p <= 1:
                    out.append((3, 2 + p, tri[(q, r)]))
                else:
                    out.append((4, 0, ni))
                    ni += 1
    return out, len(quad), len(tri), ni


def _pyr_maps(nx: int, ny: int, nz: int, z0: int, nzl: int, P: int):
    """Numbering of the C0 pyramid mesh slab of cube layers [z0, z0 + nzl)
    (see C0PyrMesh): vertex coordinates (E, 5, 3), the slab-relative global
    dof of every (pyramid, local mode), the slab's dof count and the dofs of
    one z plane."""
    nc = (nx + 1) * (ny + 1) * (nz + 1)
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), z0 + np.arange(nzl), indexing="ij")
    base = np.stack([ix.T.ravel(), iy.T.ravel(), iz.T.ravel()], axis=1)  # (cubes, 3), x fastest
    cube = (base[:, 2] * ny + base[:, 1]) * nx + base[:, 0]
    eye = np.eye(3, dtype=np.int64)
    quads = []
    for n, side in _PYR_FACES:
        a, b = [ax for ax in range(3) if ax != n]
        v0 = side * eye[n]
        quads.append(np.stack([v0, v0 + eye[a], v0 + eye[a] + eye[b], v0 + eye[b]]))
    quads = np.stack(quads)  # (6, 4, 3)
    corners = base[:, None, None, :] + quads[None]  # (cubes, 6, 4, 3)
    ncube = base.shape[0]
    pts = np.empty((ncube, 6, 5, 3))
    pts[:, :, :4] = corners
    pts[:, :, 4] = base[:, None, :] + 0.5
    pts = pts.reshape(-1, 5, 3)
    cid = (corners[..., 2] * (ny + 1) + corners[..., 1]) * (nx + 1) + corners[..., 0]
    verts = np.concatenate([cid, np.broadcast_to((nc + cube)[:, None, None], (ncube, 6, 1))], axis=2).reshape(-1, 5)
    z2 = np.concatenate([2 * corners[..., 2], np.broadcast_to((2 * base[:, 2] + 1)[:, None, None], (ncube, 6, 1))],
                        axis=2).reshape(-1, 5)
    E = verts.shape[0]
    nkey = nc + nx * ny * nz
    recs = []
    for kind, subs in ((0, tuple((i,) for i in range(5))), (1, _PYR_EDGES), (2, ((0, 1, 2, 3),)), (3, _PYR_TRIS)):
        arr = np.stack([verts[:, list(s)] for s in subs], axis=1)  # (E, n, k)
        zz = np.stack([z2[:, list(s)] for s in subs], axis=1)
        zmin, zmax = zz.min(axis=-1), zz.max(axis=-1)
        lev = np.where((zmin == zmax) & (zmin % 2 == 0), zmin, 2 * (zmin // 2) + 1)
        arr = np.sort(arr, axis=-1)
        key = np.zeros(arr.shape[:2], dtype=np.int64)
        for c in range(arr.shape[-1]):
            key = key * nkey + arr[..., c]
        recs.append((lev, np.full(arr.shape[:2], kind), key))
    recs.append(((2 * np.repeat(base[:, 2], 6) + 1)[:, None], np.full((E, 1), 4), np.arange(E, dtype=np.int64)[:, None]))
    lev = np.concatenate([r[0].ravel() for r in recs])
    kind = np.concatenate([r[1].ravel() for r in recs])
    key = np.concatenate([r[2].ravel() for r in recs])
    order_ = np.lexsort((key, kind, lev))
    srt = np.stack([lev[order_], kind[order_], key[order_]], axis=1)
    new = np.ones(len(srt), dtype=bool)
    new[1:] = np.any(srt[1:] != srt[:-1], axis=1)
    uid = np.empty(len(srt), dtype=np.int64)
    uid[order_] = np.cumsum(new) - 1
    modes, nq, nt, ni = _pyr_mode_table(P)
    usize = np.array([1, P - 1, nq, nt, ni])[srt[new, 1]]
    uoff = np.concatenate([[0], np.cumsum(usize)[:-1]])
    n_dofs = int(usize.sum())
    layer = (nx + 1) * (ny + 1) + (nx * (ny + 1) + (nx + 1) * ny) * (P - 1) + nx * ny * nq  # one z plane
    cut = np.cumsum([0, E * 5, E * 8, E, E * 4, E])
    ent = [uid[cut[k]:cut[k + 1]].reshape(E, -1) for k in range(5)]
    l2g = np.empty((E, len(modes)), dtype=np.int64)
    for m, (k, li, sub) in enumerate(modes):
        l2g[:, m] = uoff[ent[k][:, li]] + sub
    return pts, l2g, n_dofs, layer


class C0PyrMesh(_MappedC0Mesh):
    """This rank's slab of a conforming pyramid mesh: nx x ny x nz unit
    cubes, each split into six pyramids (apex = the cube centre, base = a
    cube face), each base's (eta1, eta2) along the face's two global axes in
    increasing direction from its minimum corner -- so shared base quads,
    triangular faces and edges are parameterised alike on both sides with no
    signs (the reflected half gets w|det J|) -- deformed by the global map
    of C0HexMesh, level-ordered DOFs as C0TetMesh.  y = A^T H_e A x by
    sk_c0_gather_map -> the pyramid kernels -> sk_c0_scatter_map, then the
    plane exchange.  Parity: oracle/assembly.py (pyramid section,
    conformity-checked on CPU)."""

    def __init__(self, nx: int, ny: int, nz: int, order: int, amp: float = 0.05, rank: int = 0, world: int = 1):
        import torch

        if nz < world:
            raise ValueError(f"need at least one element layer per rank: nz={nz} < world={world}")
        P = order
        self.nx, self.ny, self.nz, self.P, self.amp = nx, ny, nz, P, amp
        self.z0, self.nzl = partition(nz, world, rank)
        pts, l2g, self.n_dofs, self.layer = _pyr_maps(nx, ny, nz, self.z0, self.nzl, P)
        self.E = pts.shape[0]
        # affine image of the reference pyramid (apex at xi = (-1,-1,1)):
        # x = V0 + l1 (V1 - V0) + l2 (V3 - V0) + l3 (V4 - V0), l = (1 + xi) / 2
        dev = torch.device("cuda", torch.cuda.current_device())
        xi = torch.as_tensor(quadrature_coords(build_shape_basis(Shape.PYR, P)), device=dev)
        lam = 0.5 * (1.0 + xi)
        v = torch.as_tensor(pts, dtype=torch.float64, device=dev)  # (E, 5, 3)
        axes = torch.stack([v[:, 1] - v[:, 0], v[:, 3] - v[:, 0], v[:, 4] - v[:, 0]], dim=1)  # (E, 3, 3)
        X = v[:, None, 0, :] + torch.einsum("qk,ekc->eqc", lam, axes)
        self._setup(Shape.PYR, l2g, None, X + amp * torch.sin(0.5 * np.pi * X[..., [1, 2, 0]]),
                    either_orientation=True)
