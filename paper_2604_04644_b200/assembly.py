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

import numpy as np

from paper_2604_04644_b200 import _lib
from paper_2604_04644_b200.field_block import AccessQualifier, Block, FieldState
from paper_2604_04644_b200.geometry import deformed_factors_from_coords, quadrature_coords
from paper_2604_04644_b200.operators import helmholtz_apply
from paper_2604_04644_b200.sharding import partition
from paper_2604_04644_b200.shapes import Shape, build_shape_basis

__all__ = ["C0HexMesh", "exchange_interfaces"]


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
        if lam > 0.0:
            # gather fused into the Helmholtz tile load (no A x round trip through HBM)
            pay = self.block.payload(_lib.SK_PAYLOAD_HELMHOLTZ)
            out = self.out.device(AccessQualifier.WRITE_ONLY)
            _lib.check(
                lib.sk_helmholtz_apply_c0(self.basis.handle, _lib.SK_GEO_DEFORMED, self.nx, self.ny, self.nzl,
                                          ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(pay.data_ptr()),
                                          float(lam), ctypes.c_void_p(out.data_ptr()), s),
                "sk_helmholtz_apply_c0",
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
            lib.sk_c0_scatter(self.P, self.nx, self.ny, self.nzl, ctypes.c_void_p(loc.data_ptr()), 1,
                              ctypes.c_void_p(y.data_ptr()), s),
            "sk_c0_scatter",
        )
        exchange_interfaces(y, self.layer, group)
        return y

    def slab_slice(self) -> slice:
        """This slab's range in the global DOF vector."""
        start = self.z0 * self.P * self.layer
        return slice(start, start + self.n_dofs)
