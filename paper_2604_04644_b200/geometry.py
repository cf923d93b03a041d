"""Geometric factors: affine (Regular) and curvilinear (Deformed) elements.

Mirrors the reference ``speckern.geometry`` API (geometry.py:35-315).  The
iso-parametric metric of deformed elements (collocation derivative of the
coordinates, Duffy chain rule, pointwise det/inverse; geometry.py:161-212) is
computed on the device by the C library (``sk_geometry_*``); synthetic
deformed meshes are kept as their per-element deformation parameters and the
operator payloads are generated straight from them on the device
(``sk_payload_from_params``), so a 10^6-element block never materialises
its 10 doubles per quadrature point of factors unless asked to.
"""

from __future__ import annotations

import ctypes
import enum
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from paper_2604_04644_b200 import _lib
from paper_2604_04644_b200.shapes import Shape, ShapeBasis

__all__ = [
    "GeometryClass",
    "GeometricFactors",
    "DegenerateElementError",
    "REFERENCE_VERTICES",
    "make_affine_block",
    "make_deformed_block",
    "deformed_factors_from_coords",
    "synthetic_affine_vertices",
    "synthetic_deformation_params",
    "make_synthetic_factors",
    "quadrature_coords",
]


class GeometryClass(enum.Enum):
    REGULAR = "regular"
    DEFORMED = "deformed"


class DegenerateElementError(ValueError):
    """Nonpositive Jacobian (geometry.py:42-43)."""


REFERENCE_VERTICES = {
    Shape.HEX: np.array(
        [[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]],
        dtype=float,
    ),
    Shape.PRISM: np.array(
        [[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1], [-1, 1, 1]], dtype=float
    ),
    Shape.PYR: np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float),
    Shape.TET: np.array([[-1, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float),
}
_EDGE_VERTICES = {Shape.HEX: (1, 3, 4), Shape.PRISM: (1, 3, 4), Shape.PYR: (1, 3, 4), Shape.TET: (1, 2, 3)}


def _torch():
    import torch

    return torch


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


class GeometricFactors:
    """Metric data of one homogeneous group of elements (geometry.py:94-116).

    ``dxi_dx[..., i, j] = d xi_i / d x_j``: (E, 3, 3) regular, (E, NQ, 3, 3)
    deformed; ``jac``: |J| (E,) regular, w|J| (E, NQ) deformed.  Deformed
    factors may be held lazily as deformation parameters (``params``, E x 12)
    and materialised on demand.  Device payloads are cached per (basis
    shape, order, point counts, kind, device) and are independent of the
    block's interleave width.
    """

    def __init__(
        self,
        geometry_class: GeometryClass,
        shape: Shape,
        n_elements: int,
        dxi_dx=None,
        jac=None,
        params: np.ndarray | None = None,
        basis: ShapeBasis | None = None,
    ):
        self.geometry_class = geometry_class
        self.shape = shape
        self.n_elements = int(n_elements)
        self._dxi = dxi_dx
        self._jac = jac
        self.params = params
        self.basis = basis
        self._payloads: dict = {}
        if params is None and (dxi_dx is None or jac is None):
            raise ValueError("need either (dxi_dx, jac) or deformation params")
        if params is not None and basis is None:
            raise ValueError("lazy deformed factors need their basis")

    @property
    def deformed(self) -> bool:
        return self.geometry_class is GeometryClass.DEFORMED

    def _materialise(self):
        torch = _torch()
        b = self.basis
        dev = torch.device("cuda", torch.cuda.current_device())
        E, nq = self.n_elements, b.n_points
        prm = torch.as_tensor(self.params, dtype=torch.float64, device=dev)
        dxi = torch.empty((E, nq, 3, 3), dtype=torch.float64, device=dev)
        jac = torch.empty((E, nq), dtype=torch.float64, device=dev)
        bad = ctypes.c_int64()
        _lib.check(
            _lib.load().sk_geometry_deformed(b.handle, E, _ptr(prm), _ptr(dxi), _ptr(jac), ctypes.byref(bad), _stream()),
            "sk_geometry_deformed",
        )
        if bad.value:
            raise DegenerateElementError(f"{bad.value} quadrature points with nonpositive Jacobian")
        self._dxi, self._jac = dxi, jac

    @property
    def dxi_dx(self) -> np.ndarray:
        if self._dxi is None:
            self._materialise()
        d = self._dxi
        return d if isinstance(d, np.ndarray) else d.cpu().numpy()

    @property
    def jac(self) -> np.ndarray:
        if self._jac is None:
            self._materialise()
        j = self._jac
        return j if isinstance(j, np.ndarray) else j.cpu().numpy()

    def device_params(self, device):
        """Deformation parameters (E x 12, as doubles) on ``device``, cached:
        the input of the recomputed-metric Helmholtz variant."""
        torch = _torch()
        key = ("params", str(device))
        if key not in self._payloads:
            self._payloads[key] = torch.as_tensor(self.params, dtype=torch.float64, device=device).contiguous()
        return self._payloads[key]

    def payload(self, basis: ShapeBasis, kind: int):
        """Device payload for operator family ``kind`` (built once, cached):
        replaces Block.payload (field_block.py:309-363)."""
        torch = _torch()
        dev = torch.cuda.current_device()
        # the payload layout (lane width, point count) depends on the basis:
        # one regular GeometricFactors may serve bases of several orders
        key = (basis.shape, basis.order, basis.qcounts, kind, dev)
        if key in self._payloads:
            return self._payloads[key]
        lib = _lib.load()
        geo = _lib.SK_GEO_DEFORMED if self.deformed else _lib.SK_GEO_REGULAR
        n = ctypes.c_int64()
        _lib.check(lib.sk_payload_size(basis.handle, geo, kind, self.n_elements, ctypes.byref(n)), "sk_payload_size")
        pay = torch.empty(max(n.value, 1), dtype=torch.float64, device=torch.device("cuda", dev))
        if self.n_elements == 0:
            self._payloads[key] = pay
            return pay
        if self.params is not None and self._dxi is None:
            prm = torch.as_tensor(self.params, dtype=torch.float64, device=pay.device)
            bad = ctypes.c_int64()
            _lib.check(
                lib.sk_payload_from_params(basis.handle, kind, self.n_elements, _ptr(prm), _ptr(pay), ctypes.byref(bad), _stream()),
                "sk_payload_from_params",
            )
            if bad.value:
                raise DegenerateElementError(f"{bad.value} quadrature points with nonpositive Jacobian")
        else:
            dxi = torch.as_tensor(self._dxi, dtype=torch.float64).to(pay.device).contiguous()
            jac = torch.as_tensor(self._jac, dtype=torch.float64).to(pay.device).contiguous()
            _lib.check(
                lib.sk_payload_pack(basis.handle, geo, kind, self.n_elements, _ptr(dxi), _ptr(jac), _ptr(pay), _stream()),
                "sk_payload_pack",
            )
        self._payloads[key] = pay
        return pay

    def drop_payloads(self) -> None:
        self._payloads.clear()


def make_affine_block(shape: Shape, vertices) -> GeometricFactors:
    """Constant metric of straight-sided elements (geometry.py:119-158)."""
    verts = np.asarray(vertices, dtype=float)
    if verts.ndim == 2:
        verts = verts[None]
    nv = REFERENCE_VERTICES[shape].shape[0]
    if verts.shape[1:] != (nv, 3):
        raise ValueError(f"{shape.value} expects vertex array (n_elements, {nv}, 3), got {verts.shape}")
    edges = np.stack([verts[:, k, :] - verts[:, 0, :] for k in _EDGE_VERTICES[shape]], axis=-1)
    jm = 0.5 * edges
    det = np.linalg.det(jm)
    if np.any(det <= 0.0):
        bad = int(np.argmax(det <= 0.0))
        raise DegenerateElementError(f"element {bad} has nonpositive Jacobian {det[bad]:.3e}")
    return GeometricFactors(GeometryClass.REGULAR, shape, verts.shape[0], np.linalg.inv(jm), det)


def quadrature_coords(basis: ShapeBasis) -> np.ndarray:
    """Standard-region coordinates of the tensor points (geometry.py:234-238)."""
    e = np.stack([g.ravel() for g in np.meshgrid(*basis.eta, indexing="ij")], axis=-1)
    xi = e.copy()
    s = basis.shape
    if s is Shape.PRISM:
        xi[:, 0] = 0.5 * (1.0 + e[:, 0]) * (1.0 - e[:, 2]) - 1.0
    elif s is Shape.PYR:
        xi[:, 0] = 0.5 * (1.0 + e[:, 0]) * (1.0 - e[:, 2]) - 1.0
        xi[:, 1] = 0.5 * (1.0 + e[:, 1]) * (1.0 - e[:, 2]) - 1.0
    elif s is Shape.TET:
        xi[:, 1] = 0.5 * (1.0 + e[:, 1]) * (1.0 - e[:, 2]) - 1.0
        xi[:, 0] = 0.25 * (1.0 + e[:, 0]) * (1.0 - e[:, 1]) * (1.0 - e[:, 2]) - 1.0
    return xi


def deformed_factors_from_coords(basis: ShapeBasis, coords, either_orientation: bool = False) -> GeometricFactors:
    """Per-point factors from coordinates (E, NQ, 3) on the device
    (geometry.py:161-212).  ``either_orientation``: accept reflected
    elements with w|det J| (the assembled tet mesh; the reference rejects
    det J <= 0)."""
    torch = _torch()
    c = torch.as_tensor(np.asarray(coords, dtype=float) if not hasattr(coords, "data_ptr") else coords)
    if c.dim() == 2:
        c = c[None]
    if tuple(c.shape[1:]) != (basis.n_points, 3):
        raise ValueError(f"expected coords (n_elements, {basis.n_points}, 3), got {tuple(c.shape)}")
    dev = torch.device("cuda", torch.cuda.current_device())
    c = c.to(device=dev, dtype=torch.float64).contiguous()
    E = c.shape[0]
    dxi = torch.empty((E, basis.n_points, 3, 3), dtype=torch.float64, device=dev)
    jac = torch.empty((E, basis.n_points), dtype=torch.float64, device=dev)
    bad = ctypes.c_int64()
    fn = _lib.load().sk_geometry_from_coords_oriented if either_orientation else _lib.load().sk_geometry_from_coords
    _lib.check(fn(basis.handle, E, _ptr(c), _ptr(dxi), _ptr(jac), ctypes.byref(bad), _stream()), "sk_geometry_from_coords")
    if bad.value:
        raise DegenerateElementError(f"{bad.value} quadrature points with nonpositive Jacobian")
    return GeometricFactors(GeometryClass.DEFORMED, basis.shape, E, dxi, jac)


def make_deformed_block(basis: ShapeBasis, mapping, n_elements: int = 1) -> GeometricFactors:
    """geometry.py:215-231: ``mapping(xi)`` or ``mapping(xi, e)`` on the host,
    metric on the device."""
    xi = quadrature_coords(basis)
    if n_elements == 1:
        coords = np.asarray(mapping(xi), dtype=float)[None]
    else:
        coords = np.stack([np.asarray(mapping(xi, e), dtype=float) for e in range(n_elements)])
    return deformed_factors_from_coords(basis, coords)


# ---------------------------------------------------------------------------
# seeded synthetic meshes (geometry.py:256-315): element e depends only on
# (seed, e), so any sub-range can be generated independently


def _affine_chunk(args):
    shape, first, n, seed, jitter = args
    ref = REFERENCE_VERTICES[shape]
    out = np.empty((n, ref.shape[0], 3))
    for i in range(n):
        rng = np.random.default_rng(seed * 1_000_003 + first + i)
        mat = np.eye(3) + jitter * (rng.random((3, 3)) - 0.5)
        if np.linalg.det(mat) <= 0.0:
            mat[:, 0] = -mat[:, 0]
        out[i] = ref @ mat.T + rng.random(3)
    return out


def _deform_chunk(args):
    first, n, seed, amplitude = args
    out = np.empty((n, 12))
    for i in range(n):
        rng = np.random.default_rng(seed * 9_999_991 + 7 * (first + i) + 1)
        out[i, 0:3] = amplitude * (0.5 + 0.5 * rng.random(3))
        out[i, 3:6] = 2.0 * np.pi * rng.random(3)
        out[i, 6:9] = rng.permutation(3)
        out[i, 9:12] = rng.random(3)
    return out


def _chunked(fn, make_args, n: int, workers: int | None):
    chunk = 16384
    if n <= 2 * chunk:
        return fn(make_args(0, n))
    workers = workers or min(32, os.cpu_count() or 1)
    starts = list(range(0, n, chunk))
    jobs = [make_args(s, min(chunk, n - s)) for s in starts]
    import multiprocessing as mp

    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
        return np.concatenate(list(ex.map(fn, jobs)))


def synthetic_affine_vertices(shape: Shape, n_elements: int, seed: int = 0, jitter: float = 0.15, first: int = 0,
                              workers: int | None = None) -> np.ndarray:
    """geometry.py:256-272 (elements first .. first+n-1)."""
    return _chunked(_affine_chunk, lambda s, n: (shape, first + s, n, seed, jitter), n_elements, workers)


def synthetic_deformation_params(n_elements: int, seed: int = 0, amplitude: float = 0.05, first: int = 0,
                                 workers: int | None = None) -> np.ndarray:
    """Per-element draws of synthetic_deformation (geometry.py:275-300):
    rows amp[3], phase[3], perm[3], shift[3]."""
    amplitude = min(amplitude, 0.1)
    return _chunked(_deform_chunk, lambda s, n: (first + s, n, seed, amplitude), n_elements, workers)


def make_synthetic_factors(basis: ShapeBasis, geometry_class: GeometryClass, n_elements: int, seed: int = 0,
                           amplitude: float = 0.05, first: int = 0) -> GeometricFactors:
    """geometry.py:303-315; ``first`` selects a contiguous element range of the
    same seeded mesh (used to shard a block across GPUs)."""
    if geometry_class is GeometryClass.REGULAR:
        return make_affine_block(basis.shape, synthetic_affine_vertices(basis.shape, n_elements, seed, first=first))
    params = synthetic_deformation_params(n_elements, seed, amplitude, first=first)
    return GeometricFactors(GeometryClass.DEFORMED, basis.shape, n_elements, params=params, basis=basis)
