"""Element shapes and the per-(shape, order) basis bundle.

Mirrors the reference ``speckern.shapes`` API (shapes.py:57-179, 412-541) for
the device path.  The constant tables are built natively by the C library
(``sk_basis_create``, csrc/basis_host.cpp) and exposed here read-only for
host-side users (geometry builders, tests).
"""

from __future__ import annotations

import ctypes
import enum
from functools import lru_cache

import numpy as np

from paper_2604_04644_b200 import _lib

__all__ = [
    "Shape",
    "ShapeBasis",
    "mode_count",
    "quad_point_counts",
    "index_set",
    "build_shape_basis",
    "DEVICE_SHAPES",
]


class Shape(enum.Enum):
    """Same members and order as the reference enum (shapes.py:57-65); the
    enum index is the ABI shape id and part of the bench seed key."""

    QUAD = "quad"
    TRI = "tri"
    HEX = "hex"
    PRISM = "prism"
    PYR = "pyr"
    TET = "tet"

    @property
    def ndim(self) -> int:
        return 2 if self in (Shape.QUAD, Shape.TRI) else 3

    @property
    def abi_id(self) -> int:
        return list(Shape).index(self)


#: the shapes the device path implements (north star: 3D mixed meshes)
DEVICE_SHAPES = (Shape.HEX, Shape.PRISM, Shape.PYR, Shape.TET)


def mode_count(shape: Shape, order: int) -> int:
    """shapes.py:112-129."""
    if order < 1:
        raise ValueError(f"polynomial order must be at least 1, got {order}")
    p = order
    return {
        Shape.QUAD: (p + 1) ** 2,
        Shape.TRI: (p + 1) * (p + 2) // 2,
        Shape.HEX: (p + 1) ** 3,
        Shape.PRISM: (p + 1) ** 2 * (p + 2) // 2,
        Shape.PYR: (p + 1) * (p + 2) * (2 * p + 3) // 6,
        Shape.TET: (p + 1) * (p + 2) * (p + 3) // 6,
    }[shape]


def quad_point_counts(shape: Shape, order: int) -> tuple[int, ...]:
    """P+2 Gauss-Lobatto, P+1 Gauss-Radau-Jacobi on collapsed directions
    (shapes.py:132-139)."""
    if order < 1:
        raise ValueError(f"polynomial order must be at least 1, got {order}")
    collapsed = {
        Shape.QUAD: (False, False),
        Shape.TRI: (False, True),
        Shape.HEX: (False, False, False),
        Shape.PRISM: (False, False, True),
        Shape.PYR: (False, False, True),
        Shape.TET: (False, True, True),
    }[shape]
    return tuple(order + 1 if c else order + 2 for c in collapsed)


def index_set(shape: Shape, order: int) -> tuple[tuple[int, ...], ...]:
    """Admissible (p, q, r), lexicographic, p slowest (shapes.py:142-179)."""
    P = order
    if shape is Shape.HEX:
        return tuple((p, q, r) for p in range(P + 1) for q in range(P + 1) for r in range(P + 1))
    if shape is Shape.PRISM:
        return tuple((p, q, r) for p in range(P + 1) for q in range(P + 1) for r in range(P + 1 - p))
    if shape is Shape.PYR:
        return tuple(
            (p, q, r) for p in range(P + 1) for q in range(P + 1) for r in range(P + 1 - max(p, q))
        )
    if shape is Shape.TET:
        return tuple(
            (p, q, r) for p in range(P + 1) for q in range(P + 1 - p) for r in range(P + 1 - p - q)
        )
    if shape is Shape.QUAD:
        return tuple((p, q) for p in range(P + 1) for q in range(P + 1))
    return tuple((p, q) for p in range(P + 1) for q in range(P + 1 - p))


class ShapeBasis:
    """Handle on the native per-(shape, order) tables (replaces the
    reference dataclass, shapes.py:412-441).  ``handle`` is the
    ``sk_basis*`` every device operator takes."""

    def __init__(self, shape: Shape, order: int, qpoints: tuple[int, int, int] | None = None):
        if shape not in DEVICE_SHAPES:
            from paper_2604_04644_b200.operators import UnsupportedStrategyError

            raise UnsupportedStrategyError(f"{shape.value}: only 3D shapes are on the device path")
        lib = _lib.load()
        h = ctypes.c_void_p()
        if qpoints is None:
            _lib.check(lib.sk_basis_create(shape.abi_id, order, ctypes.byref(h)), "sk_basis_create")
        else:
            q = (ctypes.c_int * 3)(*qpoints)
            _lib.check(lib.sk_basis_create_q(shape.abi_id, order, q, ctypes.byref(h)), "sk_basis_create_q")
        self.handle = h
        self.shape = shape
        self.order = order
        cnt = (ctypes.c_int64 * 6)()
        _lib.check(lib.sk_basis_counts(h, cnt), "sk_basis_counts")
        self.qcounts = (int(cnt[0]), int(cnt[1]), int(cnt[2]))
        self.n_points = int(cnt[3])
        self.n_modes = int(cnt[4])
        # a quadrature override runs on the run-time-size device path
        # (generic.cu); the default counts on the specialised kernels
        self.generic = self.qcounts != quad_point_counts(shape, order)
        self._tables: dict[str, np.ndarray] = {}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.sk_basis_destroy(h)

    @property
    def ndim(self) -> int:
        return 3

    def table(self, name: str) -> np.ndarray:
        """Named host table from the native builder (read-only copy)."""
        if name not in self._tables:
            lib = _lib.load()
            n = ctypes.c_int64()
            _lib.check(lib.sk_basis_table(self.handle, name.encode(), None, 0, ctypes.byref(n)), "sk_basis_table")
            if n.value == 0:
                raise KeyError(name)
            out = np.empty(n.value)
            _lib.check(
                lib.sk_basis_table(
                    self.handle, name.encode(), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n.value, ctypes.byref(n)
                ),
                "sk_basis_table",
            )
            out.setflags(write=False)
            self._tables[name] = out
        return self._tables[name]

    # reference-shaped views -------------------------------------------------
    @property
    def eta(self) -> tuple[np.ndarray, ...]:
        return tuple(self.table(f"z{d}") for d in range(3))

    @property
    def weights(self) -> tuple[np.ndarray, ...]:
        return tuple(self.table(f"w{d}") for d in range(3))

    @property
    def ref_weights(self) -> np.ndarray:
        return self.table("refw")

    @property
    def dmats(self) -> tuple[np.ndarray, ...]:
        return tuple(self.table(f"D{d}").reshape(q, q) for d, q in enumerate(self.qcounts))

    @property
    def gdense(self) -> np.ndarray:
        """(n_points, 3, 3) chain-rule factors, grad_xi = G grad_eta."""
        return self.table("G").reshape(self.n_points, 3, 3)

    @property
    def modes(self) -> tuple[tuple[int, ...], ...]:
        return tuple(tuple(int(v) for v in m) for m in self.table("modes").reshape(-1, 3))

    def launch_config(self, op: int, deformed: bool = True) -> tuple[int, int, int]:
        """(elements per CTA, threads per CTA, dynamic shared bytes) of the
        kernel an operator launches for this basis and geometry class."""
        out = (ctypes.c_int64 * 3)()
        geo = _lib.SK_GEO_DEFORMED if deformed else _lib.SK_GEO_REGULAR
        _lib.check(_lib.load().sk_launch_config_geo(self.handle, op, geo, out), "sk_launch_config_geo")
        return int(out[0]), int(out[1]), int(out[2])


@lru_cache(maxsize=None)
def _cached(shape: Shape, order: int, qpoints: tuple[int, int, int] | None = None) -> ShapeBasis:
    return ShapeBasis(shape, order, qpoints)


def build_shape_basis(shape: Shape, order: int, qpoints: tuple[int, ...] | None = None) -> ShapeBasis:
    """shapes.py:521-541.  ``qpoints`` overrides the per-direction point
    counts (each at least the default, as the reference checks); the
    default counts run on the specialised kernels, any other override on the
    run-time-size dense device path (same operators, no CPU fallback)."""
    if order < 1:
        raise ValueError(f"polynomial order must be at least 1, got {order}")
    if qpoints is not None:
        qpoints = tuple(int(q) for q in qpoints)
        if len(qpoints) != 3:
            raise ValueError(f"{shape.value} needs 3 point counts, got {len(qpoints)}")
        for q, qmin in zip(qpoints, quad_point_counts(shape, order)):
            if q < qmin:
                raise ValueError(f"direction needs at least {qmin} points for order {order}, got {q}")
        if qpoints == quad_point_counts(shape, order):
            qpoints = None
    return _cached(shape, order, qpoints)
