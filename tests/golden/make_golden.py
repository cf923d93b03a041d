"""Generate the golden vectors that pin the oracle (and the product) to the
real reference implementation.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``speckern`` (the unmodified reference), evaluates the hot-path
operators with the reference's own public API and stock SUM_FAC strategy on
small seeded blocks, and writes ``tests/golden/*.npz``.  The fixtures travel
with the repo; ``/root/reference`` is never read at test time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from speckern import oracle as ref_oracle  # noqa: E402
from speckern.field_block import Block, FieldState  # noqa: E402
from speckern.geometry import GeometryClass, make_synthetic_factors  # noqa: E402
from speckern.operators import (  # noqa: E402
    OperatorKind,
    Strategy,
    apply_operator,
    bwd_trans,
    helmholtz_apply_coll,
    helmholtz_apply_noncoll,
    iproduct_wrt_base,
    iproduct_wrt_deriv_base,
    mass_apply,
    operator_flops,
    phys_deriv,
)
from speckern.shapes import Shape, build_shape_basis  # noqa: E402

SHAPES = [Shape.HEX, Shape.PRISM, Shape.PYR, Shape.TET]
TABLE_ORDERS = list(range(1, 11))
OP_ORDERS = [1, 2, 3, 4, 5, 6, 8, 10]
N_EL = 2
WIDTH = 2


def _fill(block, key):
    rng = np.random.default_rng(key)
    vals = rng.uniform(-1.0, 1.0, size=(block.n_elements, block.n_data))
    block.set_elements(np.ascontiguousarray(vals.T)[None])
    return np.ascontiguousarray(vals.T)


def tables(out):
    for shp in SHAPES:
        for P in TABLE_ORDERS:
            sb = build_shape_basis(shp, P)
            k = f"{shp.value}_P{P}"
            for d in range(3):
                out[f"{k}_z{d}"] = sb.rules[d].points
                out[f"{k}_w{d}"] = sb.rules[d].weights
                out[f"{k}_D{d}"] = sb.dmats[d]
                if sb.tables.a[d] is not None:
                    out[f"{k}_a{d}"] = sb.tables.a[d][0]
                    out[f"{k}_da{d}"] = sb.tables.a[d][1]
            for name in ("b2", "c3"):
                fam = getattr(sb.tables, name)
                if fam is not None:
                    for p, (v, dv) in enumerate(fam):
                        out[f"{k}_{name}_{p}"] = v
                        out[f"{k}_d{name}_{p}"] = dv
            out[f"{k}_refw"] = sb.ref_weights
            g = np.zeros((sb.n_points, 3, 3))
            for i in range(3):
                for j in range(3):
                    ent = sb.gmap.entries[i][j]
                    if ent is not None:
                        g[:, i, j] = ent
            out[f"{k}_G"] = g
            if P <= 4:
                out[f"{k}_bmat"] = sb.bmat
            for kind in OperatorKind:
                out[f"{k}_flops_{kind.value}"] = np.array(operator_flops(kind, shp, P, Strategy.SUM_FAC))


def operators(out):
    for shp in SHAPES:
        sidx = list(Shape).index(shp)
        for P in OP_ORDERS:
            sb = build_shape_basis(shp, P)
            for gcls in (GeometryClass.REGULAR, GeometryClass.DEFORMED):
                k = f"{shp.value}_P{P}_{gcls.value}"
                fac = make_synthetic_factors(sb, gcls, N_EL, seed=3)
                if P <= 4:
                    out[f"{k}_dxi"] = fac.dxi_dx
                    out[f"{k}_jac"] = fac.jac
                cb = Block(sb, fac, FieldState.COEFF, 1, WIDTH)
                x = _fill(cb, [3, sidx, P, 1])
                out[f"{k}_x"] = x
                out[f"{k}_bwd"] = bwd_trans(cb, Strategy.SUM_FAC).get_elements()[0]
                out[f"{k}_mass"] = mass_apply(cb, Strategy.SUM_FAC).get_elements()[0]
                for lam in (0.0, 1.0, 2.5):
                    out[f"{k}_helm_{lam}"] = helmholtz_apply_coll(cb, lam, Strategy.SUM_FAC).get_elements()[0]
                out[f"{k}_helmnc_1.0"] = helmholtz_apply_noncoll(cb, 1.0, Strategy.SUM_FAC).get_elements()[0]
                pb = Block(sb, fac, FieldState.PHYS, 1, WIDTH)
                y = _fill(pb, [3, sidx, P, 2])
                out[f"{k}_y"] = y
                out[f"{k}_iprod"] = iproduct_wrt_base(pb, Strategy.SUM_FAC).get_elements()[0]
                out[f"{k}_dphys"] = phys_deriv(pb).get_elements()
                vb = Block(sb, fac, FieldState.PHYS, 3, WIDTH)
                rng = np.random.default_rng([3, sidx, P, 3])
                v = rng.uniform(-1.0, 1.0, size=(3, sb.n_points, N_EL))
                vb.set_elements(v)
                out[f"{k}_v"] = v
                out[f"{k}_ipderiv"] = iproduct_wrt_deriv_base(vb, Strategy.SUM_FAC).get_elements()[0]
                if P <= 4:
                    e = N_EL - 1
                    out[f"{k}_dense_helm_1.0"] = ref_oracle.assemble_helmholtz(sb, fac, 1.0, e).matrix @ x[:, e]
                    out[f"{k}_dense_mass"] = ref_oracle.assemble_mass(sb, fac, e).matrix @ x[:, e]


def bench_workload(out):
    """Pins the bench workload's seeded geometry and coefficients: element e
    of a seed-0 synthetic block depends only on (seed, e) (geometry.py:288)."""
    sb = build_shape_basis(Shape.TET, 4)
    ne = 70000
    idx = np.array([0, 1, 2, 12345, 65535, 69999])
    # deformed parameters are per-element: build only the sampled elements
    from speckern.geometry import deformed_factors_from_coords, quadrature_coords, synthetic_deformation

    mapping = synthetic_deformation(Shape.TET, 0)
    xi = quadrature_coords(sb)
    coords = np.stack([mapping(xi, int(e)) for e in idx])
    fac = deformed_factors_from_coords(sb, coords)
    out["bench_tet_P4_idx"] = idx
    out["bench_tet_P4_dxi"] = fac.dxi_dx
    out["bench_tet_P4_jac"] = fac.jac
    rng = np.random.default_rng([0, list(Shape).index(Shape.TET), 4, 1])
    vals = rng.uniform(-1.0, 1.0, size=(ne, sb.n_modes))
    out["bench_tet_P4_x"] = np.ascontiguousarray(vals[idx].T)


#: quadrature overrides (shapes.py:521-541): every shape, one or more
#: directions above the default P+2 / P+1 counts
QPOINT_CASES = [
    (Shape.HEX, 2, (5, 4, 6)),
    (Shape.PRISM, 3, (6, 5, 6)),
    (Shape.PYR, 2, (5, 6, 4)),
    (Shape.TET, 3, (6, 5, 6)),
    (Shape.TET, 1, (3, 4, 2)),
]


def qpoint_operators(out):
    """Every operator on blocks whose basis carries a quadrature override."""
    for shp, P, q in QPOINT_CASES:
        sidx = list(Shape).index(shp)
        sb = build_shape_basis(shp, P, q)
        for gcls in (GeometryClass.REGULAR, GeometryClass.DEFORMED):
            k = f"{shp.value}_P{P}_q{''.join(map(str, q))}_{gcls.value}"
            fac = make_synthetic_factors(sb, gcls, N_EL, seed=5)
            out[f"{k}_dxi"] = fac.dxi_dx
            out[f"{k}_jac"] = fac.jac
            cb = Block(sb, fac, FieldState.COEFF, 1, WIDTH)
            out[f"{k}_x"] = _fill(cb, [5, sidx, P, 1])
            out[f"{k}_bwd"] = bwd_trans(cb, Strategy.SUM_FAC).get_elements()[0]
            out[f"{k}_mass"] = mass_apply(cb, Strategy.SUM_FAC).get_elements()[0]
            for lam in (0.0, 1.0):
                out[f"{k}_helm_{lam}"] = helmholtz_apply_coll(cb, lam, Strategy.SUM_FAC).get_elements()[0]
            out[f"{k}_helmnc_1.0"] = helmholtz_apply_noncoll(cb, 1.0, Strategy.SUM_FAC).get_elements()[0]
            pb = Block(sb, fac, FieldState.PHYS, 1, WIDTH)
            out[f"{k}_y"] = _fill(pb, [5, sidx, P, 2])
            out[f"{k}_iprod"] = iproduct_wrt_base(pb, Strategy.SUM_FAC).get_elements()[0]
            out[f"{k}_dphys"] = phys_deriv(pb).get_elements()
            vb = Block(sb, fac, FieldState.PHYS, 3, WIDTH)
            v = np.random.default_rng([5, sidx, P, 3]).uniform(-1.0, 1.0, size=(3, sb.n_points, N_EL))
            vb.set_elements(v)
            out[f"{k}_v"] = v
            out[f"{k}_ipderiv"] = iproduct_wrt_deriv_base(vb, Strategy.SUM_FAC).get_elements()[0]


def main():
    only_q = len(sys.argv) > 1 and sys.argv[1] == "qpoints"
    if not only_q:
        t = {}
        tables(t)
        np.savez_compressed(os.path.join(HERE, "tables.npz"), **t)
        o = {}
        operators(o)
        bench_workload(o)
        np.savez_compressed(os.path.join(HERE, "operators.npz"), **o)
    qo = {}
    qpoint_operators(qo)
    np.savez_compressed(os.path.join(HERE, "operators_qpoints.npz"), **qo)
    for name in ("tables.npz", "operators.npz", "operators_qpoints.npz"):
        print(name, os.path.getsize(os.path.join(HERE, name)) // 1024, "KiB")


if __name__ == "__main__":
    sys.exit(main())
