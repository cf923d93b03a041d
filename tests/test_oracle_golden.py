"""Pin the CPU oracle to the real reference: every table and operator output
the reference produced (tests/golden/make_golden.py) must be reproduced by the
numpy restatement in ``oracle/``."""

import os

import numpy as np
import pytest

import oracle as O

SHAPES = ["hex", "prism", "pyr", "tet"]
OP_ORDERS = [1, 2, 3, 4, 5, 6, 8, 10]
TOL = 1e-13  # max-normalised; the oracle restates the same algorithm


def _close(a, b, tol=TOL):
    assert a.shape == b.shape, (a.shape, b.shape)
    err = O.rel_diff(a, b)
    assert err <= tol, err


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", range(1, 11))
def test_tables(golden_tables, shape, P):
    g = golden_tables
    el = O.element(shape, P)
    k = f"{shape}_P{P}"
    for d in range(3):
        np.testing.assert_allclose(el.z[d], g[f"{k}_z{d}"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(el.w[d], g[f"{k}_w{d}"], rtol=1e-14, atol=0)
        _close(el.D[d], g[f"{k}_D{d}"])
        if el.a[d] is not None:
            _close(el.a[d][0], g[f"{k}_a{d}"])
            _close(el.a[d][1], g[f"{k}_da{d}"])
        else:
            assert f"{k}_a{d}" not in g
    for name in ("b2", "c3"):
        fam = getattr(el, name)
        if fam is None:
            assert f"{k}_{name}_0" not in g
            continue
        for p, (v, dv) in enumerate(fam):
            _close(v, g[f"{k}_{name}_{p}"])
            _close(dv, g[f"{k}_d{name}_{p}"])
    _close(el.refw, g[f"{k}_refw"])
    _close(el.G, g[f"{k}_G"])
    if P <= 4:
        _close(el.bmat, g[f"{k}_bmat"])
    for kind in (
        "bwdtrans",
        "iproduct",
        "physderiv",
        "iproduct_deriv",
        "mass",
        "helmholtz_noncoll",
        "helmholtz_coll",
    ):
        assert O.flops(kind, shape, P) == int(g[f"{k}_flops_{kind}"])


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", OP_ORDERS)
@pytest.mark.parametrize("geo", ["regular", "deformed"])
def test_operators(golden_ops, shape, P, geo):
    g = golden_ops
    k = f"{shape}_P{P}_{geo}"
    el = O.element(shape, P)
    geom = O.synthetic_geometry(el, geo == "deformed", 2, seed=3)
    if P <= 4:
        _close(geom.dxi, g[f"{k}_dxi"])
        _close(geom.jac, g[f"{k}_jac"])
    x, y, v = g[f"{k}_x"], g[f"{k}_y"], g[f"{k}_v"]
    _close(O.bwd_trans(el, geom, x), g[f"{k}_bwd"])
    _close(O.mass(el, geom, x), g[f"{k}_mass"])
    for lam in (0.0, 1.0, 2.5):
        _close(O.helmholtz_coll(el, geom, x, lam), g[f"{k}_helm_{lam}"])
    _close(O.helmholtz_noncoll(el, geom, x, 1.0), g[f"{k}_helmnc_1.0"])
    _close(O.iproduct_wrt_base(el, geom, y), g[f"{k}_iprod"])
    _close(O.phys_deriv(el, geom, y), g[f"{k}_dphys"])
    _close(O.iproduct_wrt_deriv_base(el, geom, v), g[f"{k}_ipderiv"])
    if P <= 4:
        e = 1
        _close(O.dense_helmholtz(el, geom, 1.0, e) @ x[:, e], g[f"{k}_dense_helm_1.0"])
        _close(O.dense_mass(el, geom, e) @ x[:, e], g[f"{k}_dense_mass"])
        # independent routes agree (reference acceptance criterion 2)
        _close(O.helmholtz_coll(el, geom, x, 1.0)[:, e], g[f"{k}_dense_helm_1.0"], 1e-11)


def test_bench_workload_seeding(golden_ops):
    """The bench's per-element seeded geometry and coefficients reproduce the
    reference's for arbitrary element indices (tiling/sharding safety)."""
    g = golden_ops
    el = O.element("tet", 4)
    idx = g["bench_tet_P4_idx"]
    params = np.concatenate([O.deformation_params(1, 0, first=int(e)) for e in idx])
    from oracle.geom import deformed_coords

    geom = O.deformed_geometry_from_coords(el, deformed_coords(el, params))
    _close(geom.dxi, g["bench_tet_P4_dxi"])
    _close(geom.jac, g["bench_tet_P4_jac"])
    x = O.bench_coeffs(O.SHAPE_INDEX["tet"], 4, el.nm, 70000, seed=0)
    _close(x[:, idx], g["bench_tet_P4_x"], 0.0)


@pytest.mark.parametrize("shape", SHAPES)
def test_two_dense_routes(shape):
    """oracle two-route agreement (reference test_oracle.py:87-96)."""
    for P in (1, 2, 3):
        el = O.element(shape, P)
        for deformed in (False, True):
            geom = O.synthetic_geometry(el, deformed, 1, seed=1)
            a = O.dense_helmholtz(el, geom, 1.5)
            b = O.dense_helmholtz_factored(el, geom, 1.5)
            assert np.max(np.abs(a - b)) / np.max(np.abs(a)) <= 1e-12


QCASES = [("hex", 2, (5, 4, 6)), ("prism", 3, (6, 5, 6)), ("pyr", 2, (5, 6, 4)), ("tet", 3, (6, 5, 6)), ("tet", 1, (3, 4, 2))]


@pytest.fixture(scope="module")
def golden_q():
    from conftest import GOLDEN

    return np.load(os.path.join(GOLDEN, "operators_qpoints.npz"))


@pytest.mark.parametrize("shape,P,q", QCASES)
@pytest.mark.parametrize("gname", ["regular", "deformed"])
def test_oracle_quadrature_override_matches_reference(golden_q, shape, P, q, gname):
    """The oracle with a qpoints override (element(shape, P, q)) reproduces
    the reference's operators on the reference's own factors."""
    k = f"{shape}_P{P}_q{''.join(map(str, q))}_{gname}"
    g = golden_q
    el = O.element(shape, P, q)
    geo = O.Geometry(gname == "deformed", g[f"{k}_dxi"], g[f"{k}_jac"])
    x, y, v = g[f"{k}_x"], g[f"{k}_y"], g[f"{k}_v"]
    tol = 1e-13
    assert O.rel_diff(O.bwd_trans(el, geo, x), g[f"{k}_bwd"]) <= tol
    assert O.rel_diff(O.mass(el, geo, x), g[f"{k}_mass"]) <= tol
    for lam in (0.0, 1.0):
        assert O.rel_diff(O.helmholtz_coll(el, geo, x, lam), g[f"{k}_helm_{lam}"]) <= tol
    assert O.rel_diff(O.helmholtz_noncoll(el, geo, x, 1.0), g[f"{k}_helmnc_1.0"]) <= tol
    assert O.rel_diff(O.iproduct_wrt_base(el, geo, y), g[f"{k}_iprod"]) <= tol
    assert O.rel_diff(O.phys_deriv(el, geo, y), g[f"{k}_dphys"]) <= tol
    assert O.rel_diff(O.iproduct_wrt_deriv_base(el, geo, v), g[f"{k}_ipderiv"]) <= tol
    assert O.rel_diff(O.synthetic_geometry(el, gname == "deformed", 2, seed=5).jac, g[f"{k}_jac"]) <= 1e-13
