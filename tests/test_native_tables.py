"""CPU tests of the native library: exported symbols match include/sk200.h,
and the natively built constant tables equal the reference's (golden) ones.
No device is needed: sk_basis_create is host-only."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import oracle as O

LIB = os.path.join(ROOT, "paper_2604_04644_b200", "libsk200.so")
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="libsk200.so not built")

SHAPES = ["hex", "prism", "pyr", "tet"]


def _declared():
    src = open(os.path.join(ROOT, "include", "sk200.h")).read()
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    from paper_2604_04644_b200 import _lib

    lib = _lib.load()
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_status_codes_and_errors():
    import paper_2604_04644_b200 as sk
    from paper_2604_04644_b200 import _lib

    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.sk_basis_create(0, 3, ctypes.byref(h)) == _lib.SK_ERR_UNSUPPORTED  # quad
    assert lib.sk_basis_create(9, 3, ctypes.byref(h)) == _lib.SK_ERR_STATE
    assert lib.sk_basis_create(2, 0, ctypes.byref(h)) == _lib.SK_ERR_ARG
    assert lib.sk_basis_create(2, 11, ctypes.byref(h)) == _lib.SK_ERR_UNSUPPORTED
    with pytest.raises(sk.UnsupportedStrategyError):
        sk.build_shape_basis(sk.Shape.QUAD, 2)
    with pytest.raises(ValueError):  # below the default counts (shapes.py:532-541)
        sk.build_shape_basis(sk.Shape.HEX, 2, qpoints=(3, 5, 5))
    q = (ctypes.c_int * 3)(4, 4, 3)
    assert lib.sk_basis_create_q(2, 2, q, ctypes.byref(h)) == _lib.SK_ERR_ARG
    b = sk.build_shape_basis(sk.Shape.TET, 3)
    # argument checks happen before any device work
    assert lib.sk_helmholtz_apply(b.handle, 1, 0, 4, 1, 1, None, None, -1.0, None, None) == _lib.SK_ERR_ARG
    assert lib.sk_mass_apply(b.handle, 1, -1, 1, 1, None, None, None, None) == _lib.SK_ERR_ARG
    assert lib.sk_bwd_trans(b.handle, 4, 0, 1, None, None, None) == _lib.SK_ERR_ARG
    # recomputed-metric Helmholtz and the streamed entry point validate before any device work
    dummy = ctypes.c_void_p(16)
    assert lib.sk_helmholtz_apply_params(b.handle, 4, 1, 1, None, None, 1.0, None, None, 16, None, None) == _lib.SK_ERR_ARG
    assert lib.sk_helmholtz_apply_params(b.handle, 4, 1, 1, dummy, dummy, -1.0, dummy, dummy, 16, None, None) == _lib.SK_ERR_ARG
    assert lib.sk_helmholtz_apply_params(b.handle, 40, 1, 1, dummy, dummy, 1.0, dummy, dummy, 24, None, None) == _lib.SK_ERR_ARG
    bq = sk.build_shape_basis(sk.Shape.TET, 3, qpoints=(6, 5, 6))
    assert lib.sk_helmholtz_apply_params(bq.handle, 4, 1, 1, dummy, dummy, 1.0, dummy, dummy, 16, None, None) == _lib.SK_ERR_UNSUPPORTED
    assert lib.sk_apply_streamed_ex(b.handle, 0, 1, 4, 1, 1, dummy, dummy, dummy, 1.0, dummy, dummy, 0, 4, None) == _lib.SK_ERR_ARG


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", range(1, 11))
def test_native_tables_match_reference(golden_tables, shape, P):
    import paper_2604_04644_b200 as sk

    g = golden_tables
    k = f"{shape}_P{P}"
    b = sk.build_shape_basis(sk.Shape(shape), P)
    assert b.qcounts == O.qcounts(shape, P)
    assert b.n_modes == O.mode_count(shape, P)
    assert b.modes == tuple(O.mode_set(shape, P))

    def close(a, ref, tol=1e-14):
        a = np.asarray(a).reshape(ref.shape)
        assert np.max(np.abs(a - ref)) <= tol * max(1.0, np.max(np.abs(ref))), (np.max(np.abs(a - ref)))

    for d in range(3):
        close(b.table(f"z{d}"), g[f"{k}_z{d}"])
        close(b.table(f"w{d}"), g[f"{k}_w{d}"])
        close(b.table(f"D{d}"), g[f"{k}_D{d}"], 1e-13)
        if f"{k}_a{d}" in g:
            close(b.table(f"a{d}"), g[f"{k}_a{d}"])
            close(b.table(f"da{d}"), g[f"{k}_da{d}"], 1e-13)
    for name, native in (("b2", "b1"), ("c3", "c2")):
        p = 0
        while f"{k}_{name}_{p}" in g:
            close(b.table(f"{native}_{p}"), g[f"{k}_{name}_{p}"])
            close(b.table(f"d{native}_{p}"), g[f"{k}_d{name}_{p}"], 1e-13)
            p += 1
    close(b.ref_weights, g[f"{k}_refw"])
    close(b.gdense, g[f"{k}_G"], 1e-14)



@pytest.mark.parametrize("shape,P,q", [("hex", 2, (5, 4, 6)), ("prism", 3, (6, 5, 6)), ("pyr", 2, (5, 6, 4)),
                                       ("tet", 3, (6, 5, 6)), ("tet", 1, (3, 4, 2))])
def test_quadrature_override_tables(shape, P, q):
    """A qpoints basis (build_shape_basis override): native rules, weights,
    collocation matrices and the dense basis matrix of the generic device
    path equal the oracle's (pinned to the reference's qpoints operators in
    test_oracle_golden.py)."""
    import oracle as O
    import paper_2604_04644_b200 as sk

    b = sk.build_shape_basis(sk.Shape(shape), P, q)
    el = O.element(shape, P, q)
    assert b.qcounts == q and b.generic and b.n_points == el.nq
    for d in range(3):
        assert np.allclose(b.table(f"z{d}"), el.z[d], rtol=0, atol=1e-14)
        assert np.allclose(b.table(f"w{d}"), el.w[d], rtol=0, atol=1e-14)
    assert np.allclose(b.ref_weights, el.refw, rtol=0, atol=1e-14)
    assert np.allclose(b.table("B").reshape(el.nq, el.nm), el.bmat, rtol=0, atol=1e-13)
