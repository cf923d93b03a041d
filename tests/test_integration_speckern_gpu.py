"""End-to-end drop-in check with the UNMODIFIED reference: real speckern
Blocks and Fields (installed in baseline/_ref by __graft_entry__.build(),
never imported from /root/reference) driven through the reference-side
binding in integration/speckern_sk200.py.  Every operator routed through
Strategy.SUM_FAC_TOP must equal speckern's own SUM_FAC output to 1e-12
(max-normalised, speckern bench.py:192-194)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TOL = 1e-12

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def speckern():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "speckern")):
        pytest.fail("reference not installed in baseline/_ref (run __graft_entry__.build() where /root/reference exists)")
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import speckern

    assert os.path.realpath(speckern.__file__).startswith(os.path.realpath(REF))
    return speckern


@pytest.fixture()
def routed(speckern):
    import speckern_sk200 as binding

    binding.install(speckern)
    yield binding
    binding.uninstall(speckern)


def _err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(a)), np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("shape", ["HEX", "PRISM", "PYR", "TET"])
@pytest.mark.parametrize("gcls", ["REGULAR", "DEFORMED"])
def test_every_operator_through_binding(speckern, shape, gcls):
    """All seven reference operators on a reference Block (interleave width
    8, ragged last group) via the binding vs speckern SUM_FAC."""
    import speckern_sk200 as binding
    from speckern import operators as ref
    from speckern.field_block import FieldState, make_field
    from speckern.geometry import GeometryClass
    from speckern.operators import Strategy
    from speckern.shapes import Shape

    S = Strategy.SUM_FAC
    T = Strategy.SUM_FAC_TOP
    field = make_field(Shape[shape], 3, GeometryClass[gcls], 53, interleave_width=8, seed=2)
    blk = field.blocks[0]
    rng = np.random.default_rng(0)
    blk.set_elements(rng.uniform(-1, 1, (blk.n_data, blk.n_elements)))
    for lam in (0.0, 1.0, 2.5):
        assert _err(binding.helmholtz_apply_coll(blk, lam, T).get_elements(),
                    ref.helmholtz_apply_coll(blk, lam, S).get_elements()) <= TOL
        assert _err(binding.helmholtz_apply_noncoll(blk, lam, T).get_elements(),
                    ref.helmholtz_apply_noncoll(blk, lam, S).get_elements()) <= TOL
    assert _err(binding.helmholtz_apply(blk, 1.0, T).get_elements(),
                ref.helmholtz_apply(blk, 1.0, S).get_elements()) <= TOL
    assert _err(binding.mass_apply(blk, T).get_elements(), ref.mass_apply(blk, S).get_elements()) <= TOL
    assert _err(binding.bwd_trans(blk, T).get_elements(), ref.bwd_trans(blk, S).get_elements()) <= TOL
    pb = blk.like(FieldState.PHYS)
    pb.set_elements(rng.uniform(-1, 1, (pb.n_data, pb.n_elements)))
    assert _err(binding.iproduct_wrt_base(pb, T).get_elements(), ref.iproduct_wrt_base(pb, S).get_elements()) <= TOL
    assert _err(binding.phys_deriv(pb).get_elements(), ref.phys_deriv(pb).get_elements()) <= TOL
    vb = blk.like(FieldState.PHYS, 3)
    vb.set_elements(rng.uniform(-1, 1, (3, vb.n_data, vb.n_elements)))
    assert _err(binding.iproduct_wrt_deriv_base(vb, T).get_elements(),
                ref.iproduct_wrt_deriv_base(vb, S).get_elements()) <= TOL


def test_mixed_field_apply_to_field_routed(speckern, routed):
    """speckern's own apply_to_field on a mixed hex/prism/pyr/tet P=6 field
    with Strategy.SUM_FAC_TOP (routed by install()) equals SUM_FAC per
    block, serially and with the reference's thread pool."""
    from speckern.field_block import make_field
    from speckern.geometry import GeometryClass
    from speckern.operators import OperatorKind, Strategy, apply_to_field
    from speckern.shapes import Shape

    field = make_field([Shape.HEX, Shape.PRISM, Shape.PYR, Shape.TET], 6, GeometryClass.DEFORMED, 24, seed=1)
    rng = np.random.default_rng(5)
    for b in field.blocks:
        b.set_elements(rng.uniform(-1, 1, (b.n_data, b.n_elements)))
    launches0 = _launches()
    for kind in (OperatorKind.HELMHOLTZ_COLL, OperatorKind.HELMHOLTZ_NONCOLL, OperatorKind.MASS):
        want = apply_to_field(kind, field, Strategy.SUM_FAC, 1.0)
        for threads in (1, 4):
            got = apply_to_field(kind, field, Strategy.SUM_FAC_TOP, 1.0, threads=threads)
            for g, w in zip(got.blocks, want.blocks):
                assert _err(g.get_elements(), w.get_elements()) <= TOL, (kind, g.shape)
    assert _launches() - launches0 >= 4 * 3 * 2  # every block ran on the device


def test_apply_operator_every_kind_routed(speckern, routed):
    """speckern.apply_operator(kind, block, SUM_FAC_TOP) for every kind."""
    from speckern.field_block import FieldState, make_field
    from speckern.geometry import GeometryClass
    from speckern.operators import OperatorKind, Strategy, apply_operator
    from speckern.shapes import Shape

    blk = make_field(Shape.TET, 4, GeometryClass.DEFORMED, 17, interleave_width=4, seed=3).blocks[0]
    rng = np.random.default_rng(1)
    blk.set_elements(rng.uniform(-1, 1, (blk.n_data, blk.n_elements)))
    pb = blk.like(FieldState.PHYS)
    pb.set_elements(rng.uniform(-1, 1, (pb.n_data, pb.n_elements)))
    vb = blk.like(FieldState.PHYS, 3)
    vb.set_elements(rng.uniform(-1, 1, (3, vb.n_data, vb.n_elements)))
    inputs = {OperatorKind.BWD_TRANS: blk, OperatorKind.MASS: blk, OperatorKind.HELMHOLTZ_COLL: blk,
              OperatorKind.HELMHOLTZ_NONCOLL: blk, OperatorKind.IPRODUCT_WRT_BASE: pb, OperatorKind.PHYS_DERIV: pb,
              OperatorKind.IPRODUCT_WRT_DERIV_BASE: vb}
    for kind, b in inputs.items():
        n0 = _launches()
        got = apply_operator(kind, b, Strategy.SUM_FAC_TOP, 0.7)
        assert _launches() > n0, kind
        want = apply_operator(kind, b, Strategy.SUM_FAC, 0.7)
        assert _err(got.get_elements(), want.get_elements()) <= TOL, kind


def test_binding_errors_are_reference_types(speckern):
    import speckern_sk200 as binding
    from speckern.field_block import FieldState, make_field
    from speckern.geometry import GeometryClass
    from speckern.operators import FieldStateError, Strategy, UnsupportedStrategyError
    from speckern.shapes import Shape

    T = Strategy.SUM_FAC_TOP
    blk = make_field(Shape.HEX, 2, GeometryClass.REGULAR, 3, seed=0).blocks[0]
    with pytest.raises(FieldStateError):
        binding.iproduct_wrt_base(blk, T)
    with pytest.raises(ValueError):
        binding.helmholtz_apply_coll(blk, -1.0, T)
    with pytest.raises(FieldStateError):
        binding.mass_apply(blk, T, out=blk.like(FieldState.PHYS))
    quad = make_field(Shape.QUAD, 2, GeometryClass.REGULAR, 3, seed=0).blocks[0]  # 2D: not on the device path
    with pytest.raises(UnsupportedStrategyError):
        binding.mass_apply(quad, T)


@pytest.mark.parametrize("gcls", ["REGULAR", "DEFORMED"])
def test_quadrature_override_blocks_through_binding(speckern, gcls):
    """speckern blocks built with a qpoints override (shapes.py:521-541) run
    through the binding on the library's run-time-size path and equal
    speckern's SUM_FAC output."""
    import speckern_sk200 as binding
    from speckern import operators as ref
    from speckern.field_block import FieldState, make_field
    from speckern.geometry import GeometryClass
    from speckern.operators import Strategy
    from speckern.shapes import Shape

    S, T = Strategy.SUM_FAC, Strategy.SUM_FAC_TOP
    for shp, P, q in ((Shape.TET, 3, (6, 5, 6)), (Shape.HEX, 2, (5, 4, 6))):
        blk = make_field(shp, P, GeometryClass[gcls], 11, interleave_width=4, seed=4, qpoints=q).blocks[0]
        rng = np.random.default_rng(2)
        blk.set_elements(rng.uniform(-1, 1, (blk.n_data, blk.n_elements)))
        assert _err(binding.helmholtz_apply_coll(blk, 1.2, T).get_elements(),
                    ref.helmholtz_apply_coll(blk, 1.2, S).get_elements()) <= TOL
        assert _err(binding.mass_apply(blk, T).get_elements(), ref.mass_apply(blk, S).get_elements()) <= TOL
        pb = blk.like(FieldState.PHYS)
        pb.set_elements(rng.uniform(-1, 1, (pb.n_data, pb.n_elements)))
        assert _err(binding.phys_deriv(pb).get_elements(), ref.phys_deriv(pb).get_elements()) <= TOL


def _launches():
    import speckern_sk200 as binding

    lib = binding._lib()
    lib.sk_launch_count.restype = __import__("ctypes").c_int64
    return int(lib.sk_launch_count())
