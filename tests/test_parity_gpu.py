"""Device parity: every operator of the device path against the reference's
golden outputs and the CPU oracle, through the public API (C ABI underneath).

Bar (BASELINE north star): max-normalised error <= 1e-12 in FP64
(reference metric bench.py:192-194)."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

SHAPES = ["hex", "prism", "pyr", "tet"]
TOL = 1e-12


@pytest.fixture(scope="module")
def sk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_04644_b200 as sk

    return sk


def _block(sk, shape, P, deformed, n, seed, width, state=None, ncomp=1):
    b = sk.build_shape_basis(sk.Shape(shape), P)
    gcls = sk.GeometryClass.DEFORMED if deformed else sk.GeometryClass.REGULAR
    fac = sk.make_synthetic_factors(b, gcls, n, seed=seed)
    return sk.Block(b, fac, state or sk.FieldState.COEFF, ncomp, width)


def _err(a, b):
    return O.rel_diff(np.asarray(a), np.asarray(b))


def _block_from(sk, shape, P, geo, width, state=None, ncomp=1):
    """Block on externally supplied GeometricFactors (identical inputs)."""
    b = sk.build_shape_basis(sk.Shape(shape), P)
    gcls = sk.GeometryClass.DEFORMED if geo.deformed else sk.GeometryClass.REGULAR
    fac = sk.GeometricFactors(gcls, sk.Shape(shape), geo.n, dxi_dx=geo.dxi, jac=geo.jac)
    return sk.Block(b, fac, state or sk.FieldState.COEFF, ncomp, width)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 6, 8, 10])
@pytest.mark.parametrize("gname", ["regular", "deformed"])
def test_golden(sk, golden_ops, shape, P, gname):
    """Against the real reference's outputs (tests/golden/make_golden.py)."""
    g = golden_ops
    k = f"{shape}_P{P}_{gname}"
    deformed = gname == "deformed"
    blk = _block(sk, shape, P, deformed, 2, 3, 2)
    blk.set_elements(g[f"{k}_x"][None])
    for lam in (0.0, 1.0, 2.5):
        got = sk.helmholtz_apply(blk, lam).get_elements()[0]
        assert _err(got, g[f"{k}_helm_{lam}"]) <= TOL, (lam, _err(got, g[f"{k}_helm_{lam}"]))
    assert _err(sk.mass_apply(blk).get_elements()[0], g[f"{k}_mass"]) <= TOL
    assert _err(sk.bwd_trans(blk).get_elements()[0], g[f"{k}_bwd"]) <= TOL
    got = sk.helmholtz_apply(blk, 1.0, form="noncoll").get_elements()[0]
    assert _err(got, g[f"{k}_helmnc_1.0"]) <= TOL
    pb = blk.like(sk.FieldState.PHYS)
    pb.set_elements(g[f"{k}_y"][None])
    assert _err(sk.iproduct_wrt_base(pb).get_elements()[0], g[f"{k}_iprod"]) <= TOL
    # phys_deriv on the reference's own factors (stored for P <= 4) or the
    # oracle's (pinned to them): see test_oracle_ragged_tiles
    if f"{k}_dxi" in g:
        geo = O.Geometry(deformed, g[f"{k}_dxi"], g[f"{k}_jac"])
    else:
        geo = O.synthetic_geometry(O.element(shape, P), deformed, 2, seed=3)
    pb2 = _block_from(sk, shape, P, geo, 2, sk.FieldState.PHYS)
    pb2.set_elements(g[f"{k}_y"][None])
    assert _err(sk.phys_deriv(pb2).get_elements(), g[f"{k}_dphys"]) <= TOL
    vb = blk.like(sk.FieldState.PHYS, 3)
    vb.set_elements(g[f"{k}_v"])
    assert _err(sk.iproduct_wrt_deriv_base(vb).get_elements()[0], g[f"{k}_ipderiv"]) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [2, 4, 7, 9])
@pytest.mark.parametrize("width", [1, 8])
def test_oracle_ragged_tiles(sk, shape, P, width):
    """Many elements (not a multiple of the CTA tile nor of the width)
    against the oracle on the same seeded mesh."""
    n = 157
    el = O.element(shape, P)
    for deformed in (False, True):
        blk = _block(sk, shape, P, deformed, n, 5, width)
        geo = O.synthetic_geometry(el, deformed, n, seed=5)
        x = O.bench_coeffs(O.SHAPE_INDEX[shape], P, el.nm, n, seed=5)
        blk.set_elements(x[None])
        for lam in (0.0, 1.3):
            got = sk.helmholtz_apply(blk, lam).get_elements()[0]
            assert _err(got, O.helmholtz_coll(el, geo, x, lam)) <= TOL
            got = sk.helmholtz_apply_noncoll(blk, lam).get_elements()[0]
            assert _err(got, O.helmholtz_noncoll(el, geo, x, lam)) <= TOL
        assert _err(sk.mass_apply(blk).get_elements()[0], O.mass(el, geo, x)) <= TOL
        y = np.random.default_rng(P).uniform(-1, 1, (el.nq, n))
        pb = blk.like(sk.FieldState.PHYS)
        pb.set_elements(y[None])
        assert _err(sk.iproduct_wrt_base(pb).get_elements()[0], O.iproduct_wrt_base(el, geo, y)) <= TOL
        # phys_deriv amplifies 1-ulp differences of the metric near collapsed
        # vertices (reference geometry perturbed by 1 ulp moves it by ~1e-11
        # at tet P=9), so it is checked on identical geometric factors
        pb2 = _block_from(sk, shape, P, geo, width, sk.FieldState.PHYS)
        pb2.set_elements(y[None])
        assert _err(sk.phys_deriv(pb2).get_elements(), O.phys_deriv(el, geo, y)) <= TOL
        v = np.random.default_rng(P + 1).uniform(-1, 1, (3, el.nq, n))
        vb = _block_from(sk, shape, P, geo, width, sk.FieldState.PHYS, 3)
        vb.set_elements(v)
        assert _err(sk.iproduct_wrt_deriv_base(vb).get_elements()[0], O.iproduct_wrt_deriv_base(el, geo, v)) <= TOL
        # and every coefficient-space operator on identical factors as well
        cb = _block_from(sk, shape, P, geo, width)
        cb.set_elements(x[None])
        assert _err(sk.helmholtz_apply(cb, 1.3).get_elements()[0], O.helmholtz_coll(el, geo, x, 1.3)) <= TOL
        assert _err(sk.bwd_trans(cb).get_elements()[0], O.bwd_trans(el, geo, x)) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [1, 3, 5, 6, 8, 10])
def test_regular_multi_tile_every_order(sk, shape, P):
    """Regular-geometry collocated Helmholtz / stiffness on several CTA tiles
    at the orders whose regular launch table (tile width, thread divisor)
    differs from the deformed one: every element against the oracle."""
    n = 301
    el = O.element(shape, P)
    blk = _block(sk, shape, P, False, n, 11, 1)
    geo = O.synthetic_geometry(el, False, n, seed=11)
    x = O.bench_coeffs(O.SHAPE_INDEX[shape], P, el.nm, n, seed=11)
    blk.set_elements(x[None])
    eb, nt, _ = blk.basis.launch_config(0, deformed=False)
    assert n > 4 * eb  # several tiles
    for lam in (0.0, 1.7):
        got = sk.helmholtz_apply(blk, lam).get_elements()[0]
        assert _err(got, O.helmholtz_coll(el, geo, x, lam)) <= TOL, (lam, eb, nt)


@pytest.mark.parametrize("shape", SHAPES)
def test_regular_factors_shared_by_two_orders(sk, shape):
    """One regular GeometricFactors serving bases of two orders (the
    reference's affine factors do not depend on the order): each order gets
    its own payload (lane widths differ), results match the oracle."""
    n = 40
    from paper_2604_04644_b200.geometry import synthetic_affine_vertices

    verts = synthetic_affine_vertices(sk.Shape(shape), n, 4)
    fac = sk.make_affine_block(sk.Shape(shape), verts)
    geo = O.affine_geometry(shape, verts)
    for P in (1, 3, 2):
        el = O.element(shape, P)
        b = sk.build_shape_basis(sk.Shape(shape), P)
        blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
        x = O.bench_coeffs(O.SHAPE_INDEX[shape], P, el.nm, n, seed=P)
        blk.set_elements(x[None])
        assert _err(sk.helmholtz_apply_noncoll(blk, 1.0).get_elements()[0], O.helmholtz_noncoll(el, geo, x, 1.0)) <= TOL
        assert _err(sk.helmholtz_apply(blk, 1.0).get_elements()[0], O.helmholtz_coll(el, geo, x, 1.0)) <= TOL
        pb = blk.like(sk.FieldState.PHYS)
        y = np.random.default_rng(P).uniform(-1, 1, (el.nq, n))
        pb.set_elements(y[None])
        assert _err(sk.phys_deriv(pb).get_elements(), O.phys_deriv(el, geo, y)) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
def test_padding_lanes_stay_zero(sk, shape):
    """Padded lanes of the lane-major layout are written as zeros
    (reference acceptance criterion 9)."""
    n, w = 13, 8
    blk = _block(sk, shape, 3, True, n, 1, w)
    el = O.element(shape, 3)
    blk.set_elements(O.bench_coeffs(O.SHAPE_INDEX[shape], 3, el.nm, n)[None])
    out = blk.like(sk.FieldState.COEFF)
    raw = out.host(sk.AccessQualifier.WRITE_ONLY)
    raw[...] = 7.0  # poison, including the padded lanes
    sk.helmholtz_apply(blk, 1.0, out=out)
    flat = out.host()[0].transpose(1, 0, 2).reshape(el.nm, -1)
    assert np.all(flat[:, n:] == 0.0)
    assert np.all(np.isfinite(flat[:, :n]))


@pytest.mark.parametrize("shape", SHAPES)
def test_device_geometry_builder(sk, shape):
    """Device iso-parametric metric == oracle restatement of
    deformed_factors_from_coords on the same seeded mesh."""
    P, n = 4, 9
    b = sk.build_shape_basis(sk.Shape(shape), P)
    fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, n, seed=2)
    geo = O.synthetic_geometry(O.element(shape, P), True, n, seed=2)
    # w|J| is well conditioned; dxi near a collapsed vertex is not (a 1-ulp
    # change of the coordinates moves the reference's own dxi by ~4e-13 at
    # P=4), so dxi gets that headroom
    assert _err(fac.dxi_dx, geo.dxi) <= 1e-11
    assert _err(fac.jac, geo.jac) <= 1e-13
    # coords route
    from oracle.geom import deformed_coords

    coords = deformed_coords(O.element(shape, P), O.deformation_params(n, 2))
    fac2 = sk.deformed_factors_from_coords(b, coords)
    assert _err(fac2.dxi_dx, geo.dxi) <= 1e-11
    assert _err(fac2.jac, geo.jac) <= 1e-13


def test_memory_region_transfer_counting(sk):
    """Repeated applies do not re-transfer (acceptance criterion 6)."""
    blk = _block(sk, "hex", 2, True, 10, 0, 1)
    el = O.element("hex", 2)
    blk.set_elements(O.bench_coeffs(2, 2, el.nm, 10)[None])
    out = blk.like(sk.FieldState.COEFF)
    for _ in range(3):
        sk.helmholtz_apply(blk, 1.0, out=out)
    assert blk.region.transfer_count == 1
    out.get_elements()
    assert out.region.transfer_count == 1


def test_large_block_properties(sk):
    """At the bench size (2^20 tets, P=4): sampled elements match the oracle
    exactly, and the operator is symmetric (u.Hv == v.Hu, size-independent)."""
    import torch

    n, P = 1 << 20, 4
    el = O.element("tet", P)
    b = sk.build_shape_basis(sk.Shape.TET, P)
    fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, n, seed=0)
    blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
    x = O.bench_coeffs(O.SHAPE_INDEX["tet"], P, el.nm, n, seed=0)
    blk.set_elements(x[None])
    hx = sk.helmholtz_apply(blk, 1.0).get_elements()[0]
    idx = np.array([0, 1, 777, 65535, 65536, 999_999, n - 1])
    params = np.concatenate([O.deformation_params(1, 0, first=int(e)) for e in idx])
    from oracle.geom import deformed_coords

    geo = O.deformed_geometry_from_coords(el, deformed_coords(el, params))
    assert _err(hx[:, idx], O.helmholtz_coll(el, geo, x[:, idx], 1.0)) <= TOL
    y = np.random.default_rng(1).uniform(-1, 1, x.shape)
    blk2 = blk.like(sk.FieldState.COEFF)
    blk2.set_elements(y[None])
    hy = sk.helmholtz_apply(blk2, 1.0).get_elements()[0]
    a, c = np.sum(x * hy), np.sum(y * hx)
    assert abs(a - c) <= 1e-12 * np.sum(np.abs(x * hy))
    del torch


@pytest.mark.parametrize("shape,P,n", [("tet", 4, 1 << 20), ("hex", 8, 1 << 16), ("pyr", 6, 1 << 18), ("prism", 10, 1 << 14)])
def test_every_element_at_scale_by_independent_routes(sk, shape, P, n):
    """Full-size blocks, EVERY element checked: the collocated kernel (Alg. 6)
    against the non-collocated one (Alg. 5: derivative-table sum
    factorisation, a different set of sweeps) -- the reference's own
    coll == noncoll identity (test_acceptance.py:129-142) -- and the
    sum-factorised mass against the StdMat/DMMA mass where one exists.  A
    skipped, duplicated or misplaced element anywhere in the block would
    break the per-element comparison (sampled oracle checks and the
    symmetry identity cannot see that)."""
    import os

    b = sk.build_shape_basis(sk.Shape(shape), P)
    fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, n, seed=3)
    blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
    xd = blk.device(sk.AccessQualifier.WRITE_ONLY)
    xd.uniform_(-1.0, 1.0)
    coll = sk.helmholtz_apply(blk, 1.0).device().view(n, -1)
    nonc = sk.helmholtz_apply_noncoll(blk, 1.0).device().view(n, -1)
    per_el = ((coll - nonc).abs().amax(dim=1) / coll.abs().amax(dim=1)).max().item()
    assert per_el <= 1e-12, per_el
    assert (coll.abs().amax(dim=1) > 0).all()  # no element left unwritten
    old = os.environ.get("SK_MASS_DENSE")
    try:
        os.environ["SK_MASS_DENSE"] = "0"
        ms = sk.mass_apply(blk).device().view(n, -1).clone()
        os.environ["SK_MASS_DENSE"] = "1"
        md = sk.mass_apply(blk).device().view(n, -1)
    finally:
        if old is None:
            os.environ.pop("SK_MASS_DENSE", None)
        else:
            os.environ["SK_MASS_DENSE"] = old
    assert ((ms - md).abs().amax(dim=1) / ms.abs().amax(dim=1)).max().item() <= 1e-12


@pytest.mark.parametrize("direct", [True, False])
@pytest.mark.parametrize("ramp", ["1", "0"])
@pytest.mark.parametrize("shape,P,width,ncomp", [("tet", 4, 1, 1), ("hex", 3, 8, 2), ("prism", 5, 3, 1)])
def test_streamed_host_apply(sk, monkeypatch, shape, P, width, ncomp, ramp, direct):
    """Host-resident input >= STREAM_MIN_BYTES: the chunk-pipelined
    H2D / kernel / D2H path (sk_apply_streamed_ex) matches the
    device-resident path bit for bit, with ragged chunks, interleave widths
    and components, ramped (default) and uniform chunk schedules, and with
    the kernels storing straight into the pinned host buffer (direct output)
    or through a D2H stage; both regions count one transfer; with a D2H
    stage the output is live in both spaces, with direct output on the host
    only (the device copy comes from one more transfer)."""
    from paper_2604_04644_b200 import operators as ops
    from paper_2604_04644_b200.field_block import MemorySpace

    monkeypatch.setenv("SK_STREAM_RAMP", ramp)
    monkeypatch.setattr(ops, "STREAM_DIRECT_OUT", direct)

    b = sk.build_shape_basis(sk.Shape(shape), P)
    n = ops.STREAM_MIN_BYTES // (8 * b.n_modes * ncomp) + 777
    fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, n, seed=4)
    x = np.random.default_rng(5).uniform(-1, 1, (ncomp, b.n_modes, n))
    for kind in ("helm", "stiff", "mass"):
        blk = sk.Block(b, fac, sk.FieldState.COEFF, ncomp, width)
        blk.set_elements(x)
        ref = sk.Block(b, fac, sk.FieldState.COEFF, ncomp, width)
        ref.set_elements(x)
        ref.device()  # device-resident: plain path
        fn = {"helm": lambda bl: sk.helmholtz_apply(bl, 1.5), "stiff": lambda bl: sk.helmholtz_apply(bl, 0.0),
              "mass": lambda bl: sk.mass_apply(bl)}[kind]
        n0 = ops._lib.launch_count()
        out = fn(blk)
        assert ops._lib.launch_count() - n0 > 1  # chunked launches
        assert blk.region.transfer_count == 1 and out.region.transfer_count == 1
        want = fn(ref).get_elements()
        got = out.get_elements()
        assert out.region.transfer_count == 1
        assert np.array_equal(got, want), kind
        assert out.region.valid(MemorySpace.DEVICE) is (not direct)
        # the device copy of the streamed output is (or becomes) identical
        assert np.array_equal(out.device().cpu().numpy(), out.host().reshape(-1))
        assert out.region.transfer_count == (2 if direct else 1)


@pytest.mark.parametrize("shape,P,n,width", [("hex", 9, 2500, 1), ("pyr", 3, 40001, 1), ("pyr", 3, 30011, 3)])
def test_persistent_tiles_at_scale(sk, shape, P, n, width):
    """(shape, P) launched as persistent CTAs (sk_tune.h kPersist): enough
    elements that every CTA strides over several tiles, exercising the
    register-staged next tile and the in-body geometry prefetch; compared
    with the oracle on every element."""
    el = O.element(shape, P)
    geo = O.synthetic_geometry(el, True, n, seed=7)
    blk = _block_from(sk, shape, P, geo, width)
    x = np.random.default_rng(3).uniform(-1, 1, (el.nm, n))
    blk.set_elements(x[None])
    blk.device()
    got = sk.helmholtz_apply(blk, 0.7).get_elements()[0]
    assert _err(got, O.helmholtz_coll(el, geo, x, 0.7)) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("width", [1, 8])
def test_dense_dmma_mass(sk, monkeypatch, shape, P, width):
    """StdMat mass on the FP64 tensor cores (sk_dense.cuh, forced with
    SK_MASS_DENSE=1) against the oracle's sum-factorised mass on every
    element: ragged 8-element groups, interleave widths, two components,
    both geometry classes (regular: |J| M_ref)."""
    monkeypatch.setenv("SK_MASS_DENSE", "1")
    n = 157
    el = O.element(shape, P)
    for deformed in (False, True):
        blk = _block(sk, shape, P, deformed, n, 9, width, ncomp=2)
        geo = O.synthetic_geometry(el, deformed, n, seed=9)
        x = np.random.default_rng(P).uniform(-1, 1, (2, el.nm, n))
        blk.set_elements(x)
        got = sk.mass_apply(blk)
        for c in range(2):
            assert _err(got.get_elements()[c], O.mass(el, geo, x[c])) <= TOL, (deformed, c)
        # padded lanes of the last group stay zero
        h = got.host().reshape(2, -1, el.nm, width)
        if n % width:
            assert not np.any(h[:, -1, :, n % width:])


def test_dense_mass_streamed_and_forced_off(sk, monkeypatch):
    """The streamed host path takes the dense kernel too; SK_MASS_DENSE=0
    (sum factorisation) gives the same result to 1e-12."""
    from paper_2604_04644_b200 import operators as ops

    b = sk.build_shape_basis(sk.Shape.TET, 2)
    n = ops.STREAM_MIN_BYTES // (8 * b.n_modes) + 333
    fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, n, seed=2)
    x = np.random.default_rng(1).uniform(-1, 1, (1, b.n_modes, n))
    res = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("SK_MASS_DENSE", flag)
        blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
        blk.set_elements(x)
        res[flag] = sk.mass_apply(blk).get_elements()
    assert _err(res["1"], res["0"]) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [2, 5, 8, 10])
def test_staged_helmholtz_matches_fused(sk, shape, P):
    """Staged collocated Helmholtz (bwd -> quadrature-point kernel ->
    unweighted B^T over element chunks, sk_helmholtz_apply_staged) against
    the oracle and the fused kernel: several chunks, a ragged last chunk,
    two components, interleave width 8, lam 0 and > 0."""
    n = 211
    el = O.element(shape, P)
    geo = O.synthetic_geometry(el, True, n, seed=13)
    blk = _block_from(sk, shape, P, geo, 8, ncomp=2)
    x = np.random.default_rng(P).uniform(-1, 1, (2, el.nm, n))
    blk.set_elements(x)
    for lam in (0.0, 0.9):
        got = sk.helmholtz_apply_staged(blk, lam, chunk_elements=48).get_elements()
        fused = sk.helmholtz_apply(blk, lam).get_elements()
        for c in range(2):
            assert _err(got[c], O.helmholtz_coll(el, geo, x[c], lam)) <= TOL, (lam, c)
        assert _err(got, fused) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 6])
def test_dense_dmma_regular_helmholtz(sk, monkeypatch, shape, P):
    """Regular-geometry collocated Helmholtz and stiffness by StdMat on the
    FP64 tensor cores (seven element-independent matrices, forced with
    SK_HELM_DENSE=1 wherever the fragments fit) against the oracle on every
    element; where no dense kernel exists the sum-factorised path runs."""
    monkeypatch.setenv("SK_HELM_DENSE", "1")
    n = 157
    el = O.element(shape, P)
    geo = O.synthetic_geometry(el, False, n, seed=12)
    for width in (1, 8):
        blk = _block(sk, shape, P, False, n, 12, width, ncomp=2)
        x = np.random.default_rng(P).uniform(-1, 1, (2, el.nm, n))
        blk.set_elements(x)
        for lam in (0.0, 1.7):
            got = sk.helmholtz_apply(blk, lam).get_elements()
            for c in range(2):
                assert _err(got[c], O.helmholtz_coll(el, geo, x[c], lam)) <= TOL, (width, lam, c)


QCASES = [("hex", 2, (5, 4, 6)), ("prism", 3, (6, 5, 6)), ("pyr", 2, (5, 6, 4)), ("tet", 3, (6, 5, 6)), ("tet", 1, (3, 4, 2))]


@pytest.mark.parametrize("shape,P,q", QCASES)
@pytest.mark.parametrize("gname", ["regular", "deformed"])
def test_quadrature_override_against_reference(sk, shape, P, q, gname):
    """build_shape_basis(shape, P, qpoints) above the default counts (the
    run-time-size device path): every operator against the reference's own
    outputs on the reference's factors (tests/golden/operators_qpoints.npz),
    and the device geometry builder against the reference's factors."""
    from conftest import GOLDEN
    import os

    g = np.load(os.path.join(GOLDEN, "operators_qpoints.npz"))
    k = f"{shape}_P{P}_q{''.join(map(str, q))}_{gname}"
    b = sk.build_shape_basis(sk.Shape(shape), P, q)
    assert b.qcounts == q and b.generic
    deformed = gname == "deformed"
    gcls = sk.GeometryClass.DEFORMED if deformed else sk.GeometryClass.REGULAR
    fac = sk.GeometricFactors(gcls, sk.Shape(shape), 2, dxi_dx=g[f"{k}_dxi"], jac=g[f"{k}_jac"])
    blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 2)
    blk.set_elements(g[f"{k}_x"][None])
    n0 = sk._lib.launch_count() if hasattr(sk, "_lib") else None
    for lam in (0.0, 1.0):
        assert _err(sk.helmholtz_apply(blk, lam).get_elements()[0], g[f"{k}_helm_{lam}"]) <= TOL, lam
    assert _err(sk.helmholtz_apply_noncoll(blk, 1.0).get_elements()[0], g[f"{k}_helmnc_1.0"]) <= TOL
    assert _err(sk.mass_apply(blk).get_elements()[0], g[f"{k}_mass"]) <= TOL
    assert _err(sk.bwd_trans(blk).get_elements()[0], g[f"{k}_bwd"]) <= TOL
    pb = blk.like(sk.FieldState.PHYS)
    pb.set_elements(g[f"{k}_y"][None])
    assert _err(sk.iproduct_wrt_base(pb).get_elements()[0], g[f"{k}_iprod"]) <= TOL
    assert _err(sk.phys_deriv(pb).get_elements(), g[f"{k}_dphys"]) <= TOL
    vb = blk.like(sk.FieldState.PHYS, 3)
    vb.set_elements(g[f"{k}_v"])
    assert _err(sk.iproduct_wrt_deriv_base(vb).get_elements()[0], g[f"{k}_ipderiv"]) <= TOL
    if deformed:
        syn = sk.make_synthetic_factors(b, gcls, 2, seed=5)
        assert _err(syn.jac, g[f"{k}_jac"]) <= 1e-13
        # operators on the device-built factors of many elements vs the oracle
        n = 37
        el = O.element(shape, P, q)
        geo = O.synthetic_geometry(el, True, n, seed=7)
        cb = sk.Block(b, sk.make_synthetic_factors(b, gcls, n, seed=7), sk.FieldState.COEFF, 1, 1)
        x = np.random.default_rng(3).uniform(-1, 1, (el.nm, n))
        cb.set_elements(x[None])
        assert _err(sk.helmholtz_apply(cb, 0.8).get_elements()[0], O.helmholtz_coll(el, geo, x, 0.8)) <= TOL
    del n0


def test_quadrature_override_validation(sk):
    with pytest.raises(ValueError):
        sk.build_shape_basis(sk.Shape.TET, 3, (5, 3, 4))  # below the default (5, 4, 4)
    assert not sk.build_shape_basis(sk.Shape.TET, 3, (5, 4, 4)).generic  # the default itself


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [1, 3, 6, 10])
def test_recomputed_metric_helmholtz(sk, shape, P):
    """Helmholtz with the metric recomputed per chunk from the deformation
    parameters (sk_helmholtz_apply_params) against the oracle on the same
    seeded deformed geometry, and bitwise against the streamed-payload
    kernel: several chunks, a ragged last chunk, two components, interleave
    width 8, lam 0 and > 0."""
    n = 203
    el = O.element(shape, P)
    blk = _block(sk, shape, P, True, n, 11, 8, ncomp=2)
    geo = O.synthetic_geometry(el, True, n, seed=11)
    x = np.random.default_rng(P).uniform(-1, 1, (2, el.nm, n))
    blk.set_elements(x)
    for lam in (0.0, 1.3):
        got = sk.helmholtz_apply_params(blk, lam, chunk_elements=48).get_elements()
        streamed = sk.helmholtz_apply(blk, lam).get_elements()
        assert np.array_equal(got, streamed), lam
        for c in range(2):
            assert _err(got[c], O.helmholtz_coll(el, geo, x[c], lam)) <= TOL, (lam, c)
    blk_default_chunk = sk.helmholtz_apply_params(blk, 0.5).get_elements()
    assert np.array_equal(blk_default_chunk, sk.helmholtz_apply(blk, 0.5).get_elements())


def test_recomputed_metric_errors(sk):
    b = sk.build_shape_basis(sk.Shape.TET, 3)
    reg = sk.Block(b, sk.make_synthetic_factors(b, sk.GeometryClass.REGULAR, 10, seed=0), sk.FieldState.COEFF, 1, 1)
    with pytest.raises(sk.UnsupportedStrategyError):
        sk.helmholtz_apply_params(reg, 1.0)
    blk = _block(sk, "tet", 3, True, 40, 0, 1)
    with pytest.raises(ValueError):
        sk.helmholtz_apply_params(blk, -1.0)
    with pytest.raises(ValueError):
        sk.helmholtz_apply_params(blk, 1.0, chunk_elements=24)  # not a multiple of 16


@pytest.mark.parametrize("shape,P,n", [("tet", 4, 50021), ("pyr", 3, 40003), ("prism", 5, 30011), ("hex", 3, 30001)])
def test_mass_at_scale(sk, shape, P, n):
    """Deformed mass over several waves of persistent CTAs (every CTA
    strides over many tiles: the TMA-fed kernel's double-buffered
    coefficient blocks and per-tile W copies, kMassTma), two components
    (the second one's offset is not 16-byte aligned for odd n * n_modes:
    register path for it), interleave width 1, ragged last tile; compared
    with the oracle on every element."""
    el = O.element(shape, P)
    geo = O.synthetic_geometry(el, True, n, seed=21)
    blk = _block_from(sk, shape, P, geo, 1, ncomp=2)
    x = np.random.default_rng(7).uniform(-1, 1, (2, el.nm, n))
    blk.set_elements(x)
    blk.device()
    got = sk.mass_apply(blk).get_elements()
    for c in range(2):
        assert _err(got[c], O.mass(el, geo, x[c])) <= TOL, c


@pytest.mark.parametrize("n", [1, 3, 17, 130])
@pytest.mark.parametrize("width", [1, 4])
def test_tma_paths_small_and_ragged(sk, n, width):
    """The TMA-fed kernels at the cells they are on for (mass pyr P=3, tet
    P=4; Helmholtz hex P=6, pyr P=5; regular tet P=9): a handful of
    elements (fewer tiles than CTAs, a ragged last tile, the register path
    for interleave width 4 and for an unaligned second component) against
    the oracle."""
    for shape, P, op, deformed in (("pyr", 3, "mass", True), ("tet", 4, "mass", True), ("hex", 6, "helm", True),
                                   ("pyr", 5, "helm", True), ("tet", 9, "helm", False)):
        el = O.element(shape, P)
        geo = O.synthetic_geometry(el, deformed, n, seed=n)
        blk = _block_from(sk, shape, P, geo, width, ncomp=2)
        x = np.random.default_rng(n).uniform(-1, 1, (2, el.nm, n))
        blk.set_elements(x)
        if op == "mass":
            got = sk.mass_apply(blk).get_elements()
            want = [O.mass(el, geo, x[c]) for c in range(2)]
        else:
            got = sk.helmholtz_apply(blk, 0.8).get_elements()
            want = [O.helmholtz_coll(el, geo, x[c], 0.8) for c in range(2)]
        for c in range(2):
            assert _err(got[c], want[c]) <= TOL, (shape, P, op, c)
