"""Elemental operators on the device: the drop-in for ``speckern.operators``.

Same functions, signatures, error types and output-block semantics as the
reference (operators.py:34-776).  Every call runs the sm_100a kernels of
``libsk200.so`` through the C ABI on the current CUDA stream; there is no CPU
path.  The strategy argument accepts ``SUM_FAC_TOP`` -- the reserved
"sum-factorisation threaded on output points" slot the reference keeps for
exactly this device work-group variant (operators.py:57, 416-420) -- and the
reference default ``SUM_FAC`` (same sum-factorised algorithm, so caller code
runs unchanged).  The dense-matrix strategies are CPU layouts and raise
``UnsupportedStrategyError``.
"""

from __future__ import annotations

import ctypes
import enum
import os

from paper_2604_04644_b200 import _lib
from paper_2604_04644_b200.field_block import AccessQualifier, Block, Field, FieldState
from paper_2604_04644_b200.geometry import GeometryClass
from paper_2604_04644_b200.shapes import Shape, mode_count, quad_point_counts

__all__ = [
    "Strategy",
    "OperatorKind",
    "UnsupportedStrategyError",
    "FieldStateError",
    "bwd_trans",
    "iproduct_wrt_base",
    "phys_deriv",
    "iproduct_wrt_deriv_base",
    "mass_apply",
    "helmholtz_apply_noncoll",
    "helmholtz_apply_coll",
    "helmholtz_apply",
    "helmholtz_apply_staged",
    "helmholtz_apply_params",
    "stiffness_apply",
    "apply_operator",
    "apply_to_field",
    "operator_flops",
    "operator_bytes",
]


class Strategy(enum.Enum):
    STD_MAT = "stdmat"
    STD_MAT_GROUPED = "stdmat_grouped"
    SUM_FAC = "sumfac"
    SUM_FAC_TOP = "sumfac_top"


class OperatorKind(enum.Enum):
    BWD_TRANS = "bwdtrans"
    IPRODUCT_WRT_BASE = "iproduct"
    PHYS_DERIV = "physderiv"
    IPRODUCT_WRT_DERIV_BASE = "iproduct_deriv"
    MASS = "mass"
    HELMHOLTZ_NONCOLL = "helmholtz_noncoll"
    HELMHOLTZ_COLL = "helmholtz_coll"


class UnsupportedStrategyError(ValueError):
    """Strategy (or shape/order) not implemented on the device path."""


class FieldStateError(ValueError):
    """Block is in the wrong coefficient/physical state for an operator."""


_DEVICE_STRATEGIES = (Strategy.SUM_FAC_TOP, Strategy.SUM_FAC)


def _check_strategy(strategy: Strategy) -> None:
    if strategy not in _DEVICE_STRATEGIES:
        raise UnsupportedStrategyError(
            f"strategy {getattr(strategy, 'value', strategy)!r} is a CPU dense-matrix layout; "
            "the device path implements the sum-factorised work-group strategy (sumfac_top)"
        )


def _require_state(block: Block, state: FieldState, op: str) -> None:
    """operators.py:530-534."""
    if block.state is not state:
        raise FieldStateError(f"{op} expects a {state.value}-state block, got {block.state.value}")


def _out_block(block: Block, out: Block | None, state: FieldState, n_components: int) -> Block:
    """operators.py:537-548."""
    if out is None:
        return block.like(state, n_components)
    if out.state is not state or out.n_components != n_components:
        raise FieldStateError(f"output block must be {state.value}-state with {n_components} component(s)")
    if out.basis is not block.basis or out.interleave_width != block.interleave_width:
        raise ValueError("output block layout does not match the input block")
    return out


def _p(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream() -> ctypes.c_void_p:
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _geo(block: Block) -> int:
    return _lib.SK_GEO_DEFORMED if block.geometry_class is GeometryClass.DEFORMED else _lib.SK_GEO_REGULAR


#: inputs at least this large (bytes) that live only in host memory are
#: applied chunk-pipelined (H2D / kernel / D2H overlapped, sk_apply_streamed);
#: smaller ones take the plain transfer-then-apply path
STREAM_MIN_BYTES = 32 << 20
#: elements per streamed chunk (0: the library default, a ramped schedule)
STREAM_CHUNK_ELEMENTS = 0
#: SK_STREAM_DIRECT=1: the kernels store the result straight into the pinned
#: host buffer (SK_STREAM_DIRECT_OUT) and the output stays host-only; off by
#: default -- it measured within 1 % of the D2H stage on B200 (the two PCIe
#: directions do not overlap fully there) and the D2H stage
#: leaves the result live on both sides
STREAM_DIRECT_OUT = os.environ.get("SK_STREAM_DIRECT", "0") == "1"


def _streamed(block: Block, out: Block, op: int, pay, lam: float) -> bool:
    """Host-resident input: run the operator pipelined over element chunks,
    leaving input and output live in both spaces (one transfer each, as the
    plain path would count them).  Returns False when not applicable."""
    reg = block.region
    if not reg.host_resident() or out is block or reg.length * 8 < STREAM_MIN_BYTES or block.basis.generic:
        return False
    import torch

    h_in, d_in = reg.buffers()
    h_out, d_out = out.region.buffers()
    flags = _lib.SK_STREAM_DIRECT_OUT if STREAM_DIRECT_OUT else 0
    _lib.check(
        _lib.load().sk_apply_streamed_ex(
            block.basis.handle, op, _geo(block), block.n_elements, block.interleave_width, block.n_components,
            _p(h_in), _p(d_in), _p(pay), float(lam), _p(d_out), _p(h_out), STREAM_CHUNK_ELEMENTS, flags, _stream(),
        ),
        "sk_apply_streamed_ex",
    )
    ev = torch.cuda.Event()
    ev.record()
    reg.mark_streamed(ev, wrote_host=False)
    if flags:
        out.region.mark_host_written(ev)
    else:
        out.region.mark_streamed(ev, wrote_host=True)
    return True


def bwd_trans(block: Block, strategy: Strategy = Strategy.SUM_FAC_TOP, out: Block | None = None) -> Block:
    """u = B uhat (operators.py:551-561)."""
    _check_strategy(strategy)
    _require_state(block, FieldState.COEFF, "bwd_trans")
    out = _out_block(block, out, FieldState.PHYS, block.n_components)
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    _lib.check(
        _lib.load().sk_bwd_trans(
            block.basis.handle, block.n_elements, block.interleave_width, block.n_components, _p(xin), _p(xout), _stream()
        ),
        "sk_bwd_trans",
    )
    return out


def iproduct_wrt_base(block: Block, strategy: Strategy = Strategy.SUM_FAC_TOP, out: Block | None = None) -> Block:
    """fhat = B^T W u (operators.py:564-574)."""
    _check_strategy(strategy)
    _require_state(block, FieldState.PHYS, "iproduct_wrt_base")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    pay = block.payload(_lib.SK_PAYLOAD_W)
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    _lib.check(
        _lib.load().sk_iproduct_wrt_base(
            block.basis.handle, _geo(block), block.n_elements, block.interleave_width, block.n_components,
            _p(xin), _p(pay), _p(xout), _stream(),
        ),
        "sk_iproduct_wrt_base",
    )
    return out


def phys_deriv(block: Block, out: Block | None = None) -> Block:
    """Cartesian derivatives at quadrature points (operators.py:577-596)."""
    _require_state(block, FieldState.PHYS, "phys_deriv")
    if block.n_components != 1:
        raise ValueError("phys_deriv expects a single-component block")
    out = _out_block(block, out, FieldState.PHYS, 3)
    pay = block.payload(_lib.SK_PAYLOAD_DERIV)
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    _lib.check(
        _lib.load().sk_phys_deriv(
            block.basis.handle, _geo(block), block.n_elements, block.interleave_width, _p(xin), _p(pay), _p(xout), _stream()
        ),
        "sk_phys_deriv",
    )
    return out


def iproduct_wrt_deriv_base(
    block: Block, strategy: Strategy = Strategy.SUM_FAC_TOP, out: Block | None = None
) -> Block:
    """fhat = sum_d (D_d B)^T W v_d (operators.py:599-619)."""
    _check_strategy(strategy)
    _require_state(block, FieldState.PHYS, "iproduct_wrt_deriv_base")
    if block.n_components != 3:
        raise ValueError(f"iproduct_wrt_deriv_base expects 3 components, got {block.n_components}")
    out = _out_block(block, out, FieldState.COEFF, 1)
    pay = block.payload(_lib.SK_PAYLOAD_W)
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    _lib.check(
        _lib.load().sk_iproduct_wrt_deriv_base(
            block.basis.handle, _geo(block), block.n_elements, block.interleave_width, _p(xin), _p(pay), _p(xout), _stream()
        ),
        "sk_iproduct_wrt_deriv_base",
    )
    return out


def mass_apply(block: Block, strategy: Strategy = Strategy.SUM_FAC_TOP, out: Block | None = None) -> Block:
    """M uhat = B^T W B uhat (operators.py:622-633)."""
    _check_strategy(strategy)
    _require_state(block, FieldState.COEFF, "mass_apply")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    pay = block.payload(_lib.SK_PAYLOAD_W)
    if _streamed(block, out, _lib.SK_STREAM_MASS, pay, 0.0):
        return out
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    _lib.check(
        _lib.load().sk_mass_apply(
            block.basis.handle, _geo(block), block.n_elements, block.interleave_width, block.n_components,
            _p(xin), _p(pay), _p(xout), _stream(),
        ),
        "sk_mass_apply",
    )
    return out


def _helmholtz(block: Block, lam: float, form: int, out: Block | None, name: str) -> Block:
    _require_state(block, FieldState.COEFF, name)
    if lam < 0.0:
        raise ValueError(f"reaction coefficient must be nonnegative, got {lam}")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    pay = block.payload(_lib.SK_PAYLOAD_HELMHOLTZ if form == _lib.SK_FORM_COLL else _lib.SK_PAYLOAD_HELMHOLTZ_NC)
    sop = _lib.SK_STREAM_HELMHOLTZ if form == _lib.SK_FORM_COLL else _lib.SK_STREAM_HELMHOLTZ_NC
    if _streamed(block, out, sop, pay, lam):
        return out
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    _lib.check(
        _lib.load().sk_helmholtz_apply(
            block.basis.handle, _geo(block), form, block.n_elements, block.interleave_width, block.n_components,
            _p(xin), _p(pay), float(lam), _p(xout), _stream(),
        ),
        "sk_helmholtz_apply",
    )
    return out


#: L2 budget of the staged variant's two quadrature-point work buffers (bytes)
STAGED_WORK_BYTES = 48 << 20


def helmholtz_apply_staged(block: Block, lam: float, out: Block | None = None, chunk_elements: int = 0) -> Block:
    """Collocated Helmholtz (Alg. 6) as three kernels per element chunk --
    BwdTrans, the quadrature-point kernel, the unweighted B^T -- with the
    intermediates in L2-sized work buffers (sk_helmholtz_apply_staged).  Same
    result as ``helmholtz_apply_coll``; kept for the fused-vs-staged
    comparison.  Deformed geometry only."""
    import torch

    _require_state(block, FieldState.COEFF, "helmholtz_apply_staged")
    if lam < 0.0:
        raise ValueError(f"reaction coefficient must be nonnegative, got {lam}")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    pay = block.payload(_lib.SK_PAYLOAD_HELMHOLTZ)
    W = block.interleave_width
    unit = 16
    while unit % W:
        unit += 16
    nq = block.basis.n_points
    chunk = chunk_elements or max(unit, STAGED_WORK_BYTES // (16 * nq) // unit * unit)
    chunk = min(chunk, -(-block.padded_elements // unit) * unit)
    work = torch.empty(2 * chunk * nq, dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    _lib.check(
        _lib.load().sk_helmholtz_apply_staged(
            block.basis.handle, _geo(block), block.n_elements, W, block.n_components, _p(xin), _p(pay), float(lam),
            _p(xout), _p(work), chunk, _stream(),
        ),
        "sk_helmholtz_apply_staged",
    )
    return out


#: L2 budget of the recomputed-metric variant's per-chunk payload (bytes)
PARAMS_WORK_BYTES = 48 << 20


def helmholtz_apply_params(block: Block, lam: float, out: Block | None = None, chunk_elements: int = 0,
                           check: bool = True) -> Block:
    """Collocated Helmholtz (Alg. 6) with the metric recomputed on the device
    per element chunk from the block's deformation parameters
    (sk_helmholtz_apply_params; SURVEY H3 option (c)): HBM traffic 8(2 NP +
    12) bytes per element instead of 8(2 NP + 7 NQ).  Same result as
    ``helmholtz_apply_coll`` on the same factors.  Needs a deformed block
    whose factors are held as parameters (``make_synthetic_factors``);
    ``check`` counts degenerate points (one stream synchronisation)."""
    import torch

    from paper_2604_04644_b200.geometry import DegenerateElementError

    _require_state(block, FieldState.COEFF, "helmholtz_apply_params")
    if lam < 0.0:
        raise ValueError(f"reaction coefficient must be nonnegative, got {lam}")
    f = block.factors
    if not f.deformed or f.params is None:
        raise UnsupportedStrategyError("helmholtz_apply_params needs deformed factors held as deformation parameters")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    W = block.interleave_width
    unit = 16
    while unit % W:
        unit += 16
    lib = _lib.load()
    per = ctypes.c_int64()
    _lib.check(lib.sk_payload_size(block.basis.handle, _lib.SK_GEO_DEFORMED, _lib.SK_PAYLOAD_HELMHOLTZ, unit,
                                   ctypes.byref(per)), "sk_payload_size")
    per_el = per.value // unit
    chunk = chunk_elements or max(unit, PARAMS_WORK_BYTES // (8 * per_el) // unit * unit)
    chunk = min(chunk, -(-block.padded_elements // unit) * unit)
    dev = torch.device("cuda", torch.cuda.current_device())
    work = torch.empty(chunk * per_el, dtype=torch.float64, device=dev)
    prm = f.device_params(dev)
    xin = block.device(AccessQualifier.READ_ONLY)
    xout = out.device(AccessQualifier.WRITE_ONLY)
    bad = ctypes.c_int64()
    _lib.check(
        lib.sk_helmholtz_apply_params(
            block.basis.handle, block.n_elements, W, block.n_components, _p(xin), _p(prm), float(lam), _p(xout),
            _p(work), chunk, ctypes.byref(bad) if check else None, _stream(),
        ),
        "sk_helmholtz_apply_params",
    )
    if bad.value:
        raise DegenerateElementError(f"{bad.value} quadrature points with nonpositive Jacobian")
    return out


def helmholtz_apply_noncoll(
    block: Block, lam: float, strategy: Strategy = Strategy.SUM_FAC_TOP, out: Block | None = None
) -> Block:
    """Alg. 5 pipeline (operators.py:636-667)."""
    _check_strategy(strategy)
    return _helmholtz(block, lam, _lib.SK_FORM_NONCOLL, out, "helmholtz_apply_noncoll")


def helmholtz_apply_coll(
    block: Block, lam: float, strategy: Strategy = Strategy.SUM_FAC_TOP, out: Block | None = None
) -> Block:
    """Alg. 6 collocated pipeline (operators.py:670-699)."""
    _check_strategy(strategy)
    return _helmholtz(block, lam, _lib.SK_FORM_COLL, out, "helmholtz_apply_coll")


def helmholtz_apply(
    block: Block,
    lam: float,
    strategy: Strategy = Strategy.SUM_FAC_TOP,
    form: str | None = None,
    out: Block | None = None,
) -> Block:
    """operators.py:702-721; sum-factorised strategies default to ``coll``."""
    if form is None:
        form = "coll"
    if form == "coll":
        return helmholtz_apply_coll(block, lam, strategy, out)
    if form == "noncoll":
        return helmholtz_apply_noncoll(block, lam, strategy, out)
    raise ValueError(f"unknown Helmholtz form: {form!r}")


def stiffness_apply(block: Block, strategy: Strategy = Strategy.SUM_FAC_TOP, out: Block | None = None) -> Block:
    """Weak Laplacian = Helmholtz with lam = 0; the W stream is
    not read."""
    return helmholtz_apply_coll(block, 0.0, strategy, out)


def apply_operator(
    kind: OperatorKind,
    block: Block,
    strategy: Strategy = Strategy.SUM_FAC_TOP,
    lam: float = 1.0,
    out: Block | None = None,
) -> Block:
    """operators.py:724-746."""
    if kind is OperatorKind.BWD_TRANS:
        return bwd_trans(block, strategy, out)
    if kind is OperatorKind.IPRODUCT_WRT_BASE:
        return iproduct_wrt_base(block, strategy, out)
    if kind is OperatorKind.PHYS_DERIV:
        return phys_deriv(block, out)
    if kind is OperatorKind.IPRODUCT_WRT_DERIV_BASE:
        return iproduct_wrt_deriv_base(block, strategy, out)
    if kind is OperatorKind.MASS:
        return mass_apply(block, strategy, out)
    if kind is OperatorKind.HELMHOLTZ_NONCOLL:
        return helmholtz_apply_noncoll(block, lam, strategy, out)
    if kind is OperatorKind.HELMHOLTZ_COLL:
        return helmholtz_apply_coll(block, lam, strategy, out)
    raise ValueError(f"unknown operator kind: {kind!r}")


def apply_to_field(
    kind: OperatorKind,
    field: Field,
    strategy: Strategy = Strategy.SUM_FAC_TOP,
    lam: float = 1.0,
    outs: list | None = None,
    threads: int = 1,
) -> Field:
    """operators.py:749-776.  Blocks are independent; they are enqueued back
    to back on the current stream (``threads`` is accepted for signature
    compatibility: the GPU overlaps the per-block kernels itself)."""
    del threads
    outs = outs if outs is not None else [None] * len(field.blocks)
    return Field([apply_operator(kind, b, strategy, lam, o) for b, o in zip(field.blocks, outs)])


# ---------------------------------------------------------------------------
# algorithmic counters (the roofline denominators)


def _bwd_flops(shape: Shape, P: int) -> int:
    """Sum-factorised B flops per element (operators.py:783-818)."""
    q1, q2, q3 = quad_point_counts(shape, P)
    p1 = P + 1
    ntri = p1 * (p1 + 1) // 2
    if shape is Shape.HEX:
        return 2 * (q1 * p1**3 + q1 * q2 * p1**2 + q1 * q2 * q3 * p1)
    step3 = 2 * q1 * q2 * q3 * p1
    if shape is Shape.PRISM:
        return 2 * q3 * p1 * ntri + 2 * p1 * q2 * p1 * q3 + step3 + 2 * q2 * p1 + 2 * q2 * q3
    if shape is Shape.PYR:
        npyr = p1 * (p1 + 1) * (2 * p1 + 1) // 6
        return 2 * q3 * npyr + 2 * p1 * q2 * p1 * q3 + step3 + 4 * q2 * q3
    if shape is Shape.TET:
        ntet = p1 * (p1 + 1) * (p1 + 2) // 6
        return 2 * q3 * ntet + 2 * q2 * q3 * ntri + step3 + 2 * q3 * P + 2 * q2 * q3 + 8 * q2 * q3
    raise ValueError(f"unsupported shape: {shape!r}")


def operator_flops(kind: OperatorKind, shape: Shape, order: int, strategy: Strategy = Strategy.SUM_FAC_TOP) -> int:
    """Per-element flops of the sum-factorised algorithm, multiply-add = 2
    (operators.py:835-876).  SUM_FAC_TOP reports the same algorithmic count
    as SUM_FAC: the kernels' own savings (G folded into the metric) are not
    credited."""
    _check_strategy(strategy)
    qc = quad_point_counts(shape, order)
    nq = qc[0] * qc[1] * qc[2]
    nm = mode_count(shape, order)
    b = _bwd_flops(shape, order)
    sweep = sum(2 * nq * q for q in qc)
    nnz = {Shape.HEX: 0, Shape.PRISM: 4, Shape.PYR: 5, Shape.TET: 6}[shape]
    metric = 2 * nq * (2 * nnz + 9) + 3 * nq
    if kind is OperatorKind.BWD_TRANS:
        return b
    if kind is OperatorKind.IPRODUCT_WRT_BASE:
        return b + nq
    if kind is OperatorKind.PHYS_DERIV:
        return sweep + metric
    if kind is OperatorKind.IPRODUCT_WRT_DERIV_BASE:
        return 3 * (b + nq) + 2 * nm
    if kind is OperatorKind.MASS:
        return 2 * b + nq
    if kind is OperatorKind.HELMHOLTZ_NONCOLL:
        return 8 * b + metric + nq + 4 * nm
    if kind is OperatorKind.HELMHOLTZ_COLL:
        return 2 * b + 2 * sweep + metric + nq + 5 * nq
    raise ValueError(f"unknown operator kind: {kind!r}")


def operator_bytes(kind: OperatorKind, shape: Shape, order: int, deformed: bool, lam: float = 1.0) -> int:
    """Algorithmic HBM bytes per element: state in/out plus metric data
    (bench.py:175-189); Helmholtz with lam = 0 (stiffness) does not read W."""
    qc = quad_point_counts(shape, order)
    nq = qc[0] * qc[1] * qc[2]
    nm = mode_count(shape, order)
    per = nq if deformed else 1
    if kind is OperatorKind.BWD_TRANS:
        return 8 * (nm + nq)
    if kind is OperatorKind.MASS:
        return 8 * (2 * nm + per)
    if kind in (OperatorKind.HELMHOLTZ_COLL, OperatorKind.HELMHOLTZ_NONCOLL):
        return 8 * (2 * nm + (6 if lam == 0.0 else 7) * per)
    if kind is OperatorKind.IPRODUCT_WRT_BASE:
        return 8 * (nq + nm + per)
    if kind is OperatorKind.PHYS_DERIV:
        return 8 * (nq + 3 * nq + 9 * per)
    if kind is OperatorKind.IPRODUCT_WRT_DERIV_BASE:
        return 8 * (3 * nq + nm + per)
    raise ValueError(f"unknown operator kind: {kind!r}")
