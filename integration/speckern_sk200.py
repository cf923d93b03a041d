"""Reference-side binding: the ctypes stub a speckern maintainer adds to route
``Strategy.SUM_FAC_TOP`` -- the slot the reference reserves for a device
work-group variant (speckern/operators.py:57, 416-420) -- to libsk200.

It takes the reference's own ``Block`` / ``Field`` objects and touches only
the reference's public data model:

* ``block.host(...)`` -- the lane-major region (field_block.py:205-265); the
  C ABI consumes exactly this layout, so a device copy is one memcpy of the
  flat buffer (``sk_copy_h2d`` / ``sk_copy_d2h``);
* ``block.factors.dxi_dx`` / ``block.factors.jac`` (geometry.py:94-116) --
  packed once per block on the device (``sk_payload_pack``) and cached in
  ``block._payload_cache`` beside the reference's own payloads
  (field_block.py:309-321);
* ``list(Shape).index(shape)``, ``basis.order`` and ``basis.qcounts`` -- the
  basis handle (``sk_basis_create_q``; a qpoints override runs the library's
  run-time-size path).

It loads nothing but ``libsk200.so`` (device memory through the library's
own ``sk_device_alloc`` / ``sk_copy_*``; no torch, no cuda-python).  ABI
status codes map onto the reference exception types (operators.py:70-75):
1 -> FieldStateError, 2 -> UnsupportedStrategyError, 3 -> ValueError.

Two ways to wire it:

* explicitly, e.g. in ``speckern/operators.py``::

      def helmholtz_apply_coll(block, lam, strategy=Strategy.SUM_FAC, out=None):
          if strategy is Strategy.SUM_FAC_TOP:
              from speckern import _sk200
              return _sk200.helmholtz_apply_coll(block, lam, strategy, out)
          ...

* or ``install()``: wraps every operator entry point of an imported speckern
  (``bwd_trans`` ... ``helmholtz_apply``, ``apply_operator``) so that
  ``SUM_FAC_TOP`` runs on the device and every other strategy runs the
  reference's own code.  ``apply_to_field`` then routes each block through
  the wrapped ``apply_operator`` unchanged (operators.py:749-776).
"""

from __future__ import annotations

import ctypes
import functools
import os
import threading

import numpy as np

SK_OK = 0
SK_GEO_REGULAR, SK_GEO_DEFORMED = 0, 1
SK_PAYLOAD_HELMHOLTZ, SK_PAYLOAD_W, SK_PAYLOAD_DERIV, SK_PAYLOAD_HELMHOLTZ_NC = 0, 1, 2, 3
SK_FORM_COLL, SK_FORM_NONCOLL = 0, 1

_LIB = None
_LOCK = threading.Lock()


def _lib():
    global _LIB
    if _LIB is None:
        with _LOCK:
            if _LIB is None:
                path = os.environ.get("SK200_LIB") or os.path.join(
                    os.path.dirname(os.path.abspath(__file__)), "..", "paper_2604_04644_b200", "libsk200.so"
                )
                lib = ctypes.CDLL(os.path.abspath(path))
                vp, i, i64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
                sig = {
                    "sk_basis_create": [i, i, ctypes.POINTER(vp)],
                    "sk_basis_create_q": [i, i, ctypes.POINTER(i), ctypes.POINTER(vp)],
                    "sk_basis_counts": [vp, ctypes.POINTER(i64)],
                    "sk_payload_size": [vp, i, i, i64, ctypes.POINTER(i64)],
                    "sk_payload_pack": [vp, i, i, i64, vp, vp, vp, vp],
                    "sk_bwd_trans": [vp, i64, i, i, vp, vp, vp],
                    "sk_iproduct_wrt_base": [vp, i, i64, i, i, vp, vp, vp, vp],
                    "sk_phys_deriv": [vp, i, i64, i, vp, vp, vp, vp],
                    "sk_iproduct_wrt_deriv_base": [vp, i, i64, i, vp, vp, vp, vp],
                    "sk_mass_apply": [vp, i, i64, i, i, vp, vp, vp, vp],
                    "sk_helmholtz_apply": [vp, i, i, i64, i, i, vp, vp, d, vp, vp],
                    "sk_device_alloc": [i64, ctypes.POINTER(vp)],
                    "sk_device_free": [vp],
                    "sk_copy_h2d": [vp, vp, i64, vp],
                    "sk_copy_d2h": [vp, vp, i64, vp],
                    "sk_stream_synchronize": [vp],
                }
                for name, args in sig.items():
                    fn = getattr(lib, name)
                    fn.argtypes = args
                    fn.restype = i
                lib.sk_last_error.restype = ctypes.c_char_p
                _LIB = lib
    return _LIB


def _check(status, what):
    if status == SK_OK:
        return
    from speckern.operators import FieldStateError, UnsupportedStrategyError

    msg = f"{what}: {(_lib().sk_last_error() or b'').decode(errors='replace')}"
    raise {1: FieldStateError, 2: UnsupportedStrategyError, 3: ValueError}.get(status, RuntimeError)(msg)


class _DevBuf:
    """A device allocation owned by the binding (MemoryRegion DEVICE space)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        _check(_lib().sk_device_alloc(max(self.nbytes, 8), ctypes.byref(p)), "sk_device_alloc")
        self.ptr = p

    def upload(self, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr, dtype=np.float64)
        assert a.nbytes <= max(self.nbytes, 8)
        _check(_lib().sk_copy_h2d(self.ptr, a.ctypes.data_as(ctypes.c_void_p), a.nbytes, None), "sk_copy_h2d")

    def download(self, arr: np.ndarray) -> None:
        assert arr.flags.c_contiguous and arr.dtype == np.float64
        _check(_lib().sk_copy_d2h(arr.ctypes.data_as(ctypes.c_void_p), self.ptr, arr.nbytes, None), "sk_copy_d2h")
        _check(_lib().sk_stream_synchronize(None), "sk_stream_synchronize")

    def __del__(self):
        try:
            _lib().sk_device_free(self.ptr)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_BASES: dict = {}


def _basis(block):
    """libsk200 basis handle for the block's (shape, order, point counts):
    the default quadrature (shapes.py:132-139) runs the specialised kernels,
    a qpoints override (shapes.py:521-541) the library's run-time-size path."""
    from speckern.shapes import Shape

    sb = block.basis
    q = tuple(int(v) for v in sb.qcounts)
    key = (sb.shape, sb.order, q)
    with _LOCK:
        if key not in _BASES:
            h = ctypes.c_void_p()
            qa = (ctypes.c_int * 3)(*q)
            _check(_lib().sk_basis_create_q(list(Shape).index(sb.shape), sb.order, qa, ctypes.byref(h)),
                   "sk_basis_create_q")
            _BASES[key] = h
        return _BASES[key]


def _geo(block) -> int:
    from speckern.geometry import GeometryClass

    return SK_GEO_DEFORMED if block.geometry_class is GeometryClass.DEFORMED else SK_GEO_REGULAR


def _payload(block, kind):
    """Device geometry payload of an operator family, built once per block
    and cached like the reference's payloads (field_block.py:309-321)."""
    key = ("sk200", kind)
    cache = block._payload_cache
    if key in cache:
        return cache[key]
    b = _basis(block)
    n = ctypes.c_int64()
    _check(_lib().sk_payload_size(b, _geo(block), kind, block.n_elements, ctypes.byref(n)), "sk_payload_size")
    pay = _DevBuf(8 * n.value)
    fac = block.factors
    dxi = _DevBuf(fac.dxi_dx.nbytes)
    jac = _DevBuf(fac.jac.nbytes)
    dxi.upload(fac.dxi_dx)
    jac.upload(fac.jac)
    _check(_lib().sk_payload_pack(b, _geo(block), kind, block.n_elements, dxi.ptr, jac.ptr, pay.ptr, None),
           "sk_payload_pack")
    _check(_lib().sk_stream_synchronize(None), "sk_stream_synchronize")
    cache[key] = pay
    return pay


def _out_block(block, out, state, ncomp):
    """operators.py:537-548 (same checks, same error types)."""
    from speckern.operators import FieldStateError

    if out is None:
        return block.like(state, ncomp)
    if out.state is not state or out.n_components != ncomp:
        raise FieldStateError(f"output block must be {state.value}-state with {ncomp} component(s)")
    if out.basis is not block.basis or out.interleave_width != block.interleave_width:
        raise ValueError("output block layout does not match the input block")
    return out


def _require(block, state, op):
    from speckern.operators import FieldStateError

    if block.state is not state:
        raise FieldStateError(f"{op} expects a {state.value}-state block, got {block.state.value}")


def _run(block, out, call, payload_kind=None):
    """Upload the block's host region, run ``call(basis, geo, d_in, pay,
    d_out)`` and write the result through ``out.host(WRITE_ONLY)``."""
    from speckern.field_block import AccessQualifier

    src = block.host(AccessQualifier.READ_ONLY)
    d_in = _DevBuf(src.nbytes)
    d_in.upload(src)
    pay = _payload(block, payload_kind).ptr if payload_kind is not None else None
    dst = out.host(AccessQualifier.WRITE_ONLY)
    d_out = _DevBuf(dst.nbytes)
    _check(call(_basis(block), _geo(block), d_in.ptr, pay, d_out.ptr), "sumfac_top apply")
    d_out.download(dst)
    return out


def _check_strategy(strategy):
    from speckern.operators import Strategy, UnsupportedStrategyError

    if strategy is not Strategy.SUM_FAC_TOP:
        raise UnsupportedStrategyError(f"libsk200 implements sumfac_top, got {strategy.value!r}")


# ---------------------------------------------------------------------------
# the seven reference operators (operators.py:551-721), SUM_FAC_TOP


def bwd_trans(block, strategy=None, out=None):
    """u = B uhat (operators.py:551-561)."""
    from speckern.field_block import FieldState

    _require(block, FieldState.COEFF, "bwd_trans")
    out = _out_block(block, out, FieldState.PHYS, block.n_components)
    E, W, C = block.n_elements, block.interleave_width, block.n_components
    return _run(block, out, lambda b, g, i, p, o: _lib().sk_bwd_trans(b, E, W, C, i, o, None))


def iproduct_wrt_base(block, strategy=None, out=None):
    """fhat = B^T W u (operators.py:564-574)."""
    from speckern.field_block import FieldState

    _require(block, FieldState.PHYS, "iproduct_wrt_base")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    E, W, C = block.n_elements, block.interleave_width, block.n_components
    return _run(block, out, lambda b, g, i, p, o: _lib().sk_iproduct_wrt_base(b, g, E, W, C, i, p, o, None),
                SK_PAYLOAD_W)


def phys_deriv(block, out=None):
    """Cartesian derivatives at the quadrature points (operators.py:577-596)."""
    from speckern.field_block import FieldState

    _require(block, FieldState.PHYS, "phys_deriv")
    if block.n_components != 1:
        raise ValueError("phys_deriv expects a single-component block")
    out = _out_block(block, out, FieldState.PHYS, block.basis.ndim)
    E, W = block.n_elements, block.interleave_width
    return _run(block, out, lambda b, g, i, p, o: _lib().sk_phys_deriv(b, g, E, W, i, p, o, None), SK_PAYLOAD_DERIV)


def iproduct_wrt_deriv_base(block, strategy=None, out=None):
    """fhat = sum_d (D_d B)^T W v_d (operators.py:599-619)."""
    from speckern.field_block import FieldState

    _require(block, FieldState.PHYS, "iproduct_wrt_deriv_base")
    d = block.basis.ndim
    if block.n_components != d:
        raise ValueError(f"iproduct_wrt_deriv_base expects {d} components, got {block.n_components}")
    out = _out_block(block, out, FieldState.COEFF, 1)
    E, W = block.n_elements, block.interleave_width
    return _run(block, out, lambda b, g, i, p, o: _lib().sk_iproduct_wrt_deriv_base(b, g, E, W, i, p, o, None),
                SK_PAYLOAD_W)


def mass_apply(block, strategy=None, out=None):
    """M uhat = B^T W B uhat (operators.py:622-633)."""
    from speckern.field_block import FieldState

    _require(block, FieldState.COEFF, "mass_apply")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    E, W, C = block.n_elements, block.interleave_width, block.n_components
    return _run(block, out, lambda b, g, i, p, o: _lib().sk_mass_apply(b, g, E, W, C, i, p, o, None), SK_PAYLOAD_W)


def _helmholtz(block, lam, out, form, name):
    from speckern.field_block import FieldState

    _require(block, FieldState.COEFF, name)
    if lam < 0.0:
        raise ValueError(f"reaction coefficient must be nonnegative, got {lam}")
    out = _out_block(block, out, FieldState.COEFF, block.n_components)
    E, W, C = block.n_elements, block.interleave_width, block.n_components
    kind = SK_PAYLOAD_HELMHOLTZ if form == SK_FORM_COLL else SK_PAYLOAD_HELMHOLTZ_NC
    return _run(block, out,
                lambda b, g, i, p, o: _lib().sk_helmholtz_apply(b, g, form, E, W, C, i, p, float(lam), o, None), kind)


def helmholtz_apply_noncoll(block, lam, strategy=None, out=None):
    """Alg. 5 pipeline (operators.py:636-667)."""
    return _helmholtz(block, lam, out, SK_FORM_NONCOLL, "helmholtz_apply_noncoll")


def helmholtz_apply_coll(block, lam, strategy=None, out=None):
    """Alg. 6 collocated pipeline (operators.py:670-699)."""
    return _helmholtz(block, lam, out, SK_FORM_COLL, "helmholtz_apply_coll")


def helmholtz_apply(block, lam, strategy=None, form=None, out=None):
    """operators.py:702-721: a sum-factorised strategy defaults to the
    collocated form (as SUM_FAC does)."""
    form = "coll" if form is None else form
    if form == "coll":
        return helmholtz_apply_coll(block, lam, strategy, out)
    if form == "noncoll":
        return helmholtz_apply_noncoll(block, lam, strategy, out)
    raise ValueError(f"unknown Helmholtz form: {form!r}")


def apply_operator(kind, block, strategy=None, lam=1.0, out=None):
    """operators.py:724-746 for SUM_FAC_TOP."""
    from speckern.operators import OperatorKind

    table = {
        OperatorKind.BWD_TRANS: lambda: bwd_trans(block, strategy, out),
        OperatorKind.IPRODUCT_WRT_BASE: lambda: iproduct_wrt_base(block, strategy, out),
        OperatorKind.PHYS_DERIV: lambda: phys_deriv(block, out),
        OperatorKind.IPRODUCT_WRT_DERIV_BASE: lambda: iproduct_wrt_deriv_base(block, strategy, out),
        OperatorKind.MASS: lambda: mass_apply(block, strategy, out),
        OperatorKind.HELMHOLTZ_NONCOLL: lambda: helmholtz_apply_noncoll(block, lam, strategy, out),
        OperatorKind.HELMHOLTZ_COLL: lambda: helmholtz_apply_coll(block, lam, strategy, out),
    }
    if kind not in table:
        raise ValueError(f"unknown operator kind: {kind!r}")
    return table[kind]()


# ---------------------------------------------------------------------------
# wiring into an imported (unmodified) speckern

_OPS = ("bwd_trans", "iproduct_wrt_base", "iproduct_wrt_deriv_base", "mass_apply", "helmholtz_apply_noncoll",
        "helmholtz_apply_coll", "helmholtz_apply", "phys_deriv", "apply_operator")
# position of the strategy argument in each reference signature
_STRATEGY_POS = {"bwd_trans": 1, "iproduct_wrt_base": 1, "iproduct_wrt_deriv_base": 1, "mass_apply": 1,
                 "helmholtz_apply_noncoll": 2, "helmholtz_apply_coll": 2, "helmholtz_apply": 2, "apply_operator": 2}


def _wrap(name, ref_fn):
    from speckern.operators import Strategy

    mine = globals()[name]
    pos = _STRATEGY_POS.get(name)

    @functools.wraps(ref_fn)
    def routed(*args, **kwargs):
        if pos is None:  # phys_deriv has no strategy argument: reference code path
            return ref_fn(*args, **kwargs)
        strategy = kwargs.get("strategy", args[pos] if len(args) > pos else None)
        if strategy is Strategy.SUM_FAC_TOP:
            return mine(*args, **kwargs)
        return ref_fn(*args, **kwargs)

    routed.__sk200_routed__ = True
    return routed


def install(speckern_module=None) -> None:
    """Route ``Strategy.SUM_FAC_TOP`` of an imported speckern to libsk200:
    the module-level operator functions (and their package re-exports) are
    wrapped, so speckern's own ``apply_operator`` / ``apply_to_field`` /
    bench drivers reach the device for SUM_FAC_TOP.  ``apply_operator`` with
    PHYS_DERIV and SUM_FAC_TOP runs the device phys_deriv as well.
    Idempotent."""
    import importlib

    sk = speckern_module or importlib.import_module("speckern")
    ops = importlib.import_module(sk.__name__ + ".operators")
    for name in _OPS:
        ref_fn = getattr(ops, name)
        if getattr(ref_fn, "__sk200_routed__", False):
            continue
        routed = _wrap(name, ref_fn)
        routed.__sk200_original__ = ref_fn
        setattr(ops, name, routed)
        if getattr(sk, name, None) is ref_fn:
            setattr(sk, name, routed)


def uninstall(speckern_module=None) -> None:
    """Undo install(): restore the reference's own functions."""
    import importlib

    sk = speckern_module or importlib.import_module("speckern")
    ops = importlib.import_module(sk.__name__ + ".operators")
    for name in _OPS:
        fn = getattr(ops, name)
        orig = getattr(fn, "__sk200_original__", None)
        if orig is None:
            continue
        setattr(ops, name, orig)
        if getattr(sk, name, None) is fn:
            setattr(sk, name, orig)
