"""Reference-side binding: the ctypes stub a speckern maintainer adds to route
``Strategy.SUM_FAC_TOP`` (the slot the reference reserves for a device
work-group variant, speckern/operators.py:57, 416-420) to libsk200.

It takes the reference's own ``Block`` objects and touches only the
reference's public data model:

* ``block.region`` host buffer (lane-major, field_block.py:205-265) -- the
  C ABI consumes exactly this layout, so the device copy is one memcpy;
* ``block.factors.dxi_dx`` / ``block.factors.jac`` (geometry.py:94-116) --
  packed once per block on the device by ``sk_payload_pack`` and cached in
  ``block._payload_cache`` like the reference's own payloads
  (field_block.py:309-321);
* ``list(Shape).index(shape)`` and ``basis.order`` -- the basis handle.

Device memory comes from cuda-python (no torch needed on the reference
side).  Errors map onto the reference exception types
(operators.py:70-75): status 1 -> FieldStateError, 2 ->
UnsupportedStrategyError, 3 -> ValueError.

Wiring inside speckern (operators.py), e.g.::

    if strategy is Strategy.SUM_FAC_TOP:
        from speckern import _sk200
        return _sk200.helmholtz_apply(block, lam, out)
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

try:  # cuda-python >= 12.x
    from cuda.bindings import runtime as cudart
except ImportError:  # pragma: no cover - older cuda-python
    from cuda import cudart

_LIB = None
SK_PAYLOAD_HELMHOLTZ, SK_PAYLOAD_W = 0, 1
SK_FORM_COLL = 0


def _lib():
    global _LIB
    if _LIB is None:
        path = os.environ.get("SK200_LIB") or os.path.join(
            os.path.dirname(os.path.abspath(__file__)), "..", "paper_2604_04644_b200", "libsk200.so"
        )
        lib = ctypes.CDLL(path)
        vp, i, i64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        lib.sk_basis_create.argtypes = [i, i, ctypes.POINTER(vp)]
        lib.sk_payload_size.argtypes = [vp, i, i, i64, ctypes.POINTER(i64)]
        lib.sk_payload_pack.argtypes = [vp, i, i, i64, vp, vp, vp, vp]
        lib.sk_helmholtz_apply.argtypes = [vp, i, i, i64, i, i, vp, vp, d, vp, vp]
        lib.sk_mass_apply.argtypes = [vp, i, i64, i, i, vp, vp, vp, vp]
        lib.sk_last_error.restype = ctypes.c_char_p
        _LIB = lib
    return _LIB


def _check(status, what):
    if status == 0:
        return
    from speckern.operators import FieldStateError, UnsupportedStrategyError

    msg = f"{what}: {_lib().sk_last_error().decode()}"
    raise {1: FieldStateError, 2: UnsupportedStrategyError, 3: ValueError}.get(status, RuntimeError)(msg)


def _cuda(ret):
    err = ret[0] if isinstance(ret, tuple) else ret
    if int(err) != 0:
        raise RuntimeError(f"CUDA error {err}")
    return ret[1] if isinstance(ret, tuple) and len(ret) > 1 else None


class _DevBuf:
    def __init__(self, nbytes):
        self.nbytes = max(int(nbytes), 8)
        self.ptr = int(_cuda(cudart.cudaMalloc(self.nbytes)))

    def upload(self, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        _cuda(cudart.cudaMemcpy(self.ptr, a.ctypes.data, a.nbytes, cudart.cudaMemcpyKind.cudaMemcpyHostToDevice))

    def download(self, arr):
        _cuda(cudart.cudaMemcpy(arr.ctypes.data, self.ptr, arr.nbytes, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost))

    def __del__(self):
        try:
            cudart.cudaFree(self.ptr)
        except Exception:
            pass


_BASES: dict = {}


def _basis(block):
    from speckern.shapes import Shape

    key = (block.shape, block.basis.order)
    if key not in _BASES:
        h = ctypes.c_void_p()
        _check(_lib().sk_basis_create(list(Shape).index(block.shape), block.basis.order, ctypes.byref(h)), "sk_basis_create")
        _BASES[key] = h
    return _BASES[key]


def _payload(block, kind):
    """Device geometry payload, built once per block (field_block.py:309-321)."""
    from speckern.geometry import GeometryClass

    key = ("sk200", kind)
    if key in block._payload_cache:
        return block._payload_cache[key]
    b = _basis(block)
    geo = 1 if block.geometry_class is GeometryClass.DEFORMED else 0
    n = ctypes.c_int64()
    _check(_lib().sk_payload_size(b, geo, kind, block.n_elements, ctypes.byref(n)), "sk_payload_size")
    pay = _DevBuf(8 * n.value)
    dxi, jac = _DevBuf(block.factors.dxi_dx.nbytes), _DevBuf(block.factors.jac.nbytes)
    dxi.upload(block.factors.dxi_dx)
    jac.upload(block.factors.jac)
    _check(_lib().sk_payload_pack(b, geo, kind, block.n_elements, dxi.ptr, jac.ptr, pay.ptr, None), "sk_payload_pack")
    _cuda(cudart.cudaDeviceSynchronize())
    block._payload_cache[key] = pay
    return pay


def _apply(block, out, kind, call):
    from speckern.field_block import AccessQualifier, FieldState
    from speckern.geometry import GeometryClass

    if block.state is not FieldState.COEFF:
        from speckern.operators import FieldStateError

        raise FieldStateError(f"expects a coeff-state block, got {block.state.value}")
    out = out if out is not None else block.like(FieldState.COEFF)
    src = block.host(AccessQualifier.READ_ONLY)
    d_in, d_out = _DevBuf(src.nbytes), _DevBuf(src.nbytes)
    d_in.upload(src)
    geo = 1 if block.geometry_class is GeometryClass.DEFORMED else 0
    _check(call(_basis(block), geo, d_in.ptr, _payload(block, kind).ptr, d_out.ptr), "apply")
    _cuda(cudart.cudaDeviceSynchronize())
    d_out.download(out.host(AccessQualifier.WRITE_ONLY))
    return out


def helmholtz_apply(block, lam, out=None):
    """SUM_FAC_TOP Helmholtz (collocated), speckern/operators.py:670-699."""
    if lam < 0.0:
        raise ValueError(f"reaction coefficient must be nonnegative, got {lam}")
    E, W, C = block.n_elements, block.interleave_width, block.n_components
    return _apply(
        block, out, SK_PAYLOAD_HELMHOLTZ,
        lambda b, geo, i, p, o: _lib().sk_helmholtz_apply(b, geo, SK_FORM_COLL, E, W, C, i, p, float(lam), o, None),
    )


def mass_apply(block, out=None):
    """SUM_FAC_TOP mass, speckern/operators.py:622-633."""
    E, W, C = block.n_elements, block.interleave_width, block.n_components
    return _apply(block, out, SK_PAYLOAD_W, lambda b, geo, i, p, o: _lib().sk_mass_apply(b, geo, E, W, C, i, p, o, None))
