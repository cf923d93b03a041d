"""ctypes binding of the C ABI in ``include/sk200.h`` (``libsk200.so``).

The library is built in-tree by ``__graft_entry__.build()`` (``make`` in
``csrc/``).  There is no fallback: if the shared object is missing every
device operator raises ``RuntimeError`` at the call site.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
#: SK200_LIB selects an alternative in-tree build (tuning variants only)
LIB_PATH = os.environ.get("SK200_LIB") or os.path.join(_HERE, "libsk200.so")

SK_OK, SK_ERR_STATE, SK_ERR_UNSUPPORTED, SK_ERR_ARG, SK_ERR_CUDA = range(5)
SK_GEO_REGULAR, SK_GEO_DEFORMED = 0, 1
SK_PAYLOAD_HELMHOLTZ, SK_PAYLOAD_W, SK_PAYLOAD_DERIV, SK_PAYLOAD_HELMHOLTZ_NC = 0, 1, 2, 3
SK_FORM_COLL, SK_FORM_NONCOLL = 0, 1
SK_STREAM_HELMHOLTZ, SK_STREAM_HELMHOLTZ_NC, SK_STREAM_MASS = 0, 1, 2
SK_STREAM_DIRECT_OUT = 1

#: every exported symbol and its (restype, argtypes)
_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_L = ctypes.c_int64
_PL = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "sk_basis_create": (_I, [_I, _I, ctypes.POINTER(_P)]),
    "sk_basis_create_q": (_I, [_I, _I, ctypes.POINTER(_I), ctypes.POINTER(_P)]),
    "sk_basis_destroy": (_I, [_P]),
    "sk_basis_counts": (_I, [_P, _PL]),
    "sk_basis_table": (_I, [_P, ctypes.c_char_p, _PD, _L, _PL]),
    "sk_payload_size": (_I, [_P, _I, _I, _L, _PL]),
    "sk_payload_pack": (_I, [_P, _I, _I, _L, _P, _P, _P, _P]),
    "sk_geometry_deformed": (_I, [_P, _L, _P, _P, _P, _PL, _P]),
    "sk_payload_from_params": (_I, [_P, _I, _L, _P, _P, _PL, _P]),
    "sk_geometry_from_coords": (_I, [_P, _L, _P, _P, _P, _PL, _P]),
    "sk_geometry_from_coords_oriented": (_I, [_P, _L, _P, _P, _P, _PL, _P]),
    "sk_bwd_trans": (_I, [_P, _L, _I, _I, _P, _P, _P]),
    "sk_iproduct_wrt_base": (_I, [_P, _I, _L, _I, _I, _P, _P, _P, _P]),
    "sk_phys_deriv": (_I, [_P, _I, _L, _I, _P, _P, _P, _P]),
    "sk_iproduct_wrt_deriv_base": (_I, [_P, _I, _L, _I, _P, _P, _P, _P]),
    "sk_mass_apply": (_I, [_P, _I, _L, _I, _I, _P, _P, _P, _P]),
    "sk_helmholtz_apply": (_I, [_P, _I, _I, _L, _I, _I, _P, _P, _D, _P, _P]),
    "sk_helmholtz_apply_staged": (_I, [_P, _I, _L, _I, _I, _P, _P, _D, _P, _P, _L, _P]),
    "sk_helmholtz_apply_params": (_I, [_P, _L, _I, _I, _P, _P, _D, _P, _P, _L, _P, _P]),
    "sk_apply_streamed": (_I, [_P, _I, _I, _L, _I, _I, _P, _P, _P, _D, _P, _P, _L, _P]),
    "sk_apply_streamed_ex": (_I, [_P, _I, _I, _L, _I, _I, _P, _P, _P, _D, _P, _P, _L, _I, _P]),
    "sk_c0_gather": (_I, [_I, _I, _I, _L, _P, _I, _P, _P]),
    "sk_c0_scatter": (_I, [_I, _I, _I, _L, _P, _I, _P, _P]),
    "sk_c0_gather_map": (_I, [_L, _I, _P, _P, _P, _I, _P, _P]),
    "sk_c0_scatter_map": (_I, [_L, _I, _P, _P, _P, _P, _I, _P, _P]),
    "sk_c0_gather_map32": (_I, [_L, _I, _P, _P, _I, _P, _P]),
    "sk_c0_scatter_map32": (_I, [_L, _I, _P, _P, _P, _I, _P, _P]),
    "sk_helmholtz_apply_c0": (_I, [_P, _I, _I, _I, _L, _P, _P, _D, _P, _P]),
    "sk_helmholtz_apply_c0_w": (_I, [_P, _I, _I, _I, _L, _P, _P, _D, _P, _L, _P]),
    "sk_helmholtz_apply_c0_mapped": (_I, [_P, _I, _L, _P, _P, _P, _D, _P, _P]),
    "sk_device_alloc": (_I, [_L, ctypes.POINTER(_P)]),
    "sk_device_free": (_I, [_P]),
    "sk_copy_h2d": (_I, [_P, _P, _L, _P]),
    "sk_copy_d2h": (_I, [_P, _P, _L, _P]),
    "sk_stream_synchronize": (_I, [_P]),
    "sk_launch_count": (_L, []),
    "sk_last_error": (ctypes.c_char_p, []),
    "sk_launch_config": (_I, [_P, _I, _PL]),
    "sk_launch_config_geo": (_I, [_P, _I, _I, _PL]),
}

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load ``libsk200.so`` once; raise loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the sm_100a library first "
                    "(python -c 'import __graft_entry__ as g; g.build()')"
                )
            lib = ctypes.CDLL(LIB_PATH)
            variant = "SK200_LIB" in os.environ  # tuning builds may predate newer entry points
            for name, (res, args) in SIGNATURES.items():
                if variant and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class DeviceError(RuntimeError):
    """CUDA failure reported by the library (status SK_ERR_CUDA)."""


def check(status: int, what: str) -> None:
    """Map an ABI status onto the reference's exception types
    (operators.py:70-75)."""
    if status == SK_OK:
        return
    msg = (load().sk_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if msg else what
    if status == SK_ERR_STATE:
        from paper_2604_04644_b200.operators import FieldStateError

        raise FieldStateError(text)
    if status == SK_ERR_UNSUPPORTED:
        from paper_2604_04644_b200.operators import UnsupportedStrategyError

        raise UnsupportedStrategyError(text)
    if status == SK_ERR_ARG:
        raise ValueError(text)
    raise DeviceError(text)


def launch_count() -> int:
    return int(load().sk_launch_count())
