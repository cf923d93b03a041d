"""Probe: the Helmholtz kernel reading its coefficients from / writing its
result to pinned host memory directly (UVA zero-copy over PCIe) vs the
chunk-pipelined streamed apply, tet P=4, 2^20 deformed elements.
GPU box: python tools/zero_copy_probe.py"""

import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2604_04644_b200 as sk  # noqa: E402
from paper_2604_04644_b200 import _lib  # noqa: E402

E = 1 << 20
b = sk.build_shape_basis(sk.Shape.TET, 4)
fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, E, seed=0)
blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
blk.device(sk.AccessQualifier.WRITE_ONLY).uniform_(-1, 1)
out = blk.like(sk.FieldState.COEFF)
ref = sk.helmholtz_apply(blk, 1.0, out=out).device().clone()
pay = blk.payload(_lib.SK_PAYLOAD_HELMHOLTZ)
n = b.n_modes * E
hin = torch.empty(n, dtype=torch.float64, pin_memory=True)
hout = torch.empty(n, dtype=torch.float64, pin_memory=True)
hin.copy_(blk.device())
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream


def zc():
    st = lib.sk_helmholtz_apply(b.handle, _lib.SK_GEO_DEFORMED, _lib.SK_FORM_COLL, E, 1, 1,
                                ctypes.c_void_p(hin.data_ptr()), ctypes.c_void_p(pay.data_ptr()), ctypes.c_double(1.0),
                                ctypes.c_void_p(hout.data_ptr()), ctypes.c_void_p(s))
    assert st == 0, st


din = blk.device()


def zc_out():  # coefficients resident on the device, result written to pinned host memory
    st = lib.sk_helmholtz_apply(b.handle, _lib.SK_GEO_DEFORMED, _lib.SK_FORM_COLL, E, 1, 1,
                                ctypes.c_void_p(din.data_ptr()), ctypes.c_void_p(pay.data_ptr()), ctypes.c_double(1.0),
                                ctypes.c_void_p(hout.data_ptr()), ctypes.c_void_p(s))
    assert st == 0, st


def zc_in():  # coefficients read from pinned host memory, result on the device
    st = lib.sk_helmholtz_apply(b.handle, _lib.SK_GEO_DEFORMED, _lib.SK_FORM_COLL, E, 1, 1,
                                ctypes.c_void_p(hin.data_ptr()), ctypes.c_void_p(pay.data_ptr()), ctypes.c_double(1.0),
                                ctypes.c_void_p(out.device().data_ptr()), ctypes.c_void_p(s))
    assert st == 0, st


for name, fn in (("zero_copy", zc), ("zero_copy_out_only", zc_out), ("zero_copy_in_only", zc_in)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    res = out.device() if name == "zero_copy_in_only" else hout.cuda()
    err = float((res - ref).abs().max() / ref.abs().max())
    print(json.dumps({"mode": name, "ms": best * 1e3, "gdof_s": n / best / 1e9, "max_rel": err}), flush=True)
# the streamed path for comparison
for _ in range(2):
    blk.host(sk.AccessQualifier.READ_WRITE)
    sk.helmholtz_apply(blk, 1.0, out=out).host()
best = 1e9
for _ in range(5):
    blk.host(sk.AccessQualifier.READ_WRITE)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk.helmholtz_apply(blk, 1.0, out=out)
    out.host()
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(json.dumps({"mode": "streamed", "ms": best * 1e3, "gdof_s": n / best / 1e9}), flush=True)
