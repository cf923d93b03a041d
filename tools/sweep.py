"""Throughput sweep over shapes x orders x operators on one GPU.

For every case the block is sized to ~``--gbytes`` of algorithmic traffic per
apply (>> 126 MB L2, no flush needed), timed with CUDA events over
``--reps`` back-to-back applies after warm-up.  Prints one JSON line per case
with GDOF/s, the HBM-roofline fraction (algorithmic bytes / time / measured
HBM peak) and the FP64 fraction (reference flop model / measured FP64 peak).

  python tools/sweep.py --ops helm,stiff,mass --shapes hex,prism,pyr,tet --orders 2-10
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _orders(s):
    if "-" in s:
        a, b = s.split("-")
        return list(range(int(a), int(b) + 1))
    return [int(x) for x in s.split(",")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="helm")
    ap.add_argument("--shapes", default="hex,prism,pyr,tet")
    ap.add_argument("--orders", default="2-10")
    ap.add_argument("--geo", default="deformed")
    ap.add_argument("--gbytes", type=float, default=2.0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--fp64-tflops", type=float, default=None)
    ap.add_argument("--chunk", type=int, default=0, help="staged variant: elements per chunk (0: default)")
    a = ap.parse_args()
    import torch

    import paper_2604_04644_b200 as sk
    from paper_2604_04644_b200 import _lib
    from paper_2604_04644_b200.geometry import synthetic_deformation_params

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    fp64 = a.fp64_tflops
    if fp64 is None:
        try:
            fp64 = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["fp64_tflops"]
        except OSError:
            fp64 = 34.2
    deformed = a.geo == "deformed"
    kinds = {"helm": (sk.OperatorKind.HELMHOLTZ_COLL, 1.0), "stiff": (sk.OperatorKind.HELMHOLTZ_COLL, 0.0),
             "mass": (sk.OperatorKind.MASS, 1.0), "helmnc": (sk.OperatorKind.HELMHOLTZ_NONCOLL, 1.0),
             "helmstaged": (sk.OperatorKind.HELMHOLTZ_COLL, 1.0), "stiffstaged": (sk.OperatorKind.HELMHOLTZ_COLL, 0.0),
             "bwd": (sk.OperatorKind.BWD_TRANS, 0.0), "iprod": (sk.OperatorKind.IPRODUCT_WRT_BASE, 0.0),
             "pderiv": (sk.OperatorKind.PHYS_DERIV, 0.0), "ipderiv": (sk.OperatorKind.IPRODUCT_WRT_DERIV_BASE, 0.0)}
    cases = []
    emax = 1
    for op in a.ops.split(","):
        kind, lam = kinds[op]
        for s in a.shapes.split(","):
            for P in _orders(a.orders):
                bel = sk.operator_bytes(kind, sk.Shape(s), P, deformed, lam)
                E = int(a.gbytes * 1e9 / bel)
                emax = max(emax, E)
                cases.append((op, kind, lam, s, P, E, bel))
    params = synthetic_deformation_params(emax, 0) if deformed else None
    for op, kind, lam, s, P, E, bel in cases:
        b = sk.build_shape_basis(sk.Shape(s), P)
        if deformed:
            fac = sk.GeometricFactors(sk.GeometryClass.DEFORMED, b.shape, E, params=params[:E], basis=b)
        else:
            fac = sk.make_synthetic_factors(b, sk.GeometryClass.REGULAR, E, seed=0)
        # input state / components per operator (GDOF/s counts coefficient DOFs throughout)
        st, nc = {"iprod": (sk.FieldState.PHYS, 1), "pderiv": (sk.FieldState.PHYS, 1),
                  "ipderiv": (sk.FieldState.PHYS, 3)}.get(op, (sk.FieldState.COEFF, 1))
        blk = sk.Block(b, fac, st, nc, 1)
        blk.device(sk.AccessQualifier.WRITE_ONLY).uniform_(-1.0, 1.0)
        out = {"bwd": lambda: blk.like(sk.FieldState.PHYS, 1), "pderiv": lambda: blk.like(sk.FieldState.PHYS, 3),
               "ipderiv": lambda: blk.like(sk.FieldState.COEFF, 1)}.get(op, lambda: blk.like(sk.FieldState.COEFF))()
        if op == "bwd":
            fn = lambda: sk.bwd_trans(blk, out=out)  # noqa: E731
        elif op == "iprod":
            fn = lambda: sk.iproduct_wrt_base(blk, out=out)  # noqa: E731
        elif op == "pderiv":
            fn = lambda: sk.phys_deriv(blk, out=out)  # noqa: E731
        elif op == "ipderiv":
            fn = lambda: sk.iproduct_wrt_deriv_base(blk, out=out)  # noqa: E731
        elif op == "mass":
            fn = lambda: sk.mass_apply(blk, out=out)  # noqa: E731
        elif op == "helmnc":
            fn = lambda: sk.helmholtz_apply_noncoll(blk, lam, out=out)  # noqa: E731
        elif op.endswith("staged"):
            fn = lambda: sk.helmholtz_apply_staged(blk, lam, out=out, chunk_elements=a.chunk)  # noqa: E731
        else:
            fn = lambda: sk.helmholtz_apply(blk, lam, out=out)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.reps):
            fn()
        t1.record()
        torch.cuda.synchronize()
        sec = t0.elapsed_time(t1) / 1e3 / a.reps
        gdof = b.n_modes * E / sec / 1e9
        flops = sk.operator_flops(kind, sk.Shape(s), P) * E
        cfg = b.launch_config({"mass": 1, "helmnc": 6, "helmstaged": 7, "stiffstaged": 7, "bwd": 2, "iprod": 3, "pderiv": 4,
                               "ipderiv": 5}.get(op, 0), deformed)
        rec = {
            "op": op, "shape": s, "P": P, "geo": a.geo, "elements": E, "ms": sec * 1e3, "gdof_s": gdof,
            "hbm_gbs": bel * E / sec / 1e9, "hbm_frac": bel * E / sec / 1e9 / hbm,
            "fp64_tflops": flops / sec / 1e12, "fp64_frac": flops / sec / 1e12 / fp64,
            "roofline_gdof_s": min(hbm * 1e9 / bel, fp64 * 1e12 / (flops / E)) * b.n_modes / 1e9,
            "eb_nt_smem": cfg,
        }
        rec["roofline_frac"] = gdof / rec["roofline_gdof_s"]
        print(json.dumps(rec), flush=True)
        del blk, out, fac
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
