"""Run one operator a few times on a synthetic block (for ncu captures).

  python tools/profile_op.py --shape tet --order 4 --elements 262144 --op helm --reps 5
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="tet")
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--elements", type=int, default=1 << 18)
    ap.add_argument("--op", default="helm", choices=["helm", "stiff", "mass", "bwd", "iprod", "pderiv", "ipderiv", "helmstaged"])
    ap.add_argument("--geo", default="deformed", choices=["deformed", "regular"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--width", type=int, default=1)
    a = ap.parse_args()
    import torch

    import paper_2604_04644_b200 as sk

    b = sk.build_shape_basis(sk.Shape(a.shape), a.order)
    gcls = sk.GeometryClass.DEFORMED if a.geo == "deformed" else sk.GeometryClass.REGULAR
    fac = sk.make_synthetic_factors(b, gcls, a.elements, seed=0)
    coeff = a.op in ("helm", "stiff", "mass", "bwd", "helmstaged")
    ncomp = 3 if a.op == "ipderiv" else 1
    blk = sk.Block(b, fac, sk.FieldState.COEFF if coeff else sk.FieldState.PHYS, ncomp, a.width)
    n = b.n_modes if coeff else b.n_points
    blk.set_elements(np.random.default_rng(0).uniform(-1, 1, (ncomp, n, a.elements)))
    blk.device()  # device-resident input: the plain (non-streamed) launch is profiled
    fn = {
        "helm": lambda: sk.helmholtz_apply(blk, 1.0),
        "helmstaged": lambda: sk.helmholtz_apply_staged(blk, 1.0),
        "stiff": lambda: sk.helmholtz_apply(blk, 0.0),
        "mass": lambda: sk.mass_apply(blk),
        "bwd": lambda: sk.bwd_trans(blk),
        "iprod": lambda: sk.iproduct_wrt_base(blk),
        "pderiv": lambda: sk.phys_deriv(blk),
        "ipderiv": lambda: sk.iproduct_wrt_deriv_base(blk),
    }[a.op]
    for _ in range(a.reps):
        fn()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
