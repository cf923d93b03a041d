"""Helmholtz / stiffness / mass parity of the loaded library (SK200_LIB
variants included) against the oracle on small blocks, every shape x order,
deformed and regular geometry:
  SK200_LIB=... python tools/check_helm.py [orders] [helm,mass]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2604_04644_b200 as sk  # noqa: E402

orders = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(range(1, 11))
ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["helm", "mass"]
worst = 0.0
for shape in ("hex", "prism", "pyr", "tet"):
    for P in orders:
        el = O.element(shape, P)
        n = 37
        b = sk.build_shape_basis(sk.Shape(shape), P)
        x = np.random.default_rng(P).uniform(-1, 1, (el.nm, n))
        for deformed in (True, False):
            gcls = sk.GeometryClass.DEFORMED if deformed else sk.GeometryClass.REGULAR
            fac = sk.make_synthetic_factors(b, gcls, n, seed=1)
            geo = O.synthetic_geometry(el, deformed, n, seed=1)
            cases = []
            if "helm" in ops:
                cases += [(f"helm lam={lam}", lambda blk, lam=lam: sk.helmholtz_apply(blk, lam),
                           lambda lam=lam: O.helmholtz_coll(el, geo, x, lam)) for lam in (0.0, 1.3)]
            if "mass" in ops:
                cases.append(("mass", lambda blk: sk.mass_apply(blk), lambda: O.mass(el, geo, x)))
            for name, fn, ref in cases:
                blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
                blk.set_elements(x[None])
                got = fn(blk).get_elements()[0]
                err = O.rel_diff(got, ref())
                worst = max(worst, err)
                if err > 1e-12:
                    print(f"FAIL {shape} P={P} {name} deformed={deformed}: {err:.3e}")
print(f"worst max-normalised error {worst:.3e}")
sys.exit(0 if worst <= 1e-12 else 1)
