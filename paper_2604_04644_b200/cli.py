"""``python -m paper_2604_04644_b200 bench ...``: the reference's benchmark
CLI (speckern/cli.py:71-120, bench.py:57-300) on the device path.

Same flags, the same CSV schema (``CSV_HEADER``, bench.py:57) and exit codes
(2 configuration error, 1 verification error; cli.py:307-315), strategy
``sumfac_top``.  Before timing, every combination is cross-checked between
two independent device routes at 1e-10 (the reference pairs two strategies,
bench.py:196-216): Helmholtz collocated vs non-collocated kernels; mass vs
``iproduct_wrt_base(bwd_trans(u))``; bwd_trans into a fresh vs a reused
output block.  Each batch is timed with the device synchronised on both
sides; ``seconds`` is the median batch time and ``dof_per_s`` = ndof x
applies per batch / seconds, as in the reference.
"""

from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

from paper_2604_04644_b200.field_block import Block, FieldState, default_interleave_width
from paper_2604_04644_b200.geometry import GeometryClass, make_synthetic_factors
from paper_2604_04644_b200.operators import (
    OperatorKind,
    Strategy,
    apply_operator,
    bwd_trans,
    iproduct_wrt_base,
    operator_flops,
)
from paper_2604_04644_b200.shapes import DEVICE_SHAPES, Shape, build_shape_basis

CSV_HEADER = "op,shape,P,strategy,geometry,form,nelem,ndof,seconds,dof_per_s,flops_per_elem"
OPS = ("mass", "helmholtz", "bwdtrans")
MIN_TIMED_SECONDS = 0.05
PAIR_TOL = 1e-10


class ConfigError(ValueError):
    """Invalid benchmark configuration (exit code 2)."""


class VerificationError(RuntimeError):
    """Device routes disagree before timing (exit code 1)."""


def _orders(text: str) -> list[int]:
    if ".." in text:
        a, b = text.split("..")
        return list(range(int(a), int(b) + 1))
    return [int(x) for x in text.split(",")]


def _shapes(text: str) -> list[Shape]:
    if text == "all":
        return list(DEVICE_SHAPES)
    try:
        return [Shape(s.strip()) for s in text.split(",")]
    except ValueError as exc:
        raise ConfigError(str(exc)) from None


def _rel(a, b) -> float:
    scale = max(float(np.max(np.abs(a))), float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale


def _sync():
    import torch

    torch.cuda.synchronize()


def _pair_check(op: str, blk: Block, lam: float, form: str) -> None:
    if op == "helmholtz":
        a = apply_operator(OperatorKind.HELMHOLTZ_COLL, blk, Strategy.SUM_FAC_TOP, lam).get_elements()
        b = apply_operator(OperatorKind.HELMHOLTZ_NONCOLL, blk, Strategy.SUM_FAC_TOP, lam).get_elements()
    elif op == "mass":
        a = apply_operator(OperatorKind.MASS, blk).get_elements()
        b = iproduct_wrt_base(bwd_trans(blk)).get_elements()
    else:
        a = bwd_trans(blk).get_elements()
        b = bwd_trans(blk, out=bwd_trans(blk)).get_elements()
    err = _rel(a, b)
    if not err <= PAIR_TOL:
        raise VerificationError(f"device routes disagree before timing: {op} {blk.shape.value} "
                                f"P={blk.basis.order} nelem={blk.n_elements}: max rel err {err:.3e}")


def run_bench(op, shapes, orders, nelems, geometry, form, lam, width, reps, warmup, seed):
    if op not in OPS:
        raise ConfigError(f"unknown op {op!r}; choose from {sorted(OPS)}")
    if reps < 3 or warmup < 1 or lam < 0 or form not in ("coll", "noncoll"):
        raise ConfigError("need reps >= 3, warmup >= 1, lambda >= 0, form in {coll, noncoll}")
    if any(n < 1 for n in nelems) or any(p < 1 for p in orders):
        raise ConfigError("element counts and orders must be positive")
    rows = []
    for shape in shapes:
        for P in orders:
            basis = build_shape_basis(shape, P)
            for ne in nelems:
                blk = Block(basis, make_synthetic_factors(basis, geometry, ne, seed=seed), FieldState.COEFF, 1, width)
                rng = np.random.default_rng([seed, list(Shape).index(shape), P, 1])
                blk.set_elements(np.ascontiguousarray(rng.uniform(-1.0, 1.0, (ne, basis.n_modes)).T)[None])
                _pair_check(op, blk, lam, form)
                blk.device()
                if op == "helmholtz":
                    kind = OperatorKind.HELMHOLTZ_COLL if form == "coll" else OperatorKind.HELMHOLTZ_NONCOLL
                else:
                    kind = OperatorKind.MASS if op == "mass" else OperatorKind.BWD_TRANS
                out = blk.like(FieldState.PHYS if kind is OperatorKind.BWD_TRANS else FieldState.COEFF)

                def once():
                    apply_operator(kind, blk, Strategy.SUM_FAC_TOP, lam, out)

                _sync()
                t0 = time.perf_counter()
                once()
                _sync()
                iters = max(1, math.ceil(MIN_TIMED_SECONDS / max(time.perf_counter() - t0, 1e-9)))
                for _ in range(warmup * iters):
                    once()
                raw = []
                for _ in range(reps):
                    _sync()
                    t0 = time.perf_counter()
                    for _ in range(iters):
                        once()
                    _sync()
                    raw.append(time.perf_counter() - t0)
                med = float(np.median(raw))
                ndof = basis.n_modes * ne
                rows.append(",".join([
                    op, shape.value, str(P), Strategy.SUM_FAC_TOP.value, geometry.value,
                    form if op == "helmholtz" else "-", str(ne), str(ndof), f"{med:.9e}",
                    f"{ndof * iters / med:.6e}", str(operator_flops(kind, shape, P)),
                ]))
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2604_04644_b200")
    sub = ap.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench", help="time operators, print the reference CSV schema")
    b.add_argument("--op", default="mass")
    b.add_argument("--shape", default="all")
    b.add_argument("--order", default="1..4")
    b.add_argument("--nelem", default="4096")
    b.add_argument("--geometry", default="regular", choices=["regular", "deformed"])
    b.add_argument("--form", default="coll")
    b.add_argument("--lambda", dest="lam", type=float, default=1.0)
    b.add_argument("--simd-width", dest="width", type=int, default=None)
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--warmup", type=int, default=1)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--csv", default=None)
    a = ap.parse_args(argv)
    try:
        rows = run_bench(a.op, _shapes(a.shape), _orders(a.order), [int(x) for x in a.nelem.split(",")],
                         GeometryClass(a.geometry), a.form, a.lam,
                         default_interleave_width() if a.width is None else a.width, a.reps, a.warmup, a.seed)
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except VerificationError as exc:
        print(f"verification failed: {exc}", file=sys.stderr)
        return 1
    text = "\n".join([CSV_HEADER] + rows) + "\n"
    if a.csv:
        with open(a.csv, "w") as fh:
            fh.write(text)
    sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
