"""CPU tests of the host mirror of the reference API: memory-region access
automaton, interleave helpers, counters, errors and the bench contract."""

import itertools
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import paper_2604_04644_b200 as sk
from paper_2604_04644_b200.field_block import AccessQualifier as AQ
from paper_2604_04644_b200.field_block import MemoryRegion, MemorySpace as MS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _Arena(MemoryRegion):
    """MemoryRegion whose DEVICE space is a host arena (no GPU here)."""

    def _alloc_device(self):
        return np.zeros(self.length)


class _Automaton:
    """Independent model of the access semantics (field_block.py:75-89;
    reference test_acceptance.py:222-246)."""

    def __init__(self):
        self.valid = {MS.HOST: False, MS.DEVICE: False}
        self.init = False
        self.transfers = 0

    def access(self, space, q):
        other = MS.DEVICE if space is MS.HOST else MS.HOST
        if q is AQ.WRITE_ONLY:
            self.valid[space], self.valid[other], self.init = True, False, True
            return True
        if not self.init:
            return False
        if not self.valid[space]:
            self.transfers += 1
            self.valid[space] = True
        if q is AQ.READ_WRITE:
            self.valid[other] = False
        return True


def test_memory_region_automaton_exhaustive():
    """Every access sequence of length <= 4 matches the model (reference
    acceptance criterion 6)."""
    ops = list(itertools.product(list(MS), list(AQ)))
    for n in range(1, 5):
        for seq in itertools.product(ops, repeat=n):
            reg, model = _Arena(4), _Automaton()
            for space, q in seq:
                ok = model.access(space, q)
                if ok:
                    reg.access(space, q)
                else:
                    with pytest.raises(sk.InitialisationError):
                        reg.access(space, q)
                assert reg.transfer_count == model.transfers
                assert reg.valid(MS.HOST) == model.valid[MS.HOST]
                assert reg.valid(MS.DEVICE) == model.valid[MS.DEVICE]


def test_memory_region_data_round_trip():
    reg = _Arena(6)
    reg.access(MS.HOST, AQ.WRITE_ONLY)[:] = np.arange(6.0)
    dev = reg.access(MS.DEVICE, AQ.READ_WRITE)
    dev *= 2.0
    assert np.array_equal(reg.access(MS.HOST, AQ.READ_ONLY), 2.0 * np.arange(6.0))
    ro = reg.access(MS.HOST, AQ.READ_ONLY)
    with pytest.raises(ValueError):
        ro[0] = 1.0
    with pytest.raises(ValueError):
        MemoryRegion(-1)


@pytest.mark.parametrize("width", [1, 3, 8])
def test_interleave_round_trip_and_padding(width):
    x = np.random.default_rng(0).standard_normal((5, 13))
    lanes = sk.interleave_array(x, width)
    assert lanes.shape == (-(-13 // width), 5, width)
    assert np.array_equal(sk.deinterleave_array(lanes, 13), x)
    flat = lanes.transpose(1, 0, 2).reshape(5, -1)
    assert np.all(flat[:, 13:] == 0.0)


@pytest.mark.parametrize("shape", ["hex", "prism", "pyr", "tet"])
def test_counts_and_flops_match_reference(golden_tables, shape):
    S = sk.Shape(shape)
    for P in range(1, 11):
        assert sk.mode_count(S, P) == O.mode_count(shape, P)
        assert sk.quad_point_counts(S, P) == O.qcounts(shape, P)
        assert sk.index_set(S, P) == tuple(O.mode_set(shape, P))
        for kind in sk.OperatorKind:
            assert sk.operator_flops(kind, S, P) == int(golden_tables[f"{shape}_P{P}_flops_{kind.value}"])


def test_bytes_model():
    b = sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, sk.Shape.TET, 4, True)
    assert b == 8 * (2 * 35 + 7 * 150) == 8960
    assert sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, sk.Shape.TET, 4, True, 0.0) == 8 * (70 + 6 * 150)
    assert sk.operator_bytes(sk.OperatorKind.MASS, sk.Shape.HEX, 4, False) == 8 * (250 + 1)


def test_strategy_and_state_errors():
    with pytest.raises(sk.UnsupportedStrategyError):
        sk.operators._check_strategy(sk.Strategy.STD_MAT)
    sk.operators._check_strategy(sk.Strategy.SUM_FAC)
    sk.operators._check_strategy(sk.Strategy.SUM_FAC_TOP)
    basis = sk.build_shape_basis(sk.Shape.HEX, 2)
    fac = sk.make_synthetic_factors(basis, sk.GeometryClass.REGULAR, 3, seed=0)
    blk = sk.Block(basis, fac, sk.FieldState.PHYS, 1, 2)
    with pytest.raises(sk.FieldStateError):
        sk.mass_apply(blk)
    cb = sk.Block(basis, fac, sk.FieldState.COEFF, 1, 2)
    with pytest.raises(ValueError):
        sk.helmholtz_apply(cb, -1.0)
    with pytest.raises(ValueError):
        sk.helmholtz_apply(cb, 1.0, form="bogus")


def test_host_geometry_matches_oracle():
    """Affine factors and deformation draws are computed on the host with the
    reference's seeding; they match the oracle bit for bit."""
    for shape in ("hex", "prism", "pyr", "tet"):
        basis = sk.build_shape_basis(sk.Shape(shape), 2)
        fac = sk.make_synthetic_factors(basis, sk.GeometryClass.REGULAR, 5, seed=7)
        geo = O.synthetic_geometry(O.element(shape, 2), False, 5, seed=7)
        assert np.array_equal(fac.dxi_dx, geo.dxi) and np.array_equal(fac.jac, geo.jac)
    from paper_2604_04644_b200.geometry import synthetic_deformation_params

    assert np.array_equal(synthetic_deformation_params(9, 3, first=11), O.deformation_params(9, 3, first=11))


def test_bench_reference_arm_contract():
    """bench.py --impl reference prints one JSON line with the contract keys."""
    env = dict(os.environ, SK_BENCH_CPU_PER_CORE="256")
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1"],
        capture_output=True, text=True, env=env, timeout=300,
    )
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "config", "higher_is_better"):
        assert key in line
    assert line["impl"] == "reference" and line["value"] > 0
    # the unmodified reference (baseline/_ref) when installed, else the oracle port
    want = "reference" if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "speckern")) else "port"
    assert line["cpu_baseline"]["kind"] == want and line["cpu_baseline"]["cores"] >= 1


def test_bench_rank_count_must_match_gpus():
    """--gpus N inside a launcher that started a different rank count fails
    loudly instead of reporting the wrong n_gpus."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, env=env, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


def test_bench_gpus_flag_relaunches_ranks():
    """--gpus 2 outside a launcher re-executes bench.py under
    torch.distributed.run with two ranks; rank 0 alone prints the line
    (n_gpus 2), the other rank exits 0 (reference arm: no GPU needed)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["SK_BENCH_CPU_PER_CORE"] = "64"
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
         "--warmup", "1"],
        capture_output=True, text=True, env=env, timeout=600,
    )
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
