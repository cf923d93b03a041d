"""SPKF field dump (reference field_block.py:433-497): files written by the
unmodified reference load bit-exactly and re-save byte-identically
(tests/golden/make_spkf.py made the fixture); CPU only."""

import os

import numpy as np
import pytest

import paper_2604_04644_b200 as sk

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_load_reference_dump_and_resave(tmp_path):
    fld = sk.load_field(os.path.join(GOLD, "field_ref.spkf"), seed=5, interleave_width=3)
    vals = np.load(os.path.join(GOLD, "field_ref.npz"))
    want = [(sk.Shape.HEX, 2, sk.FieldState.COEFF, 1), (sk.Shape.TET, 3, sk.FieldState.COEFF, 2),
            (sk.Shape.PRISM, 1, sk.FieldState.COEFF, 1)]
    assert len(fld.blocks) == 3
    for k, (blk, (shape, P, state, ncomp)) in enumerate(zip(fld.blocks, want)):
        assert (blk.shape, blk.basis.order, blk.state, blk.n_components) == (shape, P, state, ncomp)
        assert blk.interleave_width == 3
        assert np.array_equal(blk.get_elements(), vals[f"block{k}"])
    assert fld.blocks[2].geometry_class is sk.GeometryClass.REGULAR
    out = tmp_path / "again.spkf"
    sk.save_field(fld, str(out))
    assert out.read_bytes() == open(os.path.join(GOLD, "field_ref.spkf"), "rb").read()


def test_geometry_rebuilt_from_seed():
    fld = sk.load_field(os.path.join(GOLD, "field_ref.spkf"), seed=5, interleave_width=1)
    blk = fld.blocks[1]
    fac = sk.make_synthetic_factors(blk.basis, sk.GeometryClass.DEFORMED, blk.n_elements, seed=6)
    assert np.array_equal(np.asarray(blk.factors.params), np.asarray(fac.params))


def test_bad_dumps(tmp_path):
    p = tmp_path / "bad.spkf"
    p.write_bytes(b"XXXX\x01\x00\x00\x00")
    with pytest.raises(ValueError):
        sk.load_field(str(p))
    p.write_bytes(b"SPKF\x02\x00\x00\x00")
    with pytest.raises(ValueError):
        sk.load_field(str(p))


def test_interleave_round_trip():
    fld = sk.load_field(os.path.join(GOLD, "field_ref.spkf"), seed=5, interleave_width=1)
    blk = fld.blocks[1]
    w = sk.interleave(blk, 4)
    assert w.interleave_width == 4 and np.array_equal(w.get_elements(), blk.get_elements())
    back = sk.deinterleave(w)
    assert back.interleave_width == 1 and np.array_equal(back.host(), blk.host())


def test_cli_config_errors_cpu():
    """Configuration errors exit 2 before any device work (cli.py:307-315)."""
    from paper_2604_04644_b200.cli import main

    assert main(["bench", "--op", "nope"]) == 2
    assert main(["bench", "--reps", "2"]) == 2
    assert main(["bench", "--order", "0"]) == 2
