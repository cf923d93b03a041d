"""End-to-end drop-in check with the UNMODIFIED reference: real speckern
Blocks (installed in baseline/_ref, never /root/reference) driven through the
reference-side ctypes binding in integration/speckern_sk200.py; the result
must equal speckern's own SUM_FAC operator output to 1e-12."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def speckern():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "speckern")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import speckern

    return speckern


@pytest.mark.parametrize("shape", ["HEX", "PRISM", "PYR", "TET"])
@pytest.mark.parametrize("gcls", ["REGULAR", "DEFORMED"])
def test_reference_blocks_through_binding(speckern, shape, gcls):
    import speckern_sk200 as binding
    from speckern.field_block import make_field
    from speckern.geometry import GeometryClass
    from speckern.operators import Strategy, helmholtz_apply_coll, mass_apply
    from speckern.shapes import Shape

    field = make_field(Shape[shape], 4, GeometryClass[gcls], 50, interleave_width=8, seed=2)
    blk = field.blocks[0]
    rng = np.random.default_rng(0)
    blk.set_elements(rng.uniform(-1, 1, (blk.n_data, blk.n_elements)))
    for lam in (0.0, 1.0):
        ref = helmholtz_apply_coll(blk, lam, Strategy.SUM_FAC).get_elements()
        got = binding.helmholtz_apply(blk, lam).get_elements()
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    ref = mass_apply(blk, Strategy.SUM_FAC).get_elements()
    got = binding.mass_apply(blk).get_elements()
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
