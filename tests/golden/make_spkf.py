"""Generate an SPKF field dump with the unmodified reference (its own
make_field / save_field, field_block.py:388-463):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_spkf.py

Writes tests/golden/field_ref.spkf (hex P=2 COEFF 3 elements, tet P=3 COEFF
2 elements x 2 components, prism P=1 PHYS regular 2 elements) plus the
element values it holds (field_ref.npz) for the round-trip tests."""

import os

import numpy as np
from speckern.field_block import Field, make_field, save_field
from speckern.geometry import GeometryClass
from speckern.field_block import FieldState
from speckern.shapes import Shape

HERE = os.path.dirname(os.path.abspath(__file__))

a = make_field([Shape.HEX], 2, GeometryClass.DEFORMED, 3, FieldState.COEFF, 1, 1, seed=5)
b = make_field([Shape.TET], 3, GeometryClass.DEFORMED, 2, FieldState.COEFF, 2, 4, seed=6)
c = make_field([Shape.PRISM], 1, GeometryClass.REGULAR, 2, FieldState.COEFF, 1, 2, seed=7)
rng = np.random.default_rng(11)
vals = {}
for k, blk in enumerate(a.blocks + b.blocks + c.blocks):
    x = rng.uniform(-1, 1, (blk.n_components, blk.n_data, blk.n_elements))
    blk.set_elements(x)
    vals[f"block{k}"] = x
fld = Field(a.blocks + b.blocks + c.blocks)
save_field(fld, os.path.join(HERE, "field_ref.spkf"))
np.savez(os.path.join(HERE, "field_ref.npz"), **vals)
print("wrote field_ref.spkf")
