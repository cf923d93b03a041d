"""CPU oracle for the matrix-free spectral/hp operator path -- TEST INFRASTRUCTURE.

This package is a numpy restatement of the reference ``speckern`` algorithms
(``/root/reference/pkg/src/speckern``) for the hot path: 1D bases and rules,
shape tables, synthetic geometry, the sum-factorised operators and the dense
quadrature-sum oracle.  Every function cites the reference ``file:line`` it
restates.

It is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product path
(``paper_2604_04644_b200``) never imports, calls or links anything here and
fails loudly when its CUDA library is missing.

Parity pinning: ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors in ``tests/golden/`` that were produced by importing
the real reference (``tests/golden/make_golden.py``).  The restatement
evaluates the reference's lane-major kernels with one group of width E
(layout ``(n_data, E)``), which is the reference algorithm at
``interleave_width = E``.
"""

from oracle.basis1d import (  # noqa: F401
    GLL,
    GRJ1,
    GRJ2,
    jacobi,
    quad_rule,
    diff_matrix,
    psi_a,
    psi_a_d,
    psi_b,
    psi_b_d,
)
from oracle.elements import (  # noqa: F401
    SHAPES,
    SHAPE_INDEX,
    RefElement,
    element,
    mode_count,
    qcounts,
    mode_set,
)
from oracle.geom import (  # noqa: F401
    Geometry,
    affine_geometry,
    deformed_geometry_from_coords,
    synthetic_geometry,
    synthetic_affine_vertices,
    deformation_params,
    quadrature_xi,
    payload_lam,
    payload_w,
    payload_dxi,
)
from oracle.ops import (  # noqa: F401
    bwd,
    bwdt,
    colloc,
    bwd_trans,
    iproduct_wrt_base,
    phys_deriv,
    iproduct_wrt_deriv_base,
    mass,
    helmholtz_coll,
    helmholtz_noncoll,
    flops,
    bytes_per_element,
    rel_diff,
    bench_coeffs,
)
from oracle.dense import dense_mass, dense_helmholtz, dense_helmholtz_factored  # noqa: F401
