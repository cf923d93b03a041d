"""CPU checks of the tet C0 assembly restatement (oracle/assembly.py): with
every Kuhn tet's vertices in global-id order the unsigned map is conforming
-- neighbouring tets' expansions of a random global vector agree on every
shared face -- and the assembled operator (w|det J| for the reflected half)
has the C0 invariants."""

import numpy as np
import pytest

import oracle.assembly as A
from oracle.elements import mode_set


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5])
def test_tet_map_is_conforming(P):
    nx, ny, nz = 2, 2, 2
    tets, _ = A._tet_topology(nx, ny, nz)
    l2g, ls, _ = A._tet_numbering(nx, ny, nz, P)
    x = np.random.default_rng(P).standard_normal(ls[2 * nz + 1])
    owners: dict = {}
    for e, t in enumerate(tets):
        for loc in ((0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)):
            owners.setdefault(tuple(t[i] for i in loc), []).append((e, loc))
    bary = np.array([[0.2, 0.3, 0.5], [0.6, 0.25, 0.15], [0.1, 0.1, 0.8], [0.45, 0.45, 0.1], [1 / 3, 1 / 3, 1 / 3]])
    shared = 0
    for face, own in owners.items():
        if len(own) < 2:
            continue
        assert len(own) == 2
        shared += 1
        vals = []
        for e, loc in own:
            xi = bary @ A.TET_REF[list(loc)]
            vals.append(A.tet_eval(P, x[l2g[e]], A.tet_collapse(xi)))
        assert np.allclose(vals[0], vals[1], rtol=0, atol=1e-12 * max(1.0, np.abs(vals[0]).max())), (face, P)
    assert shared > 0


@pytest.mark.parametrize("P", [1, 2, 3])
def test_tet_numbering_levels(P):
    """Each slab of cube layers owns a contiguous dof range whose first and
    last plane are shared with its neighbours (the NCCL exchange layers)."""
    nx, ny, nz = 2, 3, 3
    tets, _ = A._tet_topology(nx, ny, nz)
    l2g, ls, plane = A._tet_numbering(nx, ny, nz, P)
    assert plane == (nx * P + 1) * (ny * P + 1)
    per = nx * ny * 6
    for iz in range(nz):
        blk = l2g[iz * per:(iz + 1) * per]
        assert blk.min() == ls[2 * iz] and blk.max() == ls[2 * iz + 3] - 1
        assert ls[2 * iz + 1] - ls[2 * iz] == plane
    assert len(np.unique(l2g)) == ls[2 * nz + 1]


@pytest.mark.parametrize("P", [1, 2, 3])
def test_tet_assembled_invariants(P):
    nx, ny, nz = 2, 2, 2
    n = A.tet_n_global(nx, ny, nz, P)
    l2g, _, _ = A._tet_numbering(nx, ny, nz, P)
    vert = [m for m, (p, q, r) in enumerate(mode_set("tet", P)) if (p, q, r) in ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1))]
    one = np.zeros(n)
    one[l2g[:, vert].ravel()] = 1.0
    assert np.max(np.abs(A.assembled_helmholtz_tet(nx, ny, nz, P, one, 0.0))) <= 1e-11
    vol = one @ A.assembled_helmholtz_tet(nx, ny, nz, P, one, 1.0)
    # the deformed box keeps its volume up to O(amp^3); P=1 geometry is a
    # 3x2x2-point collocation of the map (8.017 at P=1, 7.9998 at P=2)
    assert abs(vol - nx * ny * nz) <= (3e-3 if P == 1 else 1e-4) * nx * ny * nz
    rng = np.random.default_rng(2)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    a = u @ A.assembled_helmholtz_tet(nx, ny, nz, P, v, 0.9)
    b = v @ A.assembled_helmholtz_tet(nx, ny, nz, P, u, 0.9)
    assert abs(a - b) <= 1e-11 * abs(a)


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_product_tet_numbering_matches_oracle(P, world):
    """The package's vectorised slab numbering (C0TetMesh, host side) equals
    the oracle's global numbering restricted to every rank's slab."""
    from paper_2604_04644_b200.assembly import _tet_maps
    from paper_2604_04644_b200.sharding import partition

    nx, ny, nz = 2, 3, 4
    l2g_o, ls, plane = A._tet_numbering(nx, ny, nz, P)
    per = nx * ny * 6
    for r in range(world):
        z0, nzl = partition(nz, world, r)
        _, l2g, n, layer = _tet_maps(nx, ny, nz, z0, nzl, P)
        assert layer == plane
        assert np.array_equal(l2g, l2g_o[z0 * per:(z0 + nzl) * per] - ls[2 * z0])
        assert n == ls[2 * (z0 + nzl) + 1] - ls[2 * z0]


@pytest.mark.parametrize("P", [1, 3, 5])
def test_product_prism_numbering_matches_oracle(P):
    from paper_2604_04644_b200.assembly import _prism_tri_maps

    tris, _, dof, sgn, n2d = _prism_tri_maps(3, 2, P)
    od, on = A._tri_dofs(3, 2, P)
    assert on == n2d
    for t in range(len(od)):
        for k, (g, s) in od[t].items():
            assert dof[k][t] == g and sgn[k][t] == s
